"""Host-side mirror of the reference codec API (ref proj/core/include/acz/codec.hpp,
huffman.hpp, tensor.hpp, error.hpp) over the B200 C-ABI (include/acz_gpu.h).

Same names, argument meaning and error behaviour as the reference:

=====================================  ==============================================
reference (proj/core)                  here
=====================================  ==============================================
``Predictor`` codec.hpp:12-15          :class:`Predictor`
``CodecParams`` codec.hpp:17-23        :class:`CodecParams` (``validate`` -> ParamError)
``CompressedTensor`` codec.hpp:32-47   :class:`CompressedTensor` (device blob handle)
``compress`` codec.hpp:54              :func:`compress` (torch CUDA fp32 in)
``decompress`` codec.hpp:59            :func:`decompress` (torch CUDA fp32 out)
``compression_ratio`` codec.hpp:61     :func:`compression_ratio`
``blob_to_bytes/from_bytes`` :69-70    :func:`blob_to_bytes` / :func:`blob_from_bytes`
``huffman_encode/decode`` huffman.hpp  :func:`huffman_encode` / :func:`huffman_decode`
``nonzero_ratio/mean_abs`` tensor.hpp  :func:`nonzero_ratio` / :func:`mean_abs`
``Error`` hierarchy error.hpp:9-53     :class:`Error` and subclasses
=====================================  ==============================================

Every call goes to hand-written sm_100a kernels; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native
from ._native import BlobInfo


# ----------------------------------------------------------------------- errors ----
class Error(RuntimeError):
    """Base class (ref include/acz/error.hpp:9)."""


class ShapeError(Error):
    pass


class DomainError(Error):
    pass


class ParamError(Error):
    pass


class FormatError(Error):
    pass


class DecodeError(Error):
    pass


class CudaError(Error):
    pass


_STATUS = {1: ParamError, 2: DomainError, 3: FormatError, 4: DecodeError, 5: ShapeError,
           6: CudaError, 7: MemoryError, 8: ValueError}


def _check(rc: int, ctx: "Context") -> None:
    if rc:
        msg = _native.load().acz_gpu_last_error(ctx.handle)
        msg = msg.decode() if msg else ""
        raise _STATUS.get(rc, Error)(msg)


# ------------------------------------------------------------------------ params ----
class Predictor(enum.IntEnum):
    PrevValue = 0   # previous reconstructed value in the per-plane scan
    Lorenzo2d = 1   # left + top - top-left within each trailing 2-D plane


@dataclass
class CodecParams:
    eb: float = 1e-4
    quant_radius: int = 32768
    predictor: Predictor = Predictor.PrevValue

    def validate(self) -> None:
        """ref src/codec.cpp:54-59"""
        import math
        if not (self.eb > 0.0) or not math.isfinite(self.eb):
            raise ParamError("error bound must be positive")
        r = int(self.quant_radius)
        if r < 2 or r > (1 << 24) or (r & (r - 1)) != 0:
            raise ParamError("quant_radius must be a power of two in [2, 2^24]")


# ----------------------------------------------------------------------- context ----
class Context:
    """One C-ABI context per (device, thread)."""

    def __init__(self, device: int = 0):
        lib = _native.load()
        h = C.c_void_p()
        rc = lib.acz_gpu_ctx_create(device, C.byref(h))
        if rc:
            raise CudaError(f"acz_gpu_ctx_create failed ({rc}): is a CUDA device visible?")
        self.handle = h
        self.device = device

    def __del__(self):
        try:
            if self.handle:
                _native.load().acz_gpu_ctx_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(_native.load().acz_gpu_launch_count(self.handle))

    def memory_info(self, reset_peak: bool = False) -> dict:
        """Device memory held by the codec: this context's workspace, and the live / peak
        bytes of blobs in the process (acz_gpu_memory_info)."""
        ws, live, peak = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(_native.load().acz_gpu_memory_info(self.handle, C.byref(ws), C.byref(live),
                                                  C.byref(peak), int(reset_peak)), self)
        br = (C.c_uint64 * 6)()
        _check(_native.load().acz_gpu_memory_breakdown(self.handle, br, 6), self)
        names = ["symbols", "tables", "quant", "encode", "staging", "decode"]
        return {"workspace_bytes": int(ws.value), "blob_live_bytes": int(live.value),
                "blob_peak_bytes": int(peak.value),
                "workspace_breakdown": {k: int(v) for k, v in zip(names, br)}}

    def trim(self) -> None:
        """Free every workspace of this context (acz_gpu_ctx_trim); blobs are unaffected."""
        _check(_native.load().acz_gpu_ctx_trim(self.handle), self)


_tls = threading.local()


def default_context(device: Optional[int] = None) -> Context:
    import torch
    dev = torch.cuda.current_device() if device is None else device
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    if dev not in cache:
        cache[dev] = Context(dev)
    return cache[dev]


def _stream_handle(stream) -> C.c_void_p:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _dev_ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def _require_cuda_f32(t, name: str = "tensor"):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA torch.Tensor (no CPU path)")
    if t.dtype != torch.float32:
        raise TypeError(f"{name} must be float32")
    return t.contiguous()


# ------------------------------------------------------------- CompressedTensor ----
@dataclass
class CodebookEntry:
    symbol: int
    length: int


@dataclass
class Outlier:
    index: int
    value: float


class CompressedTensor:
    """Device-resident compressed blob (ref include/acz/codec.hpp:32-47). Owns its device
    buffers (canonical codebook, bitstream, outliers, decode sidecar)."""

    def __init__(self, handle: C.c_void_p, ctx: Context):
        self._h = handle
        self._ctx = ctx
        info = BlobInfo()
        _check(_native.load().acz_gpu_blob_info(handle, C.byref(info)), ctx)
        self._info = info
        self._bytes: Optional[bytes] = None

    def __del__(self):
        try:
            if self._h:
                _native.load().acz_gpu_blob_free(self._h)
                self._h = None
        except Exception:
            pass

    # scalar fields ------------------------------------------------------------
    @property
    def shape(self) -> Tuple[int, ...]:
        return tuple(int(self._info.shape[i]) for i in range(self._info.rank))

    @property
    def params(self) -> CodecParams:
        return CodecParams(self._info.eb, int(self._info.quant_radius),
                           Predictor(self._info.predictor))

    def element_count(self) -> int:
        return int(self._info.element_count)

    @property
    def bit_length(self) -> int:
        return int(self._info.bit_length)

    @property
    def uncompressed_bytes(self) -> int:
        return int(self._info.uncompressed_bytes)

    @property
    def compressed_bytes(self) -> int:
        return int(self._info.compressed_bytes)

    @property
    def device_bytes(self) -> int:
        return int(self._info.device_bytes)

    @property
    def sidecar_bytes(self) -> int:
        return int(self._info.sidecar_bytes)

    @property
    def codebook_size(self) -> int:
        return int(self._info.codebook_size)

    @property
    def outlier_count(self) -> int:
        return int(self._info.outlier_count)

    @property
    def max_code_length(self) -> int:
        return int(self._info.max_code_length)

    # array fields (parsed from the ACZ1 image) -----------------------------------
    def to_bytes(self, stream=None) -> bytes:
        if self._bytes is None:
            n = self.compressed_bytes
            buf = (C.c_uint8 * n)()
            w = C.c_uint64()
            _check(_native.load().acz_gpu_blob_to_host(self._ctx.handle, self._h, buf, n,
                                                       C.byref(w), _stream_handle(stream)),
                   self._ctx)
            self._bytes = bytes(buf)
        return self._bytes

    def sidecar(self, stream=None) -> bytes:
        n = self.sidecar_bytes
        buf = (C.c_uint8 * n)()
        w = C.c_uint64()
        _check(_native.load().acz_gpu_sidecar_to_host(self._ctx.handle, self._h, buf, n,
                                                      C.byref(w), _stream_handle(stream)),
               self._ctx)
        return bytes(buf)

    def _parsed(self):
        return parse_acz1(self.to_bytes())

    @property
    def codebook(self) -> List[CodebookEntry]:
        p = self._parsed()
        return [CodebookEntry(int(s), int(l)) for s, l in zip(p["book_sym"], p["book_len"])]

    @property
    def bitstream(self) -> bytes:
        return self._parsed()["bits"]

    @property
    def outliers(self) -> List[Outlier]:
        p = self._parsed()
        return [Outlier(int(i), float(v)) for i, v in zip(p["out_index"], p["out_value"])]


def parse_acz1(b: bytes) -> dict:
    """Field view of an ACZ1 image (format: ref include/acz/codec.hpp:63-68)."""
    mv = memoryview(b)
    pos = 0

    def take(fmt_n, dtype):
        nonlocal pos
        a = np.frombuffer(mv[pos:pos + fmt_n * np.dtype(dtype).itemsize], dtype=dtype)
        pos += fmt_n * np.dtype(dtype).itemsize
        return a

    assert bytes(mv[:4]) == b"ACZ1"
    pos = 4
    version, pred, rank = take(3, np.uint8)
    shape = take(int(rank), "<u8")
    eb = float(take(1, "<f8")[0])
    radius = int(take(1, "<u4")[0])
    nout = int(take(1, "<u4")[0])
    k = int(take(1, "<u2")[0])
    book = np.frombuffer(mv[pos:pos + 5 * k], dtype=np.dtype([("s", "<u4"), ("l", "u1")]))
    pos += 5 * k
    bit_length = int(take(1, "<u8")[0])
    nbytes = (bit_length + 7) // 8
    bits = bytes(mv[pos:pos + nbytes])
    pos += nbytes
    outl = np.frombuffer(mv[pos:pos + 12 * nout], dtype=np.dtype([("i", "<u8"), ("v", "<f4")]))
    return dict(version=int(version), predictor=int(pred), shape=tuple(int(s) for s in shape),
                eb=eb, quant_radius=radius, book_sym=book["s"].copy(), book_len=book["l"].copy(),
                bit_length=bit_length, bits=bits, out_index=outl["i"].copy(),
                out_value=outl["v"].copy())


# ---------------------------------------------------------------------- codec API ----
def compress(t, p: CodecParams = CodecParams(), stream=None,
             ctx: Optional[Context] = None) -> CompressedTensor:
    """ref include/acz/codec.hpp:54 / src/codec.cpp:61-120."""
    t = _require_cuda_f32(t)
    ctx = ctx or default_context(t.device.index)
    shape = (C.c_uint64 * max(1, t.dim()))(*t.shape)
    h = C.c_void_p()
    rc = _native.load().acz_gpu_compress(ctx.handle, _dev_ptr(t), shape, t.dim(), float(p.eb),
                                         int(p.quant_radius), int(p.predictor),
                                         _stream_handle(stream), C.byref(h))
    _check(rc, ctx)
    return CompressedTensor(h, ctx)


class AsyncCompress:
    """An asynchronous compress in flight (acz_gpu_compress_async): nothing waits for the
    GPU until :meth:`settle`. The input tensor is kept referenced until then, so that a
    blob that outgrew its predicted size can be compressed again from it."""

    def __init__(self, t, p: CodecParams, stream, ctx: "Context", h, pending: bool):
        self._ctx, self._p, self._stream = ctx, p, stream
        self._h = h if pending else None
        self._t = t if pending else None
        self.result: Optional[CompressedTensor] = None if pending else CompressedTensor(h, ctx)
        self.refits = 0
        self.refit_reason = ""

    @property
    def pending(self) -> bool:
        return self.result is None

    def settle(self, wait: bool = True) -> Optional[CompressedTensor]:
        """The CompressedTensor (bit-identical to :func:`compress`), or None while the
        compress has not finished (wait=False). Raises the errors compress() raises."""
        if self.result is not None:
            return self.result
        st = C.c_int(0)
        lib = _native.load()
        rc = lib.acz_gpu_compress_settle(self._ctx.handle, self._h, int(bool(wait)), C.byref(st))
        if rc == 0 and st.value == 0:
            return None
        if rc == 0 and st.value == 1:
            self.result = CompressedTensor(self._h, self._ctx)
            self._h = self._t = None
            return self.result
        # did not fit its predicted size (or failed): free it, compress synchronously
        if rc == 0:
            msg = lib.acz_gpu_last_error(self._ctx.handle)
            self.refit_reason = msg.decode() if msg else ""
        lib.acz_gpu_blob_free(self._h)
        self._h = None
        self.refits += 1
        self.result = compress(self._t, self._p, stream=self._stream, ctx=self._ctx)
        if self._stream is not None:
            # its encode reads the input on that stream; the caller may free the input and
            # use the blob on another stream once this returns
            self._stream.synchronize()
        self._t = None
        return self.result

    def __del__(self):
        try:
            if self._h:
                _native.load().acz_gpu_blob_free(self._h)
                self._h = None
        except Exception:
            pass


def compress_async(t, p: CodecParams = CodecParams(), stream=None,
                   ctx: Optional[Context] = None, size_tag: int = 0) -> AsyncCompress:
    """:func:`compress` without the host wait for the codebook (the training hooks' per-layer
    path): once a tensor of the same shape and parameters was compressed on this context,
    the whole compress is enqueued on the stream and the blob is sized from that earlier
    one (acz_gpu_compress_async; size_tag, e.g. a layer id, keeps the predictions of
    equally shaped tensors apart). Settle the result before using it."""
    t = _require_cuda_f32(t)
    ctx = ctx or default_context(t.device.index)
    shape = (C.c_uint64 * max(1, t.dim()))(*t.shape)
    h = C.c_void_p()
    pend = C.c_int(0)
    rc = _native.load().acz_gpu_compress_async(ctx.handle, _dev_ptr(t), shape, t.dim(),
                                               float(p.eb), int(p.quant_radius),
                                               int(p.predictor), int(size_tag),
                                               _stream_handle(stream), C.byref(h),
                                               C.byref(pend))
    _check(rc, ctx)
    return AsyncCompress(t, p, stream, ctx, h, bool(pend.value))


def decompress(c: CompressedTensor, zero_filter: bool = False, out=None, stream=None,
               ctx: Optional[Context] = None):
    """ref include/acz/codec.hpp:59 / src/codec.cpp:122-171. Returns a CUDA fp32 tensor.
    (ctx: accepted for symmetry; the blob's own context runs the decode.)"""
    import torch
    if out is None:
        out = torch.empty(c.shape, dtype=torch.float32, device=f"cuda:{c._ctx.device}")
    else:
        out = _require_cuda_f32(out, "out")
        if out.numel() != c.element_count():
            raise ShapeError("output size mismatch")
    rc = _native.load().acz_gpu_decompress(c._ctx.handle, c._h, int(bool(zero_filter)),
                                           _dev_ptr(out), _stream_handle(stream))
    _check(rc, c._ctx)
    return out


def compress_many(tensors: Sequence, p: CodecParams = CodecParams(), stream=None,
                  ctx: Optional[Context] = None, errors: str = "raise") -> List[Optional[CompressedTensor]]:
    """Batched :func:`compress` of a whole activation set (one call per training step, as
    Controller::wrap_forward does per conv layer, ref src/controller.cpp:194-230). The
    tensors' kernels overlap on the context's internal streams. errors="raise" raises the
    first failure; errors="none" returns None for failing tensors (the reference controller
    degrades such layers to pass-through, src/controller.cpp:216-220)."""
    ts = [_require_cuda_f32(t) for t in tensors]
    if not ts:
        return []
    ctx = ctx or default_context(ts[0].device.index)
    k = len(ts)
    ptrs = (C.c_void_p * k)(*[t.data_ptr() for t in ts])
    ranks = (C.c_uint32 * k)(*[t.dim() for t in ts])
    flat = [int(e) for t in ts for e in t.shape]
    shapes = (C.c_uint64 * max(1, len(flat)))(*flat)
    outs = (C.c_void_p * k)()
    status = (C.c_int * k)()
    rc = _native.load().acz_gpu_compress_batch(ctx.handle, k, ptrs, shapes, ranks, float(p.eb),
                                               int(p.quant_radius), int(p.predictor),
                                               _stream_handle(stream), outs, status)
    res = [CompressedTensor(C.c_void_p(outs[i]), ctx) if outs[i] else None for i in range(k)]
    if rc and errors == "raise":
        _check(rc, ctx)
    return res


def decompress_many(blobs: Sequence[CompressedTensor], zero_filter: bool = False, outs=None,
                    stream=None):
    """Batched :func:`decompress` (ref Controller::unwrap_backward, src/controller.cpp:234-249)."""
    import torch
    if not blobs:
        return []
    ctx = blobs[0]._ctx
    if outs is None:
        outs = [torch.empty(c.shape, dtype=torch.float32, device=f"cuda:{ctx.device}")
                for c in blobs]
    outs = [_require_cuda_f32(o, "out") for o in outs]
    for c, o in zip(blobs, outs):
        if o.numel() != c.element_count():
            raise ShapeError("output size mismatch")
    k = len(blobs)
    hs = (C.c_void_p * k)(*[c._h.value for c in blobs])
    ps = (C.c_void_p * k)(*[o.data_ptr() for o in outs])
    rc = _native.load().acz_gpu_decompress_batch(ctx.handle, k, hs, int(bool(zero_filter)), ps,
                                                 _stream_handle(stream))
    _check(rc, ctx)
    return outs


def relu_(t, stream=None, ctx: Optional[Context] = None):
    """In-place x = x > 0 ? x : 0 on the GPU (ref nn::recompute_relu,
    include/acz/nn/layers.hpp:134-157): the controller's relu-recompute zero restoration
    after an unfiltered decompress (src/controller.cpp:210-213,244)."""
    t2 = _require_cuda_f32(t)
    if t2.data_ptr() != t.data_ptr():
        raise ValueError("relu_ needs a contiguous tensor")
    ctx = ctx or default_context(t.device.index)
    _check(_native.load().acz_gpu_relu(ctx.handle, _dev_ptr(t), t.numel(),
                                       _stream_handle(stream)), ctx)
    return t


def compression_ratio(c: CompressedTensor) -> float:
    """ref src/codec.cpp:173-175"""
    return c.uncompressed_bytes / c.compressed_bytes


def blob_to_bytes(c: CompressedTensor) -> bytes:
    return c.to_bytes()


def blob_from_bytes(data: bytes, sidecar: Optional[bytes] = None, stream=None,
                    ctx: Optional[Context] = None) -> CompressedTensor:
    """ref src/codec.cpp:201-262 (same validation and FormatError messages)."""
    ctx = ctx or default_context()
    buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data or b"\0")
    sbuf = None
    if sidecar:
        sbuf = (C.c_uint8 * len(sidecar)).from_buffer_copy(sidecar)
    h = C.c_void_p()
    rc = _native.load().acz_gpu_blob_from_host(ctx.handle, buf, len(data), sbuf,
                                               len(sidecar) if sidecar else 0,
                                               _stream_handle(stream), C.byref(h))
    _check(rc, ctx)
    return CompressedTensor(h, ctx)


def compress_host(x: np.ndarray, p: CodecParams = CodecParams(), shape=None,
                  ctx: Optional[Context] = None, want_sidecar: bool = True):
    """Host tensor in, (ACZ1 bytes, sidecar bytes) out: the reference's own calling
    convention (compress on a host Tensor, blob_to_bytes)."""
    ctx = ctx or default_context()
    x = np.ascontiguousarray(x, dtype=np.float32)
    shp = tuple(x.shape) if shape is None else tuple(shape)
    cshape = (C.c_uint64 * max(1, len(shp)))(*shp)
    pa, ps = C.c_void_p(), C.c_void_p()
    na, ns = C.c_uint64(), C.c_uint64()
    lib = _native.load()
    rc = lib.acz_gpu_compress_host(ctx.handle, C.c_void_p(x.ctypes.data), cshape, len(shp),
                                   float(p.eb), int(p.quant_radius), int(p.predictor),
                                   C.byref(pa), C.byref(na),
                                   C.byref(ps) if want_sidecar else None,
                                   C.byref(ns) if want_sidecar else None)
    _check(rc, ctx)
    blob = C.string_at(pa, na.value)
    lib.acz_gpu_host_free(pa)
    side = None
    if want_sidecar:
        side = C.string_at(ps, ns.value)
        lib.acz_gpu_host_free(ps)
    return blob, side


def decompress_host(blob: bytes, n: int, zero_filter: bool = False,
                    sidecar: Optional[bytes] = None, out: Optional[np.ndarray] = None,
                    ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx or default_context()
    if out is None:
        out = np.empty(n, dtype=np.float32)
    buf = (C.c_uint8 * max(1, len(blob))).from_buffer_copy(blob or b"\0")
    sbuf = (C.c_uint8 * len(sidecar)).from_buffer_copy(sidecar) if sidecar else None
    rc = _native.load().acz_gpu_decompress_host(ctx.handle, buf, len(blob), sbuf,
                                                len(sidecar) if sidecar else 0,
                                                int(bool(zero_filter)),
                                                C.c_void_p(out.ctypes.data), n)
    _check(rc, ctx)
    return out


def compress_host_many(hosts: Sequence, p: CodecParams = CodecParams(), blob_bufs=None,
                       side_bufs=None, ctx: Optional[Context] = None, stream=None):
    """Host-buffer compress of a whole activation set (acz_gpu_compress_host_batch): host
    fp32 tensors in (page-locked torch tensors upload at full PCIe speed), ACZ1 bytes +
    decode sidecars out. Each tensor's upload and kernels run on its own stream, so the
    compression of tensor i overlaps the upload of tensor i+1. blob_bufs / side_bufs
    (optional page-locked torch uint8 tensors; default: allocated at 5 B / element) receive
    the bytes. Returns [(ACZ1 view, sidecar view)] as numpy uint8 arrays."""
    import torch
    ctx = ctx or default_context()
    if stream is not None:
        stream.synchronize()
    hs = [torch.as_tensor(h) for h in hosts]
    k = len(hs)
    if k == 0:
        return []
    for h in hs:
        if h.dtype != torch.float32 or not h.is_contiguous() or h.is_cuda:
            raise ValueError("host tensors must be contiguous fp32 CPU tensors")
    if blob_bufs is None:
        blob_bufs = [torch.empty(5 * h.numel() + (1 << 20), dtype=torch.uint8, pin_memory=True)
                     for h in hs]
    if side_bufs is None:
        side_bufs = [torch.empty(h.numel() // 8 + (1 << 20), dtype=torch.uint8, pin_memory=True)
                     for h in hs]
    blob_bufs, side_bufs = list(blob_bufs), list(side_bufs)
    sizes_b, sizes_s = [0] * k, [0] * k

    def run(idx):
        m = len(idx)
        ptrs = (C.c_void_p * m)(*[hs[i].data_ptr() for i in idx])
        ranks = (C.c_uint32 * m)(*[hs[i].dim() for i in idx])
        flat = [int(e) for i in idx for e in hs[i].shape]
        shapes = (C.c_uint64 * max(1, len(flat)))(*flat)
        bp = (C.c_void_p * m)(*[blob_bufs[i].data_ptr() for i in idx])
        bc = (C.c_uint64 * m)(*[blob_bufs[i].numel() for i in idx])
        bs = (C.c_uint64 * m)()
        sp = (C.c_void_p * m)(*[side_bufs[i].data_ptr() for i in idx])
        sc = (C.c_uint64 * m)(*[side_bufs[i].numel() for i in idx])
        ss = (C.c_uint64 * m)()
        st = (C.c_int * m)()
        rc = _native.load().acz_gpu_compress_host_batch(ctx.handle, m, ptrs, shapes, ranks,
                                                        float(p.eb), int(p.quant_radius),
                                                        int(p.predictor), bp, bc, bs, sp, sc, ss,
                                                        st)
        for j, i in enumerate(idx):
            sizes_b[i], sizes_s[i] = int(bs[j]), int(ss[j])
        return rc, [int(st[j]) for j in range(m)]

    rc, st = run(list(range(k)))
    if rc:
        # a destination smaller than the blob (small error bounds: mostly outliers, up to
        # 12 B + the code per element) reports the size it needs: grow those buffers, redo
        # only those tensors
        retry = [i for i in range(k) if st[i] == 8 and (sizes_b[i] > blob_bufs[i].numel() or
                                                        sizes_s[i] > side_bufs[i].numel())]
        if retry and all(st[i] in (0, 8) for i in range(k)):
            for i in retry:
                if sizes_b[i] > blob_bufs[i].numel():
                    blob_bufs[i] = torch.empty(sizes_b[i], dtype=torch.uint8, pin_memory=True)
                if sizes_s[i] > side_bufs[i].numel():
                    side_bufs[i] = torch.empty(sizes_s[i], dtype=torch.uint8, pin_memory=True)
            rc, st2 = run(retry)
        _check(rc, ctx)
    return [(blob_bufs[i][:sizes_b[i]].numpy(), side_bufs[i][:sizes_s[i]].numpy())
            for i in range(k)]


def decompress_host_many(blobs, zero_filter: bool = False, outs=None,
                         ctx: Optional[Context] = None, stream=None):
    """Host-buffer decompress of a whole activation set (acz_gpu_decompress_host_batch):
    [(ACZ1 bytes, sidecar or None)] (numpy uint8 arrays; page-locked memory copies at full
    PCIe speed) in, host fp32 tensors out (outs: optional page-locked torch tensors,
    default: allocated). Parses + validates like ref blob_from_bytes; uploads, decodes and
    downloads overlap across tensors. Raises the first failure's exception."""
    import torch
    ctx = ctx or default_context()
    if stream is not None:
        stream.synchronize()
    k = len(blobs)
    if k == 0:
        return []
    arrs = [np.ascontiguousarray(b, dtype=np.uint8) for b, _ in blobs]
    sides = [None if sd is None or len(sd) == 0 else np.ascontiguousarray(sd, dtype=np.uint8)
             for _, sd in blobs]
    if outs is None:
        outs = []
        for a in arrs:
            shape = _acz1_shape(a)
            outs.append(torch.empty(shape, dtype=torch.float32, pin_memory=True))
    ptrs = (C.c_void_p * k)(*[a.ctypes.data for a in arrs])
    sizes = (C.c_uint64 * k)(*[a.size for a in arrs])
    sp = (C.c_void_p * k)(*[sd.ctypes.data if sd is not None else None for sd in sides])
    ss = (C.c_uint64 * k)(*[sd.size if sd is not None else 0 for sd in sides])
    op = (C.c_void_p * k)(*[o.data_ptr() for o in outs])
    oc = (C.c_uint64 * k)(*[o.numel() for o in outs])
    st = (C.c_int * k)()
    rc = _native.load().acz_gpu_decompress_host_batch(ctx.handle, k, ptrs, sizes, sp, ss,
                                                      1 if zero_filter else 0, op, oc, st)
    _check(rc, ctx)
    res = []
    for a, o in zip(arrs, outs):
        res.append(o.view(_acz1_shape(a)) if o.numel() == int(np.prod(_acz1_shape(a))) else o)
    return res


def _acz1_shape(a) -> tuple:
    """Shape from an ACZ1 header (ref src/codec.cpp:179-191 layout); the full validation
    happens in the native parser."""
    if a.size < 7 or bytes(a[:4]) != b"ACZ1":
        raise FormatError("bad blob magic at offset 0 (expected \"ACZ1\")")
    rank = int(a[6])
    if rank == 0 or a.size < 7 + 8 * rank:
        raise FormatError("unexpected end of stream")
    return tuple(int.from_bytes(bytes(a[7 + 8 * i:15 + 8 * i]), "little") for i in range(rank))


# --------------------------------------------------------------------- statistics ----
def zero_bitmap(t, stream=None, ctx: Optional[Context] = None):
    """Fused zero-bitmap + sparsity pass: returns (int32 CUDA tensor of ceil(n/32)
    words, bit i%32 of word i/32 = x[i] != 0; nonzero count)."""
    import torch
    t = _require_cuda_f32(t)
    ctx = ctx or default_context(t.device.index)
    n = t.numel()
    bm = torch.empty((n + 31) // 32, dtype=torch.int32, device=t.device)
    nz = C.c_uint64()
    _check(_native.load().acz_gpu_zero_bitmap(ctx.handle, _dev_ptr(t), n, _dev_ptr(bm),
                                              C.byref(nz), _stream_handle(stream)), ctx)
    return bm, int(nz.value)


def nonzero_ratio(t, stream=None, ctx: Optional[Context] = None) -> float:
    """ref include/acz/tensor.hpp:91-99"""
    t = _require_cuda_f32(t)
    ctx = ctx or default_context(t.device.index)
    r = C.c_double()
    _check(_native.load().acz_gpu_nonzero_ratio(ctx.handle, _dev_ptr(t), t.numel(),
                                                _stream_handle(stream), C.byref(r)), ctx)
    return r.value


def mean_abs(t, stream=None, ctx: Optional[Context] = None) -> float:
    """ref include/acz/tensor.hpp:82-89 (parallel summation order)"""
    t = _require_cuda_f32(t)
    ctx = ctx or default_context(t.device.index)
    r = C.c_double()
    _check(_native.load().acz_gpu_mean_abs(ctx.handle, _dev_ptr(t), t.numel(),
                                           _stream_handle(stream), C.byref(r)), ctx)
    return r.value


# ------------------------------------------------------------------------ Huffman ----
@dataclass
class HuffmanCode:
    """ref include/acz/huffman.hpp:20-24"""
    codebook: List[CodebookEntry]
    bits: bytes
    bit_length: int


def huffman_encode(symbols, stream=None, ctx: Optional[Context] = None) -> HuffmanCode:
    """symbols: CUDA int32/uint32 tensor (values read as u32)."""
    import torch
    if not isinstance(symbols, torch.Tensor) or not symbols.is_cuda:
        raise TypeError("symbols must be a CUDA tensor")
    s = symbols.contiguous()
    if s.element_size() != 4:
        raise TypeError("symbols must be 32-bit")
    ctx = ctx or default_context(s.device.index)
    n = s.numel()
    cap = min(n, 1 << 26) + 1
    bsym = (C.c_uint32 * cap)()
    blen = (C.c_uint8 * cap)()
    bits_cap = 8 * n + 16
    bits = (C.c_uint8 * bits_cap)()
    k = C.c_uint32()
    bl = C.c_uint64()
    _check(_native.load().acz_gpu_huffman_encode(ctx.handle, _dev_ptr(s), n, bsym, blen, cap,
                                                 C.byref(k), bits, bits_cap, C.byref(bl),
                                                 _stream_handle(stream)), ctx)
    book = [CodebookEntry(int(bsym[i]), int(blen[i])) for i in range(k.value)]
    return HuffmanCode(book, bytes(bits)[:(bl.value + 7) // 8], int(bl.value))


def huffman_decode(codebook: Sequence[CodebookEntry], bits: bytes, bit_length: int, count: int,
                   stream=None, ctx: Optional[Context] = None):
    """ref include/acz/huffman.hpp:30-32. Returns a CUDA int32 tensor (u32 values)."""
    import torch
    ctx = ctx or default_context()
    k = len(codebook)
    bsym = (C.c_uint32 * max(1, k))(*[e.symbol for e in codebook])
    blen = (C.c_uint8 * max(1, k))(*[e.length for e in codebook])
    b = (C.c_uint8 * max(1, len(bits))).from_buffer_copy(bits or b"\0")
    out = torch.empty(max(count, 1), dtype=torch.int32, device=f"cuda:{ctx.device}")
    _check(_native.load().acz_gpu_huffman_decode(ctx.handle, bsym, blen, k, b, bit_length, count,
                                                 _dev_ptr(out), _stream_handle(stream)), ctx)
    return out[:count]


def debug_last_symbols(n: int, ctx: Optional[Context] = None):
    """Quantisation symbols of the last compress on the context (parity tests)."""
    import torch
    ctx = ctx or default_context()
    out = torch.empty(n, dtype=torch.int32, device=f"cuda:{ctx.device}")
    _check(_native.load().acz_gpu_debug_last_symbols(ctx.handle, _dev_ptr(out), n,
                                                     _stream_handle(None)), ctx)
    return out
