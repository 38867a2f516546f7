"""TEST INFRASTRUCTURE ONLY -- the parity oracle (ctypes view of oracle/liboracle.so and
oracle/_ref/libacz_ref.so).

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` legs may import this module, and only as the checker or the timed CPU
baseline. The product package (``paper_2011_09017_b200``) never imports it.

* ``Oracle``    -- our plain-C restatement of the reference codec (acz_oracle.c); every
                   function there cites the reference file:line it follows.
* ``Reference`` -- the UNMODIFIED reference codec compiled from its own sources
                   (/root/reference/proj/core/src/{codec,huffman,tensor_io}.cpp) by
                   oracle/Makefile; prebuilt .so travels to the GPU box.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libacz_ref.so")

_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_f32p = C.POINTER(C.c_float)

STATUS_NAMES = {0: "ok", 1: "ParamError", 2: "DomainError", 3: "FormatError",
                4: "DecodeError", 5: "ShapeError", 7: "OutOfMemory", 9: "Error"}


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class _oracle_result(C.Structure):
    _fields_ = [("n", C.c_uint64), ("symbols", _u32p), ("recon", _f32p),
                ("n_outliers", C.c_uint64), ("out_index", _u64p), ("out_value", _f32p),
                ("book_size", C.c_uint32), ("book_sym", _u32p), ("book_len", _u8p),
                ("bit_length", C.c_uint64), ("bits", _u8p), ("blob", _u8p),
                ("blob_size", C.c_uint64)]


@dataclass
class Artifacts:
    """Everything the codec produces for one tensor (SURVEY.md 8(d) parity gates)."""
    symbols: np.ndarray       # uint32 [n]
    recon: np.ndarray         # float32 [n] chain values
    out_index: np.ndarray     # uint64
    out_value: np.ndarray     # float32
    book_sym: np.ndarray      # uint32 canonical order
    book_len: np.ndarray      # uint8
    bit_length: int
    bits: np.ndarray          # uint8 ceil(bit_length/8)
    blob: bytes               # ACZ1


def _copy(p, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(p, shape=(n,)).astype(dtype, copy=True)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.oracle_compress.argtypes = [_f32p, _u64p, C.c_int, C.c_double, C.c_uint32, C.c_int,
                                      C.POINTER(_oracle_result), C.c_char_p, C.c_int]
        L.oracle_result_free.argtypes = [C.POINTER(_oracle_result)]
        L.oracle_compress_mt.argtypes = [_f32p, _u64p, C.c_int, C.c_double, C.c_uint32,
                                         C.c_int, C.c_int, C.POINTER(_oracle_result),
                                         C.c_char_p, C.c_int]
        L.oracle_decompress.argtypes = [_u8p, C.c_uint64, C.c_int, _f32p, C.c_uint64,
                                        C.c_char_p, C.c_int]
        L.oracle_huffman_encode.argtypes = [_u32p, C.c_uint64, C.POINTER(C.c_uint32),
                                            C.POINTER(_u32p), C.POINTER(_u8p),
                                            C.POINTER(_u8p), C.POINTER(C.c_uint64),
                                            C.c_char_p, C.c_int]
        L.oracle_huffman_decode.argtypes = [_u32p, _u8p, C.c_uint32, _u8p, C.c_uint64,
                                            C.c_uint64, _u32p, C.c_char_p, C.c_int]
        L.oracle_nonzero_ratio.argtypes = [_f32p, C.c_uint64]
        L.oracle_nonzero_ratio.restype = C.c_double
        L.oracle_mean_abs.argtypes = [_f32p, C.c_uint64]
        L.oracle_mean_abs.restype = C.c_double
        L.oracle_zero_bitmap.argtypes = [_f32p, C.c_uint64, _u32p]
        L.oracle_zero_bitmap.restype = C.c_uint64
        L.oracle_free.argtypes = [C.c_void_p]
        self.L = L

    def compress(self, x: np.ndarray, eb: float, radius: int = 32768,
                 predictor: int = 0, shape=None) -> Artifacts:
        x = np.ascontiguousarray(x, dtype=np.float32)
        shp = np.asarray(x.shape if shape is None else shape, dtype=np.uint64)
        res = _oracle_result()
        err = C.create_string_buffer(512)
        rc = self.L.oracle_compress(_ptr(x, _f32p), _ptr(shp, _u64p), len(shp), eb, radius,
                                    predictor, C.byref(res), err, 512)
        try:
            if rc:
                raise OracleError(rc, err.value.decode())
            n = res.n
            return Artifacts(
                symbols=_copy(res.symbols, n, np.uint32), recon=_copy(res.recon, n, np.float32),
                out_index=_copy(res.out_index, res.n_outliers, np.uint64),
                out_value=_copy(res.out_value, res.n_outliers, np.float32),
                book_sym=_copy(res.book_sym, res.book_size, np.uint32),
                book_len=_copy(res.book_len, res.book_size, np.uint8),
                bit_length=int(res.bit_length),
                bits=_copy(res.bits, (res.bit_length + 7) // 8, np.uint8),
                blob=bytes(_copy(res.blob, res.blob_size, np.uint8)))
        finally:
            self.L.oracle_result_free(C.byref(res))

    def compress_mt(self, x: np.ndarray, eb: float, radius: int = 32768, predictor: int = 0,
                    threads: Optional[int] = None, symbols: bool = False):
        """oracle_compress on `threads` host threads (same bytes as compress(); the plane
        ranges, counts and bit packing are split and joined in order). Returns
        (ACZ1 blob bytes, chain values float32 [n], symbols uint32 [n] or None). The chain
        values are what decompress reconstructs (ref src/codec.cpp:153-161 repeats the
        compressor's expression), so filter(recon) is the decompressed output."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        shp = np.asarray(x.shape, dtype=np.uint64)
        res = _oracle_result()
        err = C.create_string_buffer(512)
        nt = threads or min(64, os.cpu_count() or 1)
        rc = self.L.oracle_compress_mt(_ptr(x, _f32p), _ptr(shp, _u64p), len(shp), eb, radius,
                                       predictor, nt, C.byref(res), err, 512)
        try:
            if rc:
                raise OracleError(rc, err.value.decode())
            blob = np.ctypeslib.as_array(res.blob, shape=(res.blob_size,)).tobytes()
            recon = _copy(res.recon, res.n, np.float32)
            syms = _copy(res.symbols, res.n, np.uint32) if symbols else None
            return blob, recon, syms
        finally:
            self.L.oracle_result_free(C.byref(res))

    @staticmethod
    def zero_filter(recon: np.ndarray, eb: float) -> np.ndarray:
        """ref src/codec.cpp:162-164: |(double)v| <= eb -> 0.0f (on the chain values)."""
        out = recon.copy()
        out[np.abs(recon.astype(np.float64)) <= eb] = 0.0
        return out

    def decompress(self, blob: bytes, n: int, zero_filter: bool = False) -> np.ndarray:
        b = np.frombuffer(blob, dtype=np.uint8).copy()
        out = np.empty(n, dtype=np.float32)
        err = C.create_string_buffer(512)
        rc = self.L.oracle_decompress(_ptr(b, _u8p), len(b), int(zero_filter), _ptr(out, _f32p),
                                      n, err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out

    def huffman_encode(self, syms: np.ndarray):
        s = np.ascontiguousarray(syms, dtype=np.uint32)
        bs = C.c_uint32()
        psym, plen, pbits = _u32p(), _u8p(), _u8p()
        bl = C.c_uint64()
        err = C.create_string_buffer(512)
        rc = self.L.oracle_huffman_encode(_ptr(s, _u32p), len(s), C.byref(bs), C.byref(psym),
                                          C.byref(plen), C.byref(pbits), C.byref(bl), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        out = (_copy(psym, bs.value, np.uint32), _copy(plen, bs.value, np.uint8),
               _copy(pbits, (bl.value + 7) // 8, np.uint8), bl.value)
        for p in (psym, plen, pbits):
            self.L.oracle_free(C.cast(p, C.c_void_p))
        return out

    def huffman_decode(self, book_sym, book_len, bits, bit_length, count) -> np.ndarray:
        bs = np.ascontiguousarray(book_sym, dtype=np.uint32)
        bl = np.ascontiguousarray(book_len, dtype=np.uint8)
        b = np.ascontiguousarray(bits, dtype=np.uint8)
        if len(b) == 0:
            b = np.zeros(1, dtype=np.uint8)
        out = np.empty(max(count, 1), dtype=np.uint32)
        err = C.create_string_buffer(512)
        rc = self.L.oracle_huffman_decode(_ptr(bs, _u32p), _ptr(bl, _u8p), len(bs), _ptr(b, _u8p),
                                          bit_length, count, _ptr(out, _u32p), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out[:count]

    def nonzero_ratio(self, x) -> float:
        x = np.ascontiguousarray(x, dtype=np.float32).ravel()
        return self.L.oracle_nonzero_ratio(_ptr(x, _f32p), x.size)

    def mean_abs(self, x) -> float:
        x = np.ascontiguousarray(x, dtype=np.float32).ravel()
        return self.L.oracle_mean_abs(_ptr(x, _f32p), x.size)

    def zero_bitmap(self, x):
        x = np.ascontiguousarray(x, dtype=np.float32).ravel()
        bm = np.empty((x.size + 31) // 32, dtype=np.uint32)
        nz = self.L.oracle_zero_bitmap(_ptr(x, _f32p), x.size, _ptr(bm, _u32p))
        return bm, int(nz)


class Reference:
    """The unmodified reference codec (oracle/_ref/libacz_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        L.ref_compress.argtypes = [_f32p, _u64p, C.c_int, C.c_double, C.c_uint32, C.c_int,
                                   C.POINTER(_u8p), C.POINTER(C.c_uint64), C.c_char_p, C.c_int]
        L.ref_decompress.argtypes = [_u8p, C.c_uint64, C.c_int, _f32p, C.c_uint64, C.c_char_p,
                                     C.c_int]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_nonzero_ratio.argtypes = [_f32p, C.c_uint64, C.POINTER(C.c_double), C.c_char_p,
                                        C.c_int]
        L.ref_mean_abs.argtypes = [_f32p, C.c_uint64, C.POINTER(C.c_double), C.c_char_p, C.c_int]
        L.ref_huffman_encode.argtypes = [_u32p, C.c_uint64, C.POINTER(_u32p), C.POINTER(_u8p),
                                         C.POINTER(C.c_uint64), C.POINTER(_u8p),
                                         C.POINTER(C.c_uint64), C.c_char_p, C.c_int]
        L.ref_roundtrip_sharded.argtypes = [_f32p, _u64p, C.c_int, C.c_double, C.c_uint32,
                                            C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint64),
                                            C.POINTER(C.c_double), C.c_char_p, C.c_int]
        if hasattr(L, "ref_controller_run_ex"):
            L.ref_controller_run_ex.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_double,
                                                C.c_double, _f32p, _u64p, C.c_int, _f32p,
                                                C.c_uint64, _f32p, C.c_uint64, C.c_uint64,
                                                C.c_int, C.c_int, C.c_int, _f32p,
                                                C.POINTER(C.c_double), C.POINTER(C.c_char_p),
                                                C.c_char_p, C.c_int]
        if hasattr(L, "ref_controller_run"):
            L.ref_controller_run.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_double,
                                             C.c_double, _f32p, _u64p, C.c_int, _f32p,
                                             C.c_uint64, _f32p, C.c_uint64, C.c_uint64, C.c_int,
                                             C.POINTER(C.c_double), C.POINTER(C.c_char_p),
                                             C.c_char_p, C.c_int]
        self.L = L

    def controller_run(self, act, loss, mom, batch, W=1000, sigma_fraction=0.01,
                       coefficient_a=0.32, eb_min=1e-8, eb_max=1e-1, wraps=0,
                       relu_recompute=False, is_post_relu=True):
        """The unmodified reference Controller (src/controller.cpp) on one layer: collect at
        iteration 0, `wraps` wrap/unwrap passes at iteration 1, finalize. Returns a dict
        with l_bar, r, m_avg, degenerate, eb, active, held_bytes, the ledger CSV and the
        last unwrapped tensor ("back"; zero_restoration = relu-recompute when
        relu_recompute)."""
        act = np.ascontiguousarray(act, dtype=np.float32)
        loss = np.ascontiguousarray(loss, dtype=np.float32).ravel()
        mom = np.ascontiguousarray(mom, dtype=np.float32).ravel()
        shp = np.asarray(act.shape, dtype=np.uint64)
        back = np.zeros(act.shape, dtype=np.float32)
        out = (C.c_double * 8)()
        csv = C.c_char_p()
        err = C.create_string_buffer(512)
        rc = self.L.ref_controller_run_ex(int(W), sigma_fraction, coefficient_a, eb_min, eb_max,
                                          act.ctypes.data_as(_f32p), shp.ctypes.data_as(_u64p),
                                          act.ndim, loss.ctypes.data_as(_f32p), loss.size,
                                          mom.ctypes.data_as(_f32p), mom.size, int(batch),
                                          int(wraps), int(bool(relu_recompute)),
                                          int(bool(is_post_relu)), back.ctypes.data_as(_f32p),
                                          out, C.byref(csv), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        text = csv.value.decode()
        self.L.ref_free(csv)
        return dict(l_bar=out[0], r=out[1], m_avg=out[2], degenerate=bool(out[3]), eb=out[4],
                    active=bool(out[5]), held_bytes=int(out[6]), csv=text, back=back)

    def compress(self, x: np.ndarray, eb: float, radius: int = 32768, predictor: int = 0,
                 shape=None) -> bytes:
        x = np.ascontiguousarray(x, dtype=np.float32)
        shp = np.asarray(x.shape if shape is None else shape, dtype=np.uint64)
        p = _u8p()
        sz = C.c_uint64()
        err = C.create_string_buffer(512)
        rc = self.L.ref_compress(_ptr(x, _f32p), _ptr(shp, _u64p), len(shp), eb, radius,
                                 predictor, C.byref(p), C.byref(sz), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        out = bytes(_copy(p, sz.value, np.uint8))
        self.L.ref_free(C.cast(p, C.c_void_p))
        return out

    def compress_mt(self, x: np.ndarray, eb: float, radius: int = 32768, predictor: int = 0,
                    threads: Optional[int] = None, symbols: bool = False):
        """oracle_compress on `threads` host threads (same bytes as compress(); the plane
        ranges, counts and bit packing are split and joined in order). Returns
        (ACZ1 blob bytes, chain values float32 [n], symbols uint32 [n] or None). The chain
        values are what decompress reconstructs (ref src/codec.cpp:153-161 repeats the
        compressor's expression), so filter(recon) is the decompressed output."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        shp = np.asarray(x.shape, dtype=np.uint64)
        res = _oracle_result()
        err = C.create_string_buffer(512)
        nt = threads or min(64, os.cpu_count() or 1)
        rc = self.L.oracle_compress_mt(_ptr(x, _f32p), _ptr(shp, _u64p), len(shp), eb, radius,
                                       predictor, nt, C.byref(res), err, 512)
        try:
            if rc:
                raise OracleError(rc, err.value.decode())
            blob = np.ctypeslib.as_array(res.blob, shape=(res.blob_size,)).tobytes()
            recon = _copy(res.recon, res.n, np.float32)
            syms = _copy(res.symbols, res.n, np.uint32) if symbols else None
            return blob, recon, syms
        finally:
            self.L.oracle_result_free(C.byref(res))

    @staticmethod
    def zero_filter(recon: np.ndarray, eb: float) -> np.ndarray:
        """ref src/codec.cpp:162-164: |(double)v| <= eb -> 0.0f (on the chain values)."""
        out = recon.copy()
        out[np.abs(recon.astype(np.float64)) <= eb] = 0.0
        return out

    def decompress(self, blob: bytes, n: int, zero_filter: bool = False) -> np.ndarray:
        b = np.frombuffer(blob, dtype=np.uint8).copy()
        out = np.empty(n, dtype=np.float32)
        err = C.create_string_buffer(512)
        rc = self.L.ref_decompress(_ptr(b, _u8p), len(b), int(zero_filter), _ptr(out, _f32p), n,
                                   err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out

    def huffman_encode(self, syms):
        s = np.ascontiguousarray(syms, dtype=np.uint32)
        psym, plen, pbits = _u32p(), _u8p(), _u8p()
        bs, bl = C.c_uint64(), C.c_uint64()
        err = C.create_string_buffer(512)
        rc = self.L.ref_huffman_encode(_ptr(s, _u32p), len(s), C.byref(psym), C.byref(plen),
                                       C.byref(bs), C.byref(pbits), C.byref(bl), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        out = (_copy(psym, bs.value, np.uint32), _copy(plen, bs.value, np.uint8),
               _copy(pbits, (bl.value + 7) // 8, np.uint8), bl.value)
        for p in (psym, plen, pbits):
            self.L.ref_free(C.cast(p, C.c_void_p))
        return out

    def nonzero_ratio(self, x) -> float:
        x = np.ascontiguousarray(x, dtype=np.float32).ravel()
        r = C.c_double()
        err = C.create_string_buffer(256)
        rc = self.L.ref_nonzero_ratio(_ptr(x, _f32p), x.size, C.byref(r), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return r.value

    def mean_abs(self, x) -> float:
        x = np.ascontiguousarray(x, dtype=np.float32).ravel()
        r = C.c_double()
        err = C.create_string_buffer(256)
        rc = self.L.ref_mean_abs(_ptr(x, _f32p), x.size, C.byref(r), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return r.value

    def roundtrip_sharded(self, x: np.ndarray, eb: float, radius: int = 32768,
                          predictor: int = 0, shards: int = 1, threads: int = 1):
        """CPU baseline: compress+decompress(zero_filter) over batch shards on `threads`
        host threads. Returns (total ACZ1 bytes, seconds)."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        shp = np.asarray(x.shape, dtype=np.uint64)
        tot = C.c_uint64()
        sec = C.c_double()
        err = C.create_string_buffer(512)
        rc = self.L.ref_roundtrip_sharded(_ptr(x, _f32p), _ptr(shp, _u64p), len(shp), eb, radius,
                                          predictor, shards, threads, C.byref(tot), C.byref(sec),
                                          err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return tot.value, sec.value


def reference_available() -> bool:
    return os.path.exists(REF_SO)
