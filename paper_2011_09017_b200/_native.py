"""ctypes binding of the C-ABI in include/acz_gpu.h (libacz_gpu.so, built in-tree).

There is no CPU fallback: if the CUDA library is missing or no GPU is visible, loading
fails loudly. Only symbol presence can be checked without a GPU (``load(check_only=True)``).
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libacz_gpu.so")

_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_f32p = C.POINTER(C.c_float)
_vp = C.c_void_p

ACZ_MAX_RANK = 16


class BlobInfo(C.Structure):
    _fields_ = [("rank", C.c_uint32), ("shape", C.c_uint64 * ACZ_MAX_RANK), ("eb", C.c_double),
                ("quant_radius", C.c_uint32), ("predictor", C.c_uint32),
                ("element_count", C.c_uint64), ("codebook_size", C.c_uint32),
                ("bit_length", C.c_uint64), ("outlier_count", C.c_uint64),
                ("uncompressed_bytes", C.c_uint64), ("compressed_bytes", C.c_uint64),
                ("device_bytes", C.c_uint64), ("sidecar_bytes", C.c_uint64),
                ("max_code_length", C.c_uint32)]


# (name, restype, argtypes) -- exactly the functions declared in include/acz_gpu.h
SIGNATURES = [
    ("acz_gpu_ctx_create", C.c_int, [C.c_int, C.POINTER(_vp)]),
    ("acz_gpu_ctx_destroy", C.c_int, [_vp]),
    ("acz_gpu_last_error", C.c_char_p, [_vp]),
    ("acz_gpu_version", C.c_char_p, []),
    ("acz_gpu_compress", C.c_int, [_vp, _vp, _u64p, C.c_uint32, C.c_double, C.c_uint32,
                                   C.c_uint32, _vp, C.POINTER(_vp)]),
    ("acz_gpu_compress_async", C.c_int, [_vp, _vp, _u64p, C.c_uint32, C.c_double,
                                         C.c_uint32, C.c_uint32, C.c_uint64, _vp,
                                         C.POINTER(_vp), C.POINTER(C.c_int)]),
    ("acz_gpu_compress_settle", C.c_int, [_vp, _vp, C.c_int, C.POINTER(C.c_int)]),
    ("acz_gpu_decompress", C.c_int, [_vp, _vp, C.c_int, _vp, _vp]),
    ("acz_gpu_malloc", C.c_int, [_vp, C.c_uint64, _vp, C.POINTER(_vp)]),
    ("acz_gpu_free", C.c_int, [_vp, _vp, _vp]),
    ("acz_gpu_memcpy", C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_int, _vp]),
    ("acz_gpu_stream_sync", C.c_int, [_vp, _vp]),
    ("acz_gpu_relu", C.c_int, [_vp, _vp, C.c_uint64, _vp]),
    ("acz_gpu_compress_batch", C.c_int, [_vp, C.c_uint32, C.POINTER(_vp), _u64p, _u32p,
                                         C.c_double, C.c_uint32, C.c_uint32, _vp,
                                         C.POINTER(_vp), C.POINTER(C.c_int)]),
    ("acz_gpu_compress_host_batch", C.c_int, [_vp, C.c_uint32, C.POINTER(_vp), _u64p, _u32p,
                                              C.c_double, C.c_uint32, C.c_uint32, C.POINTER(_vp),
                                              _u64p, _u64p, C.POINTER(_vp), _u64p, _u64p,
                                              C.POINTER(C.c_int)]),
    ("acz_gpu_decompress_host_batch", C.c_int, [_vp, C.c_uint32, C.POINTER(_vp), _u64p,
                                                C.POINTER(_vp), _u64p, C.c_int, C.POINTER(_vp),
                                                _u64p, C.POINTER(C.c_int)]),
    ("acz_gpu_decompress_batch", C.c_int, [_vp, C.c_uint32, C.POINTER(_vp), C.c_int,
                                           C.POINTER(_vp), _vp]),
    ("acz_gpu_blob_info", C.c_int, [_vp, C.POINTER(BlobInfo)]),
    ("acz_gpu_blob_free", C.c_int, [_vp]),
    ("acz_gpu_blob_to_host", C.c_int, [_vp, _vp, _vp, C.c_uint64, _u64p, _vp]),
    ("acz_gpu_blob_from_host", C.c_int, [_vp, _vp, C.c_uint64, _vp, C.c_uint64, _vp,
                                         C.POINTER(_vp)]),
    ("acz_gpu_sidecar_to_host", C.c_int, [_vp, _vp, _vp, C.c_uint64, _u64p, _vp]),
    ("acz_gpu_compress_host", C.c_int, [_vp, _vp, _u64p, C.c_uint32, C.c_double, C.c_uint32,
                                        C.c_uint32, C.POINTER(_vp), _u64p, C.POINTER(_vp),
                                        _u64p]),
    ("acz_gpu_decompress_host", C.c_int, [_vp, _vp, C.c_uint64, _vp, C.c_uint64, C.c_int, _vp,
                                          C.c_uint64]),
    ("acz_gpu_host_free", None, [_vp]),
    ("acz_gpu_zero_bitmap", C.c_int, [_vp, _vp, C.c_uint64, _vp, _u64p, _vp]),
    ("acz_gpu_nonzero_ratio", C.c_int, [_vp, _vp, C.c_uint64, _vp, C.POINTER(C.c_double)]),
    ("acz_gpu_mean_abs", C.c_int, [_vp, _vp, C.c_uint64, _vp, C.POINTER(C.c_double)]),
    ("acz_gpu_huffman_encode", C.c_int, [_vp, _vp, C.c_uint64, _vp, _vp, C.c_uint32, _u32p, _vp,
                                         C.c_uint64, _u64p, _vp]),
    ("acz_gpu_huffman_decode", C.c_int, [_vp, _vp, _vp, C.c_uint32, _vp, C.c_uint64, C.c_uint64,
                                         _vp, _vp]),
    ("acz_gpu_profile_enable", C.c_int, [_vp, C.c_int]),
    ("acz_gpu_profile_read", C.c_int, [_vp, C.POINTER(C.c_double), _u64p]),
    ("acz_gpu_debug_counters", C.c_int, [_vp, _u64p, C.c_uint32, C.c_int]),
    ("acz_gpu_debug_last_symbols", C.c_int, [_vp, _vp, C.c_uint64, _vp]),
    ("acz_gpu_launch_count", C.c_uint64, [_vp]),
    ("acz_gpu_memory_info", C.c_int, [_vp, _u64p, _u64p, _u64p, C.c_int]),
    ("acz_gpu_ctx_trim", C.c_int, [_vp]),
    ("acz_gpu_memory_breakdown", C.c_int, [_vp, _u64p, C.c_uint32]),
]

_lib = None
_lock = threading.Lock()


def load(check_only: bool = False):
    """Load libacz_gpu.so and bind every C-ABI symbol. Raises if the library is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"CUDA extension not built: {LIB_PATH} missing (run `python -m "
                f"paper_2011_09017_b200.build` or __graft_entry__.build()); there is no CPU "
                f"fallback")
        lib = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib
