"""B200-native activation compressor (arXiv 2011.09017, "acz"): the reference's SZ-style
error-bounded codec for fp32 activations re-built as hand-written sm_100a CUDA kernels
behind a C-ABI (include/acz_gpu.h). See DESIGN.md.

Python surface mirrors ref proj/core/include/acz/codec.hpp (see codec.py).
"""
from .codec import (AsyncCompress, CodebookEntry, CodecParams, CompressedTensor, Context, CudaError,
                    DecodeError, DomainError, Error, FormatError, HuffmanCode, Outlier,
                    ParamError, Predictor, ShapeError, blob_from_bytes, blob_to_bytes, compress,
                    compress_async, compress_host, compress_host_many, compress_many, compression_ratio, debug_last_symbols,
                    decompress, decompress_host, decompress_host_many, decompress_many, default_context, huffman_decode, huffman_encode, mean_abs,
                    nonzero_ratio, parse_acz1, relu_, zero_bitmap)

__all__ = [n for n in dir() if not n.startswith("_")]
