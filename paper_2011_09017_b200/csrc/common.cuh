// Shared device helpers for the B200 activation codec (sm_100a).
//
// Exactness rules: every floating-point operation that
// the reference performs in double is reproduced with the IEEE round-to-nearest
// intrinsics (__dadd_rn/__dsub_rn/__dmul_rn/__ddiv_rn) so ptxas can never contract an
// FMA, and the translation unit is additionally compiled with --fmad=false.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "acz_gpu.h"

namespace acz_b200 {

constexpr int kLutBits = 12;             // decode lookup table: 4096 entries
constexpr int kLutSize = 1 << kLutBits;
constexpr uint32_t kMaxBook = 0xFFFF;    // ACZ1 u16 codebook size (ref src/codec.cpp:107)

// Result block written by the codebook kernel and read back by the host once per
// compress (the single synchronisation point of acz_gpu_compress).
struct BookInfo {
    unsigned long long total_bits;   // sum freq * len
    unsigned long long n_escapes;    // freq of symbol 0 == outlier count
    unsigned int book_size;          // number of distinct symbols
    unsigned int max_len;
    unsigned int flags;              // kFlag* bits below
    unsigned int pad;
};
constexpr unsigned kFlagNonFinite = 1u;  // DomainError (ref include/acz/tensor.hpp:69-73)
constexpr unsigned kFlagBookTooBig = 2u; // FormatError (ref src/codec.cpp:107-108)
constexpr unsigned kFlagDepth64 = 4u;    // DecodeError (ref src/huffman.cpp:64)
constexpr unsigned kFlagLenTooLong = 8u; // code length > 56: unsupported packing (never for n<2^44)
constexpr unsigned kFlagInternal = 16u;  // internal consistency failure (look-back timeout)

// Per-length canonical decode tables (ref src/huffman.cpp:152-166).
struct CanonTables {
    unsigned long long first_code[65];
    unsigned int first_index[65];
    unsigned int count[65];
};

__device__ __forceinline__ uint32_t bswap32(uint32_t v) { return __byte_perm(v, 0, 0x0123); }

// Exact reference arithmetic ------------------------------------------------------------

// (float)(pred + q * step) with no contraction: ref src/codec.cpp:86 and :157.
__device__ __forceinline__ float recon_value(double pred, double q, double step) {
    return __double2float_rn(__dadd_rn(pred, __dmul_rn(q, step)));
}

// One PrevValue quantisation step (ref src/codec.cpp:80-101). Returns the symbol
// (0 = escape) and writes the value stored in the chain.
__device__ __forceinline__ uint32_t quant_step(float xf, double pred, double step, double eb,
                                               double radius_d, long long radius,
                                               float* value) {
    const double orig = (double)xf;
    const double q = round(__ddiv_rn(__dsub_rn(orig, pred), step));  // ties away from zero
    if (fabs(q) < radius_d) {
        const float cand = recon_value(pred, q, step);
        if (isfinite(cand) && fabs(__dsub_rn(orig, (double)cand)) <= eb) {
            *value = cand;
            return (uint32_t)((long long)q + radius);
        }
    }
    *value = xf;
    return 0u;
}

}  // namespace acz_b200
