// K1: fused zero-bitmap + sparsity + finiteness + sum|x| pass (north_star "fused ReLU
// zero-bitmap and sparsity pass"). Predicates follow the reference exactly:
//   nonzero  : v != 0.0f              (ref include/acz/tensor.hpp:91-99, -0.0 is zero)
//   finite   : isfinite(v)            (ref include/acz/tensor.hpp:69-73 -> DomainError)
//   sum |v|  : in double              (ref include/acz/tensor.hpp:82-89). The reference sums
//              sequentially; here every thread sums its grid-stride words in order, warps
//              and CTAs combine in a fixed tree order and the last CTA adds the per-CTA
//              partials in index order, so the result is deterministic (identical for
//              identical inputs on a given grid), within 1e-12 relative of the reference.
//
// HBM-bound: 4 B read per element, 1/8 B written (bitmap). Each thread owns one 32-element
// bitmap word and reads it as 8 x 128-bit loads; a warp therefore streams 4 KiB per
// iteration. Grid = persistent, 148 SMs x 8 CTAs x 256 threads.
#include "internal.h"

namespace acz_b200 {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(256) k_stats(const float* __restrict__ x, uint64_t n,
                                               uint32_t* __restrict__ bitmap,
                                               unsigned long long* nnz, unsigned int* flags,
                                               double* sumabs, double* partials,
                                               unsigned int* ticket) {
    __shared__ double s_warp[8];
    __shared__ bool s_last;
    const uint64_t nwords = (n + 31) / 32;
    const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    unsigned long long cnt = 0;
    double sabs = 0.0;
    bool bad = false;
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t base = w * 32;
        uint32_t mask = 0;
        if (aligned && base + 32 <= n) {
            const float4* p = reinterpret_cast<const float4*>(x + base);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                float4 v = __ldcs(p + j);
                float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    mask |= (e[k] != 0.0f ? 1u : 0u) << (4 * j + k);
                    bad |= !isfinite(e[k]);
                    sabs += fabs((double)e[k]);
                }
            }
        } else {
            for (int k = 0; k < 32 && base + k < n; ++k) {
                float e = x[base + k];
                mask |= (e != 0.0f ? 1u : 0u) << k;
                bad |= !isfinite(e);
                sabs += fabs((double)e);
            }
        }
        if (bitmap) bitmap[w] = mask;
        cnt += __popc(mask);
    }
    cnt = warp_sum_u64(cnt);
    sabs = warp_sum(sabs);
    const unsigned any_bad = __any_sync(0xffffffffu, bad);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        if (cnt) atomicAdd(nnz, cnt);  // integer: order-independent
        if (any_bad) atomicOr(flags, kFlagNonFinite);
        s_warp[warp] = sabs;
    }
    if (!sumabs) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b += s_warp[w];
        partials[blockIdx.x] = b;
        __threadfence();
        s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last || warp != 0) return;
    // last CTA: lane l sums partials l, l+32, ... in order, then a fixed butterfly
    __threadfence();
    double t = 0.0;
    for (unsigned i = lane; i < gridDim.x; i += 32) t += ((volatile double*)partials)[i];
    t = warp_sum(t);
    if (lane == 0) {
        *sumabs = t;
        *ticket = 0u;  // ready for the next launch (stream-ordered)
    }
}

__global__ void k_widen_u16(const uint16_t* __restrict__ a, uint32_t* __restrict__ b, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

__global__ void k_relu(float* __restrict__ x, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const float v = x[i];
        x[i] = v > 0.0f ? v : 0.0f;  // ref include/acz/nn/layers.hpp:134-157 (NaN -> 0)
    }
}

// ACZ1 serialisation of the codebook (u32 symbol, u8 length: 5 bytes per entry) and the
// outlier list (u64 index, f32 value: 12 bytes), little-endian (ref src/codec.cpp:179-199),
// packed on the device so the blob goes to the host as plain async copies.
__global__ void k_pack_acz1(const uint32_t* __restrict__ bsym, const uint8_t* __restrict__ blen,
                            uint32_t k, const unsigned long long* __restrict__ oidx,
                            const float* __restrict__ oval, uint64_t nout,
                            uint8_t* __restrict__ book_out, uint8_t* __restrict__ outl_out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += stride) {
        const uint32_t v = bsym[i];
        uint8_t* q = book_out + 5 * i;
        q[0] = (uint8_t)v;
        q[1] = (uint8_t)(v >> 8);
        q[2] = (uint8_t)(v >> 16);
        q[3] = (uint8_t)(v >> 24);
        q[4] = blen[i];
    }
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nout; i += stride) {
        const unsigned long long a = oidx[i];
        const uint32_t b = __float_as_uint(oval[i]);
        uint8_t* q = outl_out + 12 * i;
#pragma unroll
        for (int j = 0; j < 8; ++j) q[j] = (uint8_t)(a >> (8 * j));
#pragma unroll
        for (int j = 0; j < 4; ++j) q[8 + j] = (uint8_t)(b >> (8 * j));
    }
}

// Several small copies in one launch, executed by SMs instead of a copy engine: a copy engine
// queues them behind multi-megabyte host transfers of other streams, which would stall this
// stream's next kernel (or, for the BookInfo read-back into mapped host memory, the host).
__global__ void k_copy_regions(CopyRegions r) {
    for (int k = 0; k < r.n; ++k) {
        const char* src = static_cast<const char*>(r.src[k]);
        char* dst = static_cast<char*>(r.dst[k]);
        const uint64_t bytes = r.bytes[k];
        const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
        const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
        if ((((uintptr_t)src | (uintptr_t)dst | bytes) & 3) == 0) {
            const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src);
            uint32_t* d4 = reinterpret_cast<uint32_t*>(dst);
            for (uint64_t i = t; i < bytes / 4; i += stride) d4[i] = s4[i];
        } else {
            for (uint64_t i = t; i < bytes; i += stride) dst[i] = src[i];
        }
    }
    if (r.to_host) __threadfence_system();  // mapped host destination
}

// Inverse of k_pack_acz1: the raw ACZ1 codebook (5-byte entries) and outlier records
// (12 bytes), uploaded as they lie in the host blob, into the blob's device arrays.
__global__ void k_unpack_acz1(const uint8_t* __restrict__ raw, uint32_t k, uint64_t nout,
                              uint32_t* __restrict__ bsym, uint8_t* __restrict__ blen,
                              unsigned long long* __restrict__ oidx, float* __restrict__ oval) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += stride) {
        const uint8_t* q = raw + 5 * i;
        bsym[i] = (uint32_t)q[0] | ((uint32_t)q[1] << 8) | ((uint32_t)q[2] << 16) |
                  ((uint32_t)q[3] << 24);
        blen[i] = q[4];
    }
    const uint8_t* ro = raw + 5ull * k;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nout; i += stride) {
        const uint8_t* q = ro + 12 * i;
        unsigned long long a = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) a |= (unsigned long long)q[j] << (8 * j);
        uint32_t b = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) b |= (uint32_t)q[8 + j] << (8 * j);
        oidx[i] = a;
        oval[i] = __uint_as_float(b);
    }
}

// Sidecar binding of a device blob (acz_binding in common.cuh), written to *out.
__global__ void __launch_bounds__(256) k_blob_digest(const uint32_t* __restrict__ bsym,
                                                     const uint8_t* __restrict__ blen, uint32_t k,
                                                     const uint8_t* __restrict__ bits,
                                                     uint64_t nbytes, uint64_t h0,
                                                     unsigned long long* out) {
    __shared__ unsigned long long s_sum;
    __shared__ uint64_t s_v[64];
    if (threadIdx.x == 0) s_sum = 0ull;
    // the 64 bitstream samples of acz_bits_digest, loaded by 64 threads at once (one thread
    // loading them in its mixing loop waits out 64 memory round trips)
    if (threadIdx.x < 64) {
        const uint64_t i = threadIdx.x;
        const uint64_t pos = nbytes >= 8 ? (nbytes - 8) * i / 63 : 0;
        uint64_t v = 0;
        for (int j = 0; j < 8; ++j)
            if (pos + j < nbytes) v |= (uint64_t)bits[pos + j] << (8 * j);
        s_v[i] = v;
    }
    __syncthreads();
    unsigned long long t = 0;
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) t += acz_book_term(bsym[i], blen[i], i);
    atomicAdd(&s_sum, t);  // integer sum mod 2^64: order-independent
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t h = acz_mix64(nbytes);  // == acz_bits_digest(bits, nbytes)
        for (int i = 0; i < 64; ++i) h = acz_mix64(h ^ (s_v[i] + (uint64_t)i));
        *out = acz_binding(h0, s_sum, h);
    }
}

}  // namespace

cudaError_t launch_blob_digest(const uint32_t* bsym, const uint8_t* blen, uint32_t k,
                               const uint8_t* bits, uint64_t nbytes, uint64_t h0,
                               unsigned long long* out, cudaStream_t s, uint64_t* launches) {
    k_blob_digest<<<1, 256, 0, s>>>(bsym, blen, k, bits, nbytes, h0, out);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_unpack_acz1(const uint8_t* raw, uint32_t k, uint64_t nout, uint32_t* bsym,
                               uint8_t* blen, unsigned long long* oidx, float* oval, int sms,
                               cudaStream_t s, uint64_t* launches) {
    const uint64_t m = k > nout ? k : nout;
    if (m == 0) return cudaSuccess;
    const uint64_t want = (m + 255) / 256;
    const unsigned grid = (unsigned)(want < (uint64_t)sms * 4 ? want : (uint64_t)sms * 4);
    k_unpack_acz1<<<grid, 256, 0, s>>>(raw, k, nout, bsym, blen, oidx, oval);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_copy_regions(const CopyRegions& r, int sms, cudaStream_t s,
                                uint64_t* launches) {
    uint64_t most = 0;
    for (int k = 0; k < r.n; ++k) most = r.bytes[k] > most ? r.bytes[k] : most;
    if (most == 0) return cudaSuccess;
    const uint64_t want = (most / 4 + 255) / 256;
    const unsigned grid = (unsigned)(want < (uint64_t)sms ? (want ? want : 1) : (uint64_t)sms);
    k_copy_regions<<<grid, 256, 0, s>>>(r);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_pack_acz1(const uint32_t* bsym, const uint8_t* blen, uint32_t k,
                             const unsigned long long* oidx, const float* oval, uint64_t nout,
                             uint8_t* book_out, uint8_t* outl_out, int sms, cudaStream_t s,
                             uint64_t* launches) {
    const uint64_t m = k > nout ? k : nout;
    if (m == 0) return cudaSuccess;
    const uint64_t want = (m + 255) / 256;
    const unsigned grid = (unsigned)(want < (uint64_t)sms * 4 ? want : (uint64_t)sms * 4);
    k_pack_acz1<<<grid, 256, 0, s>>>(bsym, blen, k, oidx, oval, nout, book_out, outl_out);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_relu(float* x, uint64_t n, int sms, cudaStream_t s, uint64_t* launches) {
    k_relu<<<(unsigned)(sms * 8), 256, 0, s>>>(x, n);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_widen_u16(const uint16_t* a, uint32_t* b, uint64_t n, int sms, cudaStream_t s,
                             uint64_t* launches) {
    k_widen_u16<<<(unsigned)(sms * 8), 256, 0, s>>>(a, b, n);
    ++*launches;
    return cudaGetLastError();
}

size_t stats_partials(int sms) { return (size_t)sms * 8; }

cudaError_t launch_stats(const float* x, uint64_t n, uint32_t* bitmap,
                         unsigned long long* d_nnz, unsigned int* d_flags, double* d_sumabs,
                         double* d_partials, unsigned int* d_ticket, int sms, cudaStream_t s,
                         uint64_t* launches) {
    const uint64_t nwords = (n + 31) / 32;
    uint64_t blocks = (nwords + 255) / 256;
    const uint64_t cap = stats_partials(sms);
    if (blocks > cap) blocks = cap;
    if (blocks == 0) blocks = 1;
    k_stats<<<(unsigned)blocks, 256, 0, s>>>(x, n, bitmap, d_nnz, d_flags, d_sumabs,
                                             d_partials, d_ticket);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace acz_b200
