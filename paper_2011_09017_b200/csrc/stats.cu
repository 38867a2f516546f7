// K1: fused zero-bitmap + sparsity + finiteness + sum|x| pass (north_star "fused ReLU
// zero-bitmap and sparsity pass"). Predicates follow the reference exactly:
//   nonzero  : v != 0.0f              (ref include/acz/tensor.hpp:91-99, -0.0 is zero)
//   finite   : isfinite(v)            (ref include/acz/tensor.hpp:69-73 -> DomainError)
//   sum |v|  : in double              (ref include/acz/tensor.hpp:82-89; parallel order)
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
                                               double* sumabs) {
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
    if ((threadIdx.x & 31) == 0) {
        if (cnt) atomicAdd(nnz, cnt);
        if (sumabs) atomicAdd(sumabs, sabs);
        if (any_bad) atomicOr(flags, kFlagNonFinite);
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

}  // namespace

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

cudaError_t launch_stats(const float* x, uint64_t n, uint32_t* bitmap,
                         unsigned long long* d_nnz, unsigned int* d_flags, double* d_sumabs,
                         int sms, cudaStream_t s, uint64_t* launches) {
    const uint64_t nwords = (n + 31) / 32;
    uint64_t blocks = (nwords + 255) / 256;
    const uint64_t cap = (uint64_t)sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks == 0) blocks = 1;
    k_stats<<<(unsigned)blocks, 256, 0, s>>>(x, n, bitmap, d_nnz, d_flags, d_sumabs);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace acz_b200
