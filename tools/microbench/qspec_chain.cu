// Microbenchmark: dependent-chain latency per element of the speculative block step (qspec,
// csrc/common.cuh) vs the step-by-step reference step (qstep), one warp, each lane its own
// plane of ReLU(N(0,1))-like data in shared memory (development tool).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a --fmad=false -I paper_2011_09017_b200/csrc -I include tools/microbench/qspec_chain.cu -o /tmp/qspec_chain
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"
using namespace acz_b200;

constexpr int N = 320;

template <int V>
__global__ void k_chain(const float* __restrict__ x, uint32_t* out, QParams p, long long* cyc) {
    __shared__ float xs[32][N + 1];
    const int lane = threadIdx.x & 31;
    for (int i = 0; i < N; ++i) xs[lane][i] = x[(size_t)lane * N + i];
    __syncwarp();
    double r = 0.0;
    uint32_t acc = 0;
    long long t0 = clock64();
    if (V == 0) {
        for (int i = 0; i < N; ++i) {
            double v;
            acc = acc * 31 + qstep((double)xs[lane][i], xs[lane][i], r, p, &v);
            r = v;
        }
    } else {
        for (int i = 0; i < N; i += 8) {
            uint32_t sy[8];
            auto xat = [&](int u) { return xs[lane][i + u]; };
            auto emit = [&](int u, uint32_t s, float) { sy[u] = s; };
            if (!qspec<8>(xat, emit, r, p)) qexact<8>(xat, emit, r, p);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = acc * 31 + sy[u];
        }
    }
    long long t1 = clock64();
    out[lane] = acc + (uint32_t)(r * 1000);
    if (lane == 0) *cyc = t1 - t0;
}

int main() {
    float* h = new float[32 * N];
    uint64_t s = 88172645463325252ull;
    for (int i = 0; i < 32 * N; ++i) {
        double a = 0;
        for (int k = 0; k < 4; ++k) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; a += (s >> 11) * 0x1p-53; }
        a = (a - 2.0) * 1.7320508;
        h[i] = a > 0 ? (float)a : 0.0f;
    }
    float* d; uint32_t* o; long long* c;
    cudaMalloc(&d, 4 * 32 * N); cudaMalloc(&o, 128); cudaMalloc(&c, 8);
    cudaMemcpy(d, h, 4 * 32 * N, cudaMemcpyHostToDevice);
    QParams p = make_qparams(1e-3, 32768);
    for (int rep = 0; rep < 3; ++rep) {
        long long cq = 0, cs = 0;
        k_chain<0><<<1, 32>>>(d, o, p, c); cudaMemcpy(&cq, c, 8, cudaMemcpyDeviceToHost);
        k_chain<1><<<1, 32>>>(d, o, p, c); cudaMemcpy(&cs, c, 8, cudaMemcpyDeviceToHost);
        printf("cycles/step: qstep %.1f  qspec<8> %.1f\n", (double)cq / N, (double)cs / N);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
