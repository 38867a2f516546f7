// Microbenchmark: FP64 / conversion throughput and dependent-chain latency on B200.
// Informs the design of the exact per-plane recurrence.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

#define ITERS 4096

__global__ void k_dadd_tp(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < ITERS; ++i) {
    x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a);
    x4 = __dadd_rn(x4, b); x5 = __dadd_rn(x5, b); x6 = __dadd_rn(x6, b); x7 = __dadd_rn(x7, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_f2f_tp(float* out, float a) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < ITERS; ++i) {
    // float -> double -> float round trips (F2F.F64.F32 + F2F.F32.F64)
    x0 = __double2float_rn((double)x0 + 0.0) + a; x1 = __double2float_rn((double)x1) + a;
    x2 = __double2float_rn((double)x2) + a; x3 = __double2float_rn((double)x3) + a;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}
__global__ void k_fadd_tp(float* out, float a) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < ITERS; ++i) {
    x0 = __fadd_rn(x0, a); x1 = __fadd_rn(x1, a); x2 = __fadd_rn(x2, a); x3 = __fadd_rn(x3, a);
    x4 = __fadd_rn(x4, a); x5 = __fadd_rn(x5, a); x6 = __fadd_rn(x6, a); x7 = __fadd_rn(x7, a);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
// chain latency: r = fl32(fl64(r + c)) via conversions
__global__ void k_chain_cvt(float* out, const double* c, long long* cyc) {
  float r = 0.0f;
  double cc = c[threadIdx.x & 7];
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
    r = __double2float_rn(__dadd_rn((double)r, cc));
    cc = -cc;
  }
  long long t1 = clock64();
  out[threadIdx.x] = r; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// chain latency via magic-constant rounding to 24 significant bits, state kept in double
__device__ __forceinline__ double round_to_f32(double y) {
  int hi = __double2hiint(y);
  int m = (hi & 0x7FF00000) + ((29 << 20) | (1 << 19));
  double M = __hiloint2double(m, 0);
  return __dsub_rn(__dadd_rn(y, M), M);
}
__global__ void k_chain_magic(double* out, const double* c, long long* cyc) {
  double r = 0.0;
  double cc = c[threadIdx.x & 7];
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
    r = round_to_f32(__dadd_rn(r, cc));
    cc = -cc;
  }
  long long t1 = clock64();
  out[threadIdx.x] = r; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dadd_lat(double* out, double a, long long* cyc) {
  double r = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) r = __dadd_rn(r, a);
  long long t1 = clock64();
  out[threadIdx.x] = r; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_i2d_tp(double* out, int a) {
  int x = threadIdx.x; double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < ITERS; ++i) {
    s0 += (double)(x + i); s1 += (double)(x ^ i); s2 += (double)(x - i); s3 += (double)(x | i);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n4) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n4; i += st) b[i] = a[i];
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount; int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("device %s sms=%d clock=%d MHz\n", p.name, sms, clk_khz / 1000);
  double* dout; float* fout; long long* cyc; double* dc;
  cudaMalloc(&dout, 1 << 26); cudaMalloc(&fout, 1 << 26); cudaMalloc(&cyc, 64); cudaMalloc(&dc, 64);
  double hc[8] = {0.7000000000000001, -0.5, 1.2345678, 0.002, 3.3, -2.2, 0.0123, 1e-3};
  cudaMemcpy(dc, hc, 64, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms * 8, threads = 256; float ms;
  auto tp = [&](const char* name, double ops_per_thread, auto launch) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = ops_per_thread * blocks * threads;
    printf("%-28s %8.3f ms  %8.1f Gop/s  %6.1f op/clk/SM (at %d MHz)\n", name, ms, ops / ms / 1e6,
           ops / (ms * 1e-3) / sms / (clk_khz * 1e3), clk_khz / 1000);
  };
  tp("DADD throughput", 8.0 * ITERS, [&] { k_dadd_tp<<<blocks, threads>>>(dout, 1.0, 2.0); });
  tp("FADD throughput", 8.0 * ITERS, [&] { k_fadd_tp<<<blocks, threads>>>(fout, 1.0f); });
  tp("F2F f32->f64->f32 pairs", 4.0 * ITERS, [&] { k_f2f_tp<<<blocks, threads>>>(fout, 1.0f); });
  tp("I2F.F64 throughput", 4.0 * ITERS, [&] { k_i2d_tp<<<blocks, threads>>>(dout, 1); });
  long long hcyc;
  k_dadd_lat<<<1, 32>>>(dout, 1.0, cyc); cudaMemcpy(&hcyc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DADD latency: %.2f cyc\n", (double)hcyc / ITERS);
  k_chain_cvt<<<1, 32>>>(fout, dc, cyc); cudaMemcpy(&hcyc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("chain step (cvt f32<->f64 + DADD): %.2f cyc\n", (double)hcyc / ITERS);
  k_chain_magic<<<1, 32>>>(dout, dc, cyc); cudaMemcpy(&hcyc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("chain step (magic rounding, 3 DADD): %.2f cyc\n", (double)hcyc / ITERS);
  size_t n = (size_t)1 << 30; float4 *a, *b; cudaMalloc(&a, n); cudaMalloc(&b, n);
  cudaMemset(a, 0, n);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); k_copy<<<sms * 16, 512>>>(a, b, n / 16); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("float4 copy 1 GiB: %.3f ms = %.1f GB/s (r+w)\n", ms, 2.0 * n / ms / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
