// K2: the quantiser (ref src/codec.cpp:61-104).
//
// The reference recurrence is serial per plane: each prediction reads the reconstructed
// float of the previous element, computed in double and rounded to float (SURVEY.md sec. 0
// fact 1). Bit-exact symbols therefore require the recurrence itself.
//
// Version 1 (this file): one thread per plane, the exact recurrence in registers.
// Output: one u32 symbol per element (0 = escape), the chain state before every
// `interval`-th element (decode sidecar), and a non-finite flag (DomainError).
#include "internal.h"

namespace acz_b200 {

namespace {

// PrevValue (ref src/codec.cpp:41): pred = at == 0 ? 0 : recon[at-1].
__global__ void __launch_bounds__(128) k_quant_prev_serial(const float* __restrict__ x,
                                                           PlaneGeom g, double eb, double step,
                                                           uint32_t radius,
                                                           uint32_t* __restrict__ sym,
                                                           float* __restrict__ side_state,
                                                           uint64_t interval,
                                                           unsigned int* flags) {
    const uint64_t plane = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (plane >= g.planes) return;
    const uint64_t P = g.plane_size;
    const uint64_t base = plane * P;
    const double radius_d = (double)radius;
    const long long R = radius;
    float r = 0.0f;
    bool bad = false;
    uint64_t to_side = base % interval;  // elements since the last sidecar point
    to_side = to_side == 0 ? 0 : interval - to_side;
    for (uint64_t i = 0; i < P; ++i) {
        const uint64_t flat = base + i;
        const float xf = __ldg(x + flat);
        bad |= !isfinite(xf);
        const double pred = i == 0 ? 0.0 : (double)r;
        if (to_side == 0) {
            side_state[flat / interval] = i == 0 ? 0.0f : r;
            to_side = interval;
        }
        --to_side;
        float v;
        sym[flat] = quant_step(xf, pred, step, eb, radius_d, R, &v);
        r = v;
    }
    if (bad) atomicOr(flags, kFlagNonFinite);
}

// Lorenzo2d (ref src/codec.cpp:42-47): pred = (left + top) - topleft in double, neighbours
// outside the plane are 0. One thread per plane; the previous row lives in row_scratch.
__global__ void __launch_bounds__(128) k_quant_lorenzo_serial(const float* __restrict__ x,
                                                              PlaneGeom g, double eb,
                                                              double step, uint32_t radius,
                                                              uint32_t* __restrict__ sym,
                                                              float* __restrict__ row_scratch,
                                                              unsigned int* flags) {
    const uint64_t plane = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (plane >= g.planes) return;
    const uint64_t rows = g.rows, cols = g.cols;
    const uint64_t base = plane * g.plane_size;
    float* row = row_scratch + plane * cols;
    const double radius_d = (double)radius;
    const long long R = radius;
    bool bad = false;
    for (uint64_t r = 0; r < rows; ++r) {
        float left = 0.0f, topleft = 0.0f;
        for (uint64_t c = 0; c < cols; ++c) {
            const uint64_t flat = base + r * cols + c;
            const float xf = __ldg(x + flat);
            bad |= !isfinite(xf);
            const float top = r > 0 ? row[c] : 0.0f;
            const double dl = c > 0 ? (double)left : 0.0;
            const double dt = r > 0 ? (double)top : 0.0;
            const double dtl = (r > 0 && c > 0) ? (double)topleft : 0.0;
            const double pred = __dsub_rn(__dadd_rn(dl, dt), dtl);
            float v;
            sym[flat] = quant_step(xf, pred, step, eb, radius_d, R, &v);
            topleft = top;
            row[c] = v;
            left = v;
        }
    }
    if (bad) atomicOr(flags, kFlagNonFinite);
}

}  // namespace

cudaError_t launch_quant(const QuantArgs& a, int sms, cudaStream_t s, uint64_t* launches) {
    (void)sms;
    const unsigned threads = 128;
    const uint64_t blocks = (a.g.planes + threads - 1) / threads;
    if (a.predictor == ACZ_PRED_PREV) {
        k_quant_prev_serial<<<(unsigned)blocks, threads, 0, s>>>(
            a.x, a.g, a.eb, a.step, a.radius, a.sym, a.side_state, a.interval, a.flags);
    } else {
        k_quant_lorenzo_serial<<<(unsigned)blocks, threads, 0, s>>>(
            a.x, a.g, a.eb, a.step, a.radius, a.sym, a.row_scratch, a.flags);
    }
    ++*launches;
    return cudaGetLastError();
}

}  // namespace acz_b200
