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

// PrevValue (ref src/codec.cpp:41): pred = at == 0 ? 0 : recon[at-1]. One thread per plane,
// one warp per 32 consecutive planes. The planes are streamed through shared memory in
// tiles of 32 elements per plane: a warp load covers 32 consecutive elements of ONE plane
// (coalesced cp.async, double-buffered), each lane then walks its own plane's row of the
// tile (conflict-free, padded stride), and the symbols leave through a transposed tile with
// coalesced stores. The chain itself (about 90 cycles of dependent FP64 latency per element)
// is the reference recurrence, exact.
constexpr int kQW = 4;    // warps per CTA
// qspec rounding of the thread-per-plane chains: magic add (1) or F2F (0)
#ifndef ACZ_SERIAL_MAGIC
#define ACZ_SERIAL_MAGIC 0
#endif
// qspec blocks of a tile unrolled (the next block's loads overlap the current chain)
#ifndef ACZ_SERIAL_BLOCK_UNROLL
#define ACZ_SERIAL_BLOCK_UNROLL 4
#endif
constexpr int kSerialBlockUnroll = ACZ_SERIAL_BLOCK_UNROLL;
constexpr int kQT = 32;   // tile width (elements per plane)

// x tiles, double-buffered; a lane overwrites the x slot it has just consumed with the
// symbol (as a u32), so the same tile is then read back transposed for the stores.
struct SerialSmem {
    uint32_t xs[kQW][2][32][kQT + 1];
};

template <typename SymT>
__global__ void __launch_bounds__(kQW * 32) k_quant_prev_serial(const float* __restrict__ x,
                                                                PlaneGeom g, QParams qp,
                                                                SymT* __restrict__ sym,
                                                                float* __restrict__ side_state,
                                                                uint64_t interval,
                                                                unsigned int* flags) {
    __shared__ SerialSmem S;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t plane0 = ((uint64_t)blockIdx.x * kQW + w) * 32;
    if (plane0 >= g.planes) return;
    const int np = (int)min((uint64_t)32, g.planes - plane0);
    const uint64_t P = g.plane_size;
    const uint64_t ntiles = (P + kQT - 1) / kQT;
    const float* xw = x + plane0 * P;
    SymT* sw = sym + plane0 * P;
    auto issue = [&](uint64_t t) {
        const uint64_t j0 = t * kQT;
        const int cnt = (int)min((uint64_t)kQT, P - j0);
        if (lane < cnt) {
            const float* src = xw + j0 + lane;
            uint32_t* dst = &S.xs[w][t & 1][0][lane];
            if (np == 32) {  // (every warp but the last: unrolled, all copies in flight)
#pragma unroll
                for (int p = 0; p < 32; ++p) cp_async4(dst + p * (kQT + 1), src + (uint64_t)p * P);
            } else {
                for (int p = 0; p < np; ++p, src += P, dst += kQT + 1) cp_async4(dst, src);
            }
        }
        cp_async_commit();
    };
    const bool active = lane < np;
    const uint64_t base = (plane0 + lane) * P;  // my plane's flat offset
    uint64_t next_side = ((base + interval - 1) / interval) * interval - base;  // plane-relative
    double r = 0.0;
    bool bad = false;
    issue(0);
    for (uint64_t t = 0; t < ntiles; ++t) {
        if (t + 1 < ntiles) {
            issue(t + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        const uint64_t j0 = t * kQT;
        const int cnt = (int)min((uint64_t)kQT, P - j0);
        if (active) {
            uint32_t* xr = S.xs[w][t & 1][lane];
            // sidecar point inside this tile (interval >= 32: at most one)
            const int js = next_side - j0 < (uint64_t)cnt ? (int)(next_side - j0) : -1;
            if (js >= 0) next_side += interval;
            if (cnt == kQT) {
                // whole tile: blocks of 8 speculative steps (qspec), exact redo on a miss
#pragma unroll kSerialBlockUnroll
                for (int jb = 0; jb < kQT; jb += 8) {
                    float xv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        xv[u] = __uint_as_float(xr[jb + u]);
                        bad |= !isfinite(xv[u]);
                    }
                    const float r0 = (float)r;
                    float st = r0;  // chain value before element js (if js is in this block)
                    uint32_t sy[8];
                    auto emit = [&](int u, uint32_t s, float sv) {
                        sy[u] = s;
                        if (js == jb + u + 1) st = sv;
                    };
                    if (qspec<8, ACZ_SERIAL_MAGIC != 0>([&](int u) { return xv[u]; }, emit, r, qp)) {
#pragma unroll
                        for (int u = 0; u < 8; ++u) xr[jb + u] = sy[u];
                    } else {
                        // exact redo from the tile (x is still in place)
                        st = r0;
                        qexact<8>([&](int u) { return __uint_as_float(xr[jb + u]); },
                                  [&](int u, uint32_t s, float sv) {
                                      xr[jb + u] = s;
                                      if (js == jb + u + 1) st = sv;
                                  },
                                  r, qp);
                    }
                    if ((unsigned)(js - jb) < 8u) side_state[(base + j0 + js) / interval] = st;
                }
            } else {
#pragma unroll 4
            for (int j = 0; j < cnt; ++j) {
                const float xf = __uint_as_float(xr[j]);
                bad |= !isfinite(xf);
                if (j == js) side_state[(base + j0 + j) / interval] = (float)r;
                double v;
                xr[j] = qstep((double)xf, xf, r, qp, &v);  // r == 0 at the plane start
                r = v;
            }
            }
        }
        __syncwarp();
        if (lane < cnt) {
            SymT* dst = sw + j0 + lane;
            const uint32_t* src = &S.xs[w][t & 1][0][lane];
            if (np == 32) {  // unrolled: the 32 shared loads issue before the stores
                SymT v[32];
#pragma unroll
                for (int p = 0; p < 32; ++p) v[p] = (SymT)src[p * (kQT + 1)];
#pragma unroll
                for (int p = 0; p < 32; ++p) dst[(uint64_t)p * P] = v[p];
            } else {
                for (int p = 0; p < np; ++p, dst += P, src += kQT + 1) *dst = (SymT)*src;
            }
        }
        __syncwarp();
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, kFlagNonFinite);
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

// Lorenzo2d by anti-diagonal wavefront: element (r, c) needs the
// reconstructions of (r, c-1), (r-1, c) -- diagonal d-1 -- and (r-1, c-1) -- diagonal d-2 --
// so all elements of one anti-diagonal are independent. A warp owns a plane and walks its
// rows+cols-1 diagonals; the last two diagonals' reconstructions live in shared memory,
// indexed by row. Bit-identical to the row-major recurrence (same expression per element).
__global__ void __launch_bounds__(32) k_quant_lorenzo_wave(const float* __restrict__ x,
                                                           PlaneGeom g, QParams qp,
                                                           uint32_t* __restrict__ sym,
                                                           unsigned int* flags) {
    extern __shared__ float diag[];  // 3 x rows
    const uint64_t plane = blockIdx.x;
    if (plane >= g.planes) return;
    const int lane = threadIdx.x;
    const int rows = (int)g.rows, cols = (int)g.cols;
    const uint64_t base = plane * g.plane_size;
    const float* xp = x + base;
    uint32_t* sp = sym + base;
    float* d0 = diag;             // diagonal d   (being written)
    float* d1 = diag + rows;      // diagonal d-1
    float* d2 = diag + 2 * rows;  // diagonal d-2
    bool bad = false;
    for (int d = 0; d < rows + cols - 1; ++d) {
        const int r_lo = d - (cols - 1) > 0 ? d - (cols - 1) : 0;
        const int r_hi = d < rows - 1 ? d : rows - 1;
        for (int r = r_lo + lane; r <= r_hi; r += 32) {
            const int c = d - r;
            const uint64_t off = (uint64_t)r * cols + c;
            const float xf = __ldg(xp + off);
            bad |= !isfinite(xf);
            const double dl = c > 0 ? (double)d1[r] : 0.0;
            const double dt = r > 0 ? (double)d1[r - 1] : 0.0;
            const double dtl = (r > 0 && c > 0) ? (double)d2[r - 1] : 0.0;
            const double pred = __dsub_rn(__dadd_rn(dl, dt), dtl);
            double v;
            sp[off] = qstep((double)xf, xf, pred, qp, &v);
            d0[r] = (float)v;
        }
        __syncwarp();
        float* t = d2;
        d2 = d1;
        d1 = d0;
        d0 = t;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, kFlagNonFinite);
}

}  // namespace

cudaError_t launch_quant(const QuantArgs& a, int sms, cudaStream_t s, uint64_t* launches) {
    (void)sms;
    if (a.predictor == ACZ_PRED_PREV) {
        const uint64_t warps = (a.g.planes + 31) / 32;
        const uint64_t blocks = (warps + kQW - 1) / kQW;
        const QParams qp = make_qparams(a.eb, a.radius);
        if (a.sym16)
            k_quant_prev_serial<uint16_t><<<(unsigned)blocks, kQW * 32, 0, s>>>(
                a.x, a.g, qp, a.sym16, a.side_state, a.interval, a.flags);
        else
            k_quant_prev_serial<uint32_t><<<(unsigned)blocks, kQW * 32, 0, s>>>(
                a.x, a.g, qp, a.sym, a.side_state, a.interval, a.flags);
    } else if (a.g.rows > 1 && a.g.rows <= kLorenzoWaveRows) {
        const QParams qp = make_qparams(a.eb, a.radius);
        k_quant_lorenzo_wave<<<(unsigned)a.g.planes, 32, 3 * 4 * a.g.rows, s>>>(a.x, a.g, qp,
                                                                              a.sym, a.flags);
    } else {  // single rows (no wavefront) or very tall planes: row-major, thread per plane
        const unsigned threads = 128;
        const uint64_t blocks = (a.g.planes + threads - 1) / threads;
        k_quant_lorenzo_serial<<<(unsigned)blocks, threads, 0, s>>>(
            a.x, a.g, a.eb, a.step, a.radius, a.sym, a.row_scratch, a.flags);
    }
    ++*launches;
    return cudaGetLastError();
}

}  // namespace acz_b200
