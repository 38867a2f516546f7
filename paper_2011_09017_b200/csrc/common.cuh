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

constexpr int kLutBits = 14;             // decode lookup table: 16384 entries (64 KiB smem);
                                         // codes > 14 bits are ~2% of activation symbols
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
    unsigned int slow;               // 1: more leaves than the shared-memory codebook holds
};
constexpr unsigned kFlagNonFinite = 1u;  // DomainError (ref include/acz/tensor.hpp:69-73)
constexpr unsigned kFlagBookTooBig = 2u; // FormatError (ref src/codec.cpp:107-108)
constexpr unsigned kFlagDepth64 = 4u;    // DecodeError (ref src/huffman.cpp:64)
constexpr unsigned kFlagLenTooLong = 8u; // code length > 56: unsupported packing (never for n<2^44)
constexpr unsigned kFlagInternal = 16u;  // internal consistency failure (look-back timeout)

// Sidecar binding (ACZS v3): ties a decode sidecar to one blob. Host (blob_from_host) and
// device (k_blob_digest, at sidecar export) compute the same value from the header hash h0,
// the codebook (order-independent sum of per-entry mixes, so a CTA can reduce it) and 64
// 8-byte samples of the bitstream at fixed positions plus its length.
__host__ __device__ inline uint64_t acz_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t acz_book_term(uint32_t sym, uint32_t len, uint64_t i) {
    return acz_mix64((((uint64_t)sym << 8) | len) + i * 0xD1B54A32D192ED03ull);
}
// bits: the bitstream's byte image (nbytes = ceil(bit_length / 8)).
__host__ __device__ inline uint64_t acz_bits_digest(const uint8_t* bits, uint64_t nbytes) {
    uint64_t h = acz_mix64(nbytes);
    for (int i = 0; i < 64; ++i) {
        const uint64_t pos = nbytes >= 8 ? (nbytes - 8) * (uint64_t)i / 63 : 0;
        uint64_t v = 0;
        for (int j = 0; j < 8; ++j)
            if (pos + j < nbytes) v |= (uint64_t)bits[pos + j] << (8 * j);
        h = acz_mix64(h ^ (v + (uint64_t)i));
    }
    return h;
}
__host__ __device__ inline uint64_t acz_binding(uint64_t h0, uint64_t book_sum, uint64_t bits_digest) {
    return acz_mix64(h0 ^ acz_mix64(book_sum ^ acz_mix64(bits_digest)));
}

// Per-length canonical decode tables (ref src/huffman.cpp:152-166).
struct CanonTables {
    unsigned long long first_code[65];
    unsigned int first_index[65];
    unsigned int count[65];
};

__device__ __forceinline__ uint32_t bswap32(uint32_t v) { return __byte_perm(v, 0, 0x0123); }

// Asynchronous global -> shared copies (LDGSTS): a loop of these issues every load before
// any completes, unlike a load/store loop whose iterations each wait out the memory latency.
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Bulk (TMA) global -> shared copies completed on an mbarrier (sm_90+ / sm_100a) --------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// bytes: a multiple of 16; both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

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

// Exact (double)(float)y for a double y, without the F2F pipe (7.4 conversions / clk / SM
// measured vs 62.5 DADD): adding and subtracting M = 1.5 * 2^(e+29) rounds y to 24
// significant bits, ties to even, exactly like the F32 conversion. Valid when the result is
// a normal float below 2^127; other exponents (zero, subnormal, overflow) take the
// conversion path so inf/denormal behaviour is the reference's.
__device__ __forceinline__ double rn32d(double y) {
    const int hi = __double2hiint(y);
    const int ex = (hi >> 20) & 0x7FF;
    if (ex < 1023 - 126 || ex > 1023 + 126) return (double)__double2float_rn(y);
    const double M = __hiloint2double((ex << 20) + ((29 << 20) | (1 << 19)), 0);
    return __dsub_rn(__dadd_rn(y, M), M);
}

// ACZ_QSPEC_F2F=0: qspec rounds the chain with the magic add (rn32d) instead of the F2F round trip
#ifndef ACZ_QSPEC_F2F
#define ACZ_QSPEC_F2F 1  // measured: F2F 1.26 ms vs magic add 1.32 ms (AlexNet conv1 K2b)
#endif

// Parameters of the reference quantisation step.
struct QParams {
    double eb, step, inv_step, radius_d;
    long long R;
    int exact_div;  // 1/step not usable (absurdly small eb): always divide
};

// The reference quantisation step (ref src/codec.cpp:80-101), bit-exact:
//   q = round((x - pred) / step)   ties away from zero, correctly rounded quotient
//   accept iff |q| < R, cand = fl32(pred + q*step) finite, |x - cand| <= eb
// The quotient is a reciprocal multiply; round(RN(d/step)) can differ from round(d*inv)
// only within a few ulps of a half-integer, where the guard falls back to __ddiv_rn.
// Rounding to an integer uses the 1.5*2^52 magic add, whose low word is q itself (no F2I);
// the guard is evaluated off the dependency chain and only consulted at the end.
// Returns the symbol (0 = escape); *r receives the chain value (a float, as a double).
// The fragile-quotient fallback is inline and branched around (a call on the chain costs
// ~120 cycles per step on B200: tools/microbench/qchain.cu).
__device__ __forceinline__ uint32_t qstep(double orig, float xf, double pred, const QParams& p,
                                          double* r) {
    (void)xf;
    const double d = __dsub_rn(orig, pred);
    const double t = __dmul_rn(d, p.inv_step);  // for the fragility guard (off the chain)
    const double M52 = 6755399441055744.0;       // 1.5 * 2^52
    // one fused op on the chain: round(d*inv) by the magic add, d*inv unrounded. It can
    // differ from round(t) only when d*inv is within an ulp of a half-integer, where the
    // guard below sees |t - q| ~ 0.5 and recomputes q by exact division
    double tm = __fma_rn(d, p.inv_step, M52);
    double q = __dsub_rn(tm, M52);
    // plain F2F round trip: the shortest dependent chain measured on B200
    // (tools/microbench/qchain.cu: 162 cycles/step vs 190-282 for magic-add rounding)
    float cf = __double2float_rn(__dadd_rn(pred, __dmul_rn(q, p.step)));
    const bool fragile = p.exact_div || 0.5 - fabs(t - q) <= fabs(t) * 0x1p-44 + 0x1p-60;
    if (fragile) {
        q = round(__ddiv_rn(d, p.step));
        tm = fabs(q) < 0x1p51 ? __dadd_rn(q, M52) : M52;
        cf = __double2float_rn(__dadd_rn(pred, __dmul_rn(q, p.step)));
    }
    const double c = (double)cf;
    const bool ok = fabs(q) < p.radius_d && isfinite(cf) && fabs(__dsub_rn(orig, c)) <= p.eb;
    *r = ok ? c : orig;
    return ok ? (uint32_t)(__double2loint(tm) + (int)p.R) : 0u;
}

// float bits of a double that holds an exact normal float value (integer pipe only)
__device__ __forceinline__ float f32_of_exact(double c) {
    const unsigned hi = (unsigned)__double2hiint(c), lo = (unsigned)__double2loint(c);
    const unsigned t = hi - (896u << 20);  // rebias the exponent (1023 - 127)
    return __uint_as_float((t & 0x80000000u) | ((t << 3) & 0x7FFFFFF8u) | (lo >> 29));
}

// (double)f on the integer pipe for zero and normal floats; subnormal / inf / nan set `special`
__device__ __forceinline__ double f64_of_f32(float f, bool& special) {
    const unsigned u = __float_as_uint(f);
    const unsigned e = (u >> 23) & 0xFFu;
    special |= e == 0xFFu || (e == 0 && (u << 1) != 0);
    const unsigned hi = (u & 0x80000000u) | (e ? ((u & 0x7FFFFFFFu) >> 3) + (896u << 20) : 0u);
    return __hiloint2double((int)hi, (int)(u << 29));
}

// N reference steps from chain value r, speculating that every step is accepted and has a
// non-fragile quotient (the common case): the chain carries each step's candidate
// reconstruction straight into the next prediction, and the acceptance test, the radius
// test and the fragility guard -- which qstep() has to resolve before it can select the
// chain value -- run off the chain: the dependent path per step is DADD, DFMA, DADD, DMUL,
// DADD and the F2F round trip. (The magic-add rounding of rn32d instead of F2F, which keeps
// the chain off the 7.4/clk/SM conversion pipe, measured slower: AlexNet conv1 K2b 1.32 vs
// 1.26 ms; ACZ_QSPEC_F2F=0 selects it by default, kMagic per call site, where the input
// widening runs on the integer pipe too; it also measured slower in the exact replay and in
// K2a, whose chains are throughput- rather than latency-bound.) Off the chain the fragility guard is one DFMA: |d*inv - q| >= 0.5 - 2^-19 covers qstep's
// 0.5 - |t - q| <= |t| 2^-44 + 2^-60 for every |t| < 2^24 (larger quotients exceed any
// radius and are redone anyway). xat(u) returns input u of the block, emit(u, sym, value)
// receives every step's symbol and chain value (speculatively: on a miss the caller's
// qexact() emits the same positions again). Returns true (and advances r) when no step
// escaped, was rejected, needed the exact quotient or left the normal float range: the
// emitted values then equal what qstep() gives step by step.
template <int N, bool kMagic = ACZ_QSPEC_F2F == 0, class XAt, class Emit>
__device__ __forceinline__ bool qspec(XAt xat, Emit emit, double& r, const QParams& p) {
    const double M52 = 6755399441055744.0;  // 1.5 * 2^52
    bool bad = p.exact_div != 0;
    double rr = r;
#pragma unroll
    for (int u = 0; u < N; ++u) {
        const float xf = xat(u);
        const double orig = kMagic ? f64_of_f32(xf, bad) : (double)xf;
        const double d = __dsub_rn(orig, rr);
        const double tm = __fma_rn(d, p.inv_step, M52);
        const double q = __dsub_rn(tm, M52);
        const double y = __dadd_rn(rr, __dmul_rn(q, p.step));
        double c;
        float cf;
        if (!kMagic) {
            cf = __double2float_rn(y);
            c = (double)cf;
            bad |= !isfinite(cf);
        } else {
            const int ex = (__double2hiint(y) >> 20) & 0x7FF;
            bad |= (unsigned)(ex - (1023 - 126)) > 252u;  // zero, subnormal, overflow: qstep
            const double M = __hiloint2double((ex << 20) + ((29 << 20) | (1 << 19)), 0);
            c = __dsub_rn(__dadd_rn(y, M), M);
            cf = f32_of_exact(c);
        }
        // off the chain: fragility guard, radius and acceptance tests
        bad |= fabs(__fma_rn(d, p.inv_step, -q)) >= 0.5 - 0x1p-19;
        bad |= !(fabs(q) < p.radius_d);
        bad |= !(fabs(__dsub_rn(orig, c)) <= p.eb);
        emit(u, (uint32_t)(__double2loint(tm) + (int)p.R), cf);
        rr = c;
    }
    if (!bad) r = rr;
    return !bad;
}

// The same block step by step with qstep() (the fallback of qspec()).
template <int N, class XAt, class Emit>
__device__ __forceinline__ void qexact(XAt xat, Emit emit, double& r, const QParams& p) {
#pragma unroll 1
    for (int u = 0; u < N; ++u) {
        const float xf = xat(u);
        double v;
        const uint32_t s = qstep((double)xf, xf, r, p, &v);
        emit(u, s, (float)v);
        r = v;
    }
}

__host__ inline QParams make_qparams(double eb, uint32_t radius) {
    QParams p;
    p.eb = eb;
    p.step = 2.0 * eb;
    p.inv_step = 1.0 / p.step;
    p.radius_d = (double)radius;
    p.R = radius;
    // the reciprocal path needs a finite, normal 1/step and |t| well inside 2^51
    p.exact_div = !(p.inv_step < 1e300 && p.step < 1e300) ? 1 : 0;
    return p;
}

}  // namespace acz_b200
