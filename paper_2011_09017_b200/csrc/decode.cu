// K6 Huffman decode + K7 reconstruction (ref src/huffman.cpp:137-189, src/codec.cpp:122-171).
//
// k_decode_prev   : one lane per sidecar chunk (`interval` symbols, 32 chunks per warp, a
//                   persistent CTA of 18 warps per SM). The sidecar gives the chunk's bit
//                   offset and the chain state before its first element, so every chunk
//                   decodes and reconstructs independently and bit-exactly. Canonical decode
//                   via a 16384-entry shared-memory LUT (codes <= kLutBits = 14 bits; entries
//                   of longer-code prefixes carry the code-length range), per-length
//                   canonical limits for longer codes; outputs leave through a transposed
//                   32 x 8 tile (coalesced stores).
// k_decode_lorenzo: Lorenzo2d, one thread per plane (sidecar interval = plane size).
// k_scan_decode   : sequential whole-stream decode used to (re)build the sidecar of a
//                   foreign ACZ1 blob and to validate it exactly like the reference
//                   (truncation / no-match DecodeError, outlier FormatErrors).
// k_chain_states  : thread-per-plane chain replay producing the sidecar chain states.
#include <cstdlib>

#include "internal.h"

namespace acz_b200 {

namespace {

struct BitReader {
    const uint32_t* w;
    uint64_t nwords, wi;
    unsigned long long buf;
    int nb;

    __device__ __forceinline__ uint32_t fetch(uint64_t i) const {
        return i < nwords ? bswap32(__ldg(w + i)) : 0u;
    }
    __device__ __forceinline__ void init(const uint32_t* words, uint64_t nw, uint64_t pos) {
        w = words;
        nwords = nw;
        wi = pos >> 5;
        const int off = (int)(pos & 31);
        const unsigned long long a = fetch(wi), b = fetch(wi + 1);
        wi += 2;
        buf = ((a << 32) | b) << off;
        nb = 64 - off;
    }
    __device__ __forceinline__ void refill() {
        if (nb <= 32) {
            buf |= (unsigned long long)fetch(wi++) << (32 - nb);
            nb += 32;
        }
    }
    __device__ __forceinline__ uint32_t peek() const { return (uint32_t)(buf >> (64 - kLutBits)); }
    __device__ __forceinline__ void skip(int k) {
        buf <<= k;
        nb -= k;
    }
    // 64-bit window of the stream starting at absolute bit `pos`
    __device__ __forceinline__ unsigned long long window(uint64_t pos) const {
        const uint64_t i = pos >> 5;
        const int off = (int)(pos & 31);
        const unsigned long long a = fetch(i), b = fetch(i + 1), c = fetch(i + 2);
        const unsigned long long hi = (a << 32) | b;
        return off ? (hi << off) | (c << off >> 32) : hi;
    }
};

// Decodes one symbol at absolute position *pos. Returns the code length (0 = no
// codeword of length <= 64 matches).
__device__ __forceinline__ uint32_t decode_one(BitReader& br, uint64_t& pos,
                                               const uint32_t* s_lut, const CanonTables& ct,
                                               const uint32_t* book_sym, uint32_t* sym) {
    br.refill();
    const uint32_t e = s_lut[br.peek()];
    uint32_t len = e & 31;
    if (len) {
        *sym = e >> 5;
        br.skip((int)len);
        pos += len;
        return len;
    }
    // long code (> 12 bits): canonical ranges per length
    const unsigned long long win = br.window(pos);
    for (uint32_t l = kLutBits + 1; l <= 64; ++l) {
        if (!ct.count[l]) continue;
        const unsigned long long c = win >> (64 - l);
        if (c >= ct.first_code[l] && c - ct.first_code[l] < ct.count[l]) {
            *sym = __ldg(book_sym + ct.first_index[l] + (uint32_t)(c - ct.first_code[l]));
            pos += l;
            br.init(br.w, br.nwords, pos);
            return l;
        }
    }
    return 0;
}

__device__ __forceinline__ void load_tables(const uint32_t* lut, const CanonTables* canon,
                                            uint32_t* s_lut, CanonTables* s_ct) {
    // 64 KiB LUT: asynchronous 16-byte copies, all in flight at once
    for (int i = threadIdx.x; i < kLutSize / 4; i += blockDim.x) cp_async16(s_lut + 4 * i, lut + 4 * i);
    cp_async_commit();
    for (int i = threadIdx.x; i < 65; i += blockDim.x) {
        s_ct->first_code[i] = canon->first_code[i];
        s_ct->first_index[i] = canon->first_index[i];
        s_ct->count[i] = canon->count[i];
    }
    cp_async_wait<0>();
    __syncthreads();
}

// Canonical decode limits (left-aligned): the code length of a 64-bit window w is the
// smallest l with (w >> (64 - l)) < limit[l]; codes of length l are [nc[l], limit[l]).
struct Limits {
    unsigned long long nc[65];
    unsigned long long lim[65];
    uint32_t off[65];  // first_index[l] - nc[l] (mod 2^32): book index = code + off[l]
    int maxlen;
};

__device__ __forceinline__ void build_limits(const CanonTables& ct, Limits* L) {
    if (threadIdx.x == 0) {
        unsigned long long nc = 0;
        L->nc[0] = 0;
        L->lim[0] = 0;
        for (int l = 1; l <= 64; ++l) {
            nc = (l == 1) ? 0 : ((L->nc[l - 1] + ct.count[l - 1]) << 1);
            L->nc[l] = nc;
            L->lim[l] = nc + ct.count[l];
            L->off[l] = ct.first_index[l] - (uint32_t)nc;
            if (ct.count[l]) L->maxlen = l;
        }
    }
}

// K6+K7 (PrevValue). A task = 32 consecutive sidecar chunks (`interval` symbols each, a
// multiple of 32); a warp takes one task at a time, lane = chunk. Persistent CTAs (one per SM,
// kDW warps) load the 64 KiB decode LUT and the long-code book entries once. Per task the
// warp stages the contiguous bitstream span of its 32 chunks into shared memory with
// asynchronous 16-byte copies; every lane then decodes its chunk from its sidecar bit offset
// with two shared loads + a funnel shift per symbol and reconstructs it with the exact
// reference expression from the sidecar chain state (ref src/codec.cpp:143-164). Outputs go
// through a transposed 32 x kTW shared tile, so every global store writes one 32-byte sector
// of each of four chunks (the narrow tile and u16 long-code entries fit 18 warps per SM). The outlier cursor of a chunk is found by binary search over the
// (sorted) outlier indices at its first escape. A span larger than the staging window
// (very long codes) decodes from global memory through the same code.
constexpr int kDW = 18;           // warps per CTA (one CTA per SM)
constexpr int kTW = 8;            // output tile: kTW elements of each of the 32 chunks
constexpr int kTR = 32 / kTW;     // chunks one store instruction covers
constexpr int kDStage = 1792;     // staged stream words per warp (7 KiB, a multiple of 4:
                                  // 32 x 128 symbols at up to 14 bits/symbol)
constexpr int kLongCap = 6144;    // book entries of codes longer than kLutBits kept in smem
                                  // (as u16: symbols of a radius <= 32768 alphabet)
constexpr size_t kDecSmem =
    4ull * kLutSize + 2ull * kLongCap + 4ull * kDW * (kDStage + 32 * (kTW + 1));
// ACZ_DEC_MAGIC=1: the decoder rounds the chain by the magic add (no F2F; A/B)
#ifndef ACZ_DEC_MAGIC
#define ACZ_DEC_MAGIC 0  // measured slower: AlexNet step decode 0.46 -> 0.54 ms
#endif
// debug (development builds, -DACZ_DEC_STATS=1): prologue, staging, loop cycles; tasks
#ifndef ACZ_DEC_STATS
#define ACZ_DEC_STATS 0
#endif
__device__ unsigned long long g_dclk[4];

__device__ __forceinline__ uint32_t lower_bound_u64(const unsigned long long* a, uint32_t n,
                                                    unsigned long long key) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(a + mid) < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

template <bool kStaged, typename PosT>
__device__ __forceinline__ void decode_chunk(const DecodeArgs& a, const uint32_t* bits, PosT p,
                                             const uint32_t* s_lut, const uint16_t* lbook,
                                             uint32_t lfirst, const Limits& lim,
                                             const CanonTables& ct, uint32_t cnt,
                                             uint64_t start, double r, uint32_t snext,
                                             float* tile, float (*s_out)[kTW + 1], uint64_t chunk0,
                                             int lane) {
    const uint32_t I = (uint32_t)a.interval;
    const uint32_t P32 = (uint32_t)min(a.g.plane_size, (uint64_t)0xFFFFFFFFu);
    const int R = (int)a.radius;
    const double step = a.step;
    // q = sym - R as a double without an int->double conversion: hi:lo = 1.5*2^52 + sym
    const double magic = 6755399441055744.0 + (double)R;
    // zero filter |v| <= eb on a float v  <=>  |v| <= the largest float <= eb
    float zthr = -1.0f;
    if (a.zero_filter) {
        zthr = __double2float_rd(a.eb);
    }
    uint32_t oi = 0xFFFFFFFFu;  // outlier cursor, found at the first escape
    auto word = [&](PosT i) -> uint32_t {
        return bswap32(kStaged ? bits[i] : __ldg(bits + i));
    };
    // one symbol: parse (LUT, long codes by canonical limits), reconstruct
    // (ref src/codec.cpp:143-164; r is an exact float held in a double)
    auto step_one = [&](uint32_t gidx, bool reset) -> float {
        const PosT i = p >> 5;
        const uint32_t o = (uint32_t)p & 31u;
        const uint32_t w0 = word(i), w1 = word(i + 1);
        const uint32_t top = __funnelshift_l(w1, w0, o);  // stream bits [p, p+32)
        const uint32_t e = s_lut[top >> (32 - kLutBits)];
        uint32_t len = e & 31, sym = e >> 5;
        if (!len) {
            // long code: canonical limit search on a 64-bit window
            const uint32_t w2 = word(i + 2);
            const unsigned long long win =
                ((unsigned long long)top << 32) | __funnelshift_l(w2, w1, o);
            // the LUT entry bounds the length for this prefix (huffman.cu write_tables)
            len = (e >> 5) & 127;
            const uint32_t lmax = e >> 12;
            while (len < lmax && (win >> (64 - len)) >= lim.lim[len]) ++len;
            const unsigned long long c = win >> (64 - len);
            const uint32_t idx = (uint32_t)c + lim.off[len];
            sym = lbook ? lbook[idx - lfirst] : __ldg(a.book_sym + idx);
        }
        p += len;
        float v;
        if (sym == 0) {
            if (oi == 0xFFFFFFFFu)
                oi = lower_bound_u64(a.out_index, (uint32_t)a.n_outliers, start + gidx);
            v = __ldg(a.out_value + oi);
            ++oi;
            r = (double)v;
        } else {
            const double q = __dsub_rn(__hiloint2double(0x43380000, (int)sym), magic);
            const double pred = reset ? 0.0 : r;
            const double y = __dadd_rn(pred, __dmul_rn(q, step));
#if ACZ_DEC_MAGIC
            // RN32(y) as an exact double by the magic add (rn32d) and its float bits on the
            // integer pipe: no F2F conversion per symbol (7.4/clk/SM); zero, subnormal and
            // huge results take the conversions
            const int ex = (__double2hiint(y) >> 20) & 0x7FF;
            if ((unsigned)(ex - (1023 - 126)) <= 252u) {
                const double M = __hiloint2double((ex << 20) + ((29 << 20) | (1 << 19)), 0);
                r = __dsub_rn(__dadd_rn(y, M), M);
                v = f32_of_exact(r);
            } else {
                v = __double2float_rn(y);
                r = (double)v;
            }
#else
            v = __double2float_rn(y);
            r = (double)v;
#endif
        }
        return fabsf(v) <= zthr ? 0.0f : v;
    };
    for (uint32_t t0 = 0; t0 < I; t0 += kTW) {
        if (t0 < cnt) {
            const uint32_t m = min((uint32_t)kTW, cnt - t0);
            // (a per-lane fast path without the plane-start test diverges across the warp's
            // lanes on small planes and measured slower)
#pragma unroll 4
            for (uint32_t j = 0; j < m; ++j) {
                const bool reset = t0 + j == snext;  // plane start: the predictor resets
                if (reset) snext += P32;
                tile[j] = step_one(t0 + j, reset);
            }
        }
        __syncwarp();
        // coalesced stores: lane group h writes elements [t0, t0+kTW) of chunk chunk0 + c + h
        {
            const uint32_t h = (uint32_t)lane / kTW, e0 = (uint32_t)lane % kTW;
            float* dst = a.out + (chunk0 + h) * I + t0 + e0;
            const float* src = &s_out[h][e0];
            if ((chunk0 + 32) * I <= a.g.n) {  // all 32 chunks complete (every task but the last)
#pragma unroll
                for (int c = 0; c < 32; c += kTR, dst += kTR * I, src += kTR * (kTW + 1)) *dst = *src;
            } else {
                for (int c = 0; c < 32; c += kTR, dst += kTR * I, src += kTR * (kTW + 1)) {
                    const uint64_t e = (chunk0 + c + h) * I + t0 + e0;
                    if (e < a.g.n) *dst = *src;
                }
            }
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(kDW * 32, 1) k_decode_prev(DecodeArgs a) {
    extern __shared__ uint32_t dsm[];
    const long long tk0 = clock64();
    uint32_t* s_lut = dsm;                // 64 KiB
    uint16_t* s_lbook = reinterpret_cast<uint16_t*>(dsm + kLutSize);  // long-code book entries
    __shared__ CanonTables s_ct;
    __shared__ Limits s_lim;
    const uint32_t lfirst = __ldg(&a.canon->first_index[kLutBits + 1]);
    const bool lstaged = a.book_size - lfirst <= (uint32_t)kLongCap && a.radius <= 32768u;
    if (lstaged)
        for (uint32_t i = threadIdx.x; i < a.book_size - lfirst; i += blockDim.x)
            s_lbook[i] = (uint16_t)__ldg(a.book_sym + lfirst + i);
    load_tables(a.lut, a.canon, s_lut, &s_ct);  // commits and waits for all async copies
    build_limits(s_ct, &s_lim);
    __syncthreads();
    const uint16_t* lbook = lstaged ? s_lbook : nullptr;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t* s_bits = dsm + kLutSize + kLongCap / 2 + w * (kDStage + 32 * (kTW + 1));
    float(*s_out)[kTW + 1] = reinterpret_cast<float(*)[kTW + 1]>(s_bits + kDStage);
    float* tile = s_out[lane];
    if (ACZ_DEC_STATS && lane == 0) atomicAdd(&g_dclk[0], (unsigned long long)(clock64() - tk0));
    const uint64_t ntasks = (a.nchunks + 31) / 32;
    const uint64_t I = a.interval;
    for (uint64_t task = (uint64_t)blockIdx.x * kDW + w; task < ntasks;
         task += (uint64_t)gridDim.x * kDW) {
        const long long tk1 = clock64();
        const uint64_t chunk0 = task * 32;
        const uint64_t chunk = chunk0 + lane;
        const bool active = chunk < a.nchunks;
        const uint64_t start = chunk * I;
        const uint32_t cnt = active ? (uint32_t)min(I, a.g.n - start) : 0u;
        const uint64_t pos = active ? a.side_bitoff[chunk] : 0;
        const double r = active ? (double)a.side_state[chunk] : 0.0;
        // chunk offset of the first plane start in the chunk (the next ones follow every P)
        const uint64_t pin64 = start % a.g.plane_size;
        const uint32_t pin =
            pin64 == 0 ? 0u : (uint32_t)min(a.g.plane_size - pin64, (uint64_t)0xFFFFFFFFu);
        // the task's stream span [b0, b1) in bits, staged as words [w0, w0 + nw)
        const uint64_t b0 = __shfl_sync(0xffffffffu, pos, 0);
        const uint64_t b1 = chunk0 + 32 < a.nchunks ? a.side_bitoff[chunk0 + 32] : a.bit_length;
        const uint64_t w0 = (b0 >> 5) & ~3ull;         // 16-byte aligned start
        const uint64_t nw = ((b1 + 31) >> 5) + 3 - w0;  // + 3 words of look-ahead
        if (nw <= (uint64_t)kDStage) {
            // the words array is padded by 32 words, so the rounded-up tail is readable
            for (uint64_t i = lane; i < (nw + 3) / 4; i += 32)
                cp_async16(s_bits + 4 * i, a.words + w0 + 4 * i);
            cp_async_commit();
            cp_async_wait<0>();
            __syncwarp();
            const long long tk2 = clock64();
            decode_chunk<true, uint32_t>(a, s_bits, (uint32_t)(pos - w0 * 32), s_lut, lbook, lfirst,
                                         s_lim, s_ct, cnt, start, r, pin, tile, s_out, chunk0, lane);
            if (ACZ_DEC_STATS && lane == 0) {
                atomicAdd(&g_dclk[1], (unsigned long long)(tk2 - tk1));
                atomicAdd(&g_dclk[2], (unsigned long long)(clock64() - tk2));
                atomicAdd(&g_dclk[3], 1ull);
            }
        } else {
            decode_chunk<false, uint64_t>(a, a.words, pos, s_lut, lbook, lfirst, s_lim, s_ct, cnt,
                                          start, r, pin, tile, s_out, chunk0, lane);
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(128) k_decode_lorenzo(DecodeArgs a) {
    extern __shared__ uint32_t s_lut[];
    __shared__ CanonTables s_ct;
    load_tables(a.lut, a.canon, s_lut, &s_ct);
    const uint64_t plane = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (plane >= a.g.planes) return;
    const uint64_t rows = a.g.rows, cols = a.g.cols;
    const uint64_t base = plane * a.g.plane_size;
    uint64_t pos = a.side_bitoff[plane];
    uint32_t oi = a.side_outl[plane];
    float* row = a.row_scratch + plane * cols;
    const long long R = a.radius;
    BitReader br;
    br.init(a.words, a.nwords, pos);
    for (uint64_t r = 0; r < rows; ++r) {
        float left = 0.0f, topleft = 0.0f;
        for (uint64_t c = 0; c < cols; ++c) {
            const uint64_t flat = base + r * cols + c;
            uint32_t sym = 0;
            decode_one(br, pos, s_lut, s_ct, a.book_sym, &sym);
            const float top = r > 0 ? row[c] : 0.0f;
            float v;
            if (sym == 0) {
                v = __ldg(a.out_value + oi);
                ++oi;
            } else {
                const double dl = c > 0 ? (double)left : 0.0;
                const double dt = r > 0 ? (double)top : 0.0;
                const double dtl = (r > 0 && c > 0) ? (double)topleft : 0.0;
                const double pred = __dsub_rn(__dadd_rn(dl, dt), dtl);
                v = recon_value(pred, (double)((long long)sym - R), a.step);
            }
            topleft = top;
            row[c] = v;
            left = v;
            a.out[flat] = (a.zero_filter && fabs((double)v) <= a.eb) ? 0.0f : v;
        }
    }
}

// Lorenzo2d decode for the wavefront path: (1) a thread per plane decodes the plane's
// symbols from its sidecar bit offset into a scratch array; (2) a warp per plane rebuilds
// the values by anti-diagonals (see k_quant_lorenzo_wave), escapes taking their outlier by
// binary search over the plane's slice of the (sorted) outlier list.
__global__ void __launch_bounds__(128) k_lorenzo_syms(DecodeArgs a, uint32_t* __restrict__ syms) {
    extern __shared__ uint32_t s_lut[];
    __shared__ CanonTables s_ct;
    load_tables(a.lut, a.canon, s_lut, &s_ct);
    const uint64_t chunk = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (chunk >= a.nchunks) return;
    const uint64_t start = chunk * a.interval;
    const uint64_t cnt = min(a.interval, a.g.n - start);
    uint64_t pos = a.side_bitoff[chunk];
    BitReader br;
    br.init(a.words, a.nwords, pos);
    for (uint64_t i = 0; i < cnt; ++i) {
        uint32_t sym = 0;
        decode_one(br, pos, s_lut, s_ct, a.book_sym, &sym);
        syms[start + i] = sym;
    }
}

__global__ void __launch_bounds__(32) k_decode_lorenzo_wave(DecodeArgs a,
                                                            const uint32_t* __restrict__ syms) {
    extern __shared__ float diag[];  // 3 x rows
    const uint64_t plane = blockIdx.x;
    if (plane >= a.g.planes) return;
    const int lane = threadIdx.x;
    const int rows = (int)a.g.rows, cols = (int)a.g.cols;
    const uint64_t base = plane * a.g.plane_size;
    const uint32_t* sp = syms + base;
    float* op = a.out + base;
    // the plane's outliers lie between the prefixes of its first and one-past-last chunks
    const uint64_t c0 = base / a.interval, c1 = (base + a.g.plane_size - 1) / a.interval + 1;
    const uint32_t o0 = a.side_outl[c0];
    const uint32_t o1 = c1 < a.nchunks ? a.side_outl[c1] : (uint32_t)a.n_outliers;
    const long long R = a.radius;
    const float zthr = a.zero_filter ? __double2float_rd(a.eb) : -1.0f;
    float* d0 = diag;
    float* d1 = diag + rows;
    float* d2 = diag + 2 * rows;
    for (int d = 0; d < rows + cols - 1; ++d) {
        const int r_lo = d - (cols - 1) > 0 ? d - (cols - 1) : 0;
        const int r_hi = d < rows - 1 ? d : rows - 1;
        for (int r = r_lo + lane; r <= r_hi; r += 32) {
            const int c = d - r;
            const uint64_t off = (uint64_t)r * cols + c;
            const uint32_t sym = __ldg(sp + off);
            float v;
            if (sym == 0) {
                uint32_t lo = o0, hi = o1;  // the outlier record of flat index base + off
                const unsigned long long key = base + off;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (__ldg(a.out_index + mid) < key) lo = mid + 1; else hi = mid;
                }
                v = __ldg(a.out_value + lo);
            } else {
                const double dl = c > 0 ? (double)d1[r] : 0.0;
                const double dt = r > 0 ? (double)d1[r - 1] : 0.0;
                const double dtl = (r > 0 && c > 0) ? (double)d2[r - 1] : 0.0;
                const double pred = __dsub_rn(__dadd_rn(dl, dt), dtl);
                v = recon_value(pred, (double)((long long)sym - R), a.step);
            }
            d0[r] = v;
            op[off] = fabsf(v) <= zthr ? 0.0f : v;
        }
        __syncwarp();
        float* t = d2;
        d2 = d1;
        d1 = d0;
        d0 = t;
    }
}

// Single-thread sequential decode of the whole stream (foreign blobs, generic Huffman).
__global__ void k_scan_decode(ScanArgs a) {
    extern __shared__ uint32_t s_lut[];
    __shared__ CanonTables s_ct;
    load_tables(a.lut, a.canon, s_lut, &s_ct);
    if (threadIdx.x != 0) return;
    BitReader br;
    br.init(a.words, a.nwords, 0);
    uint64_t pos = 0;
    uint64_t oi = 0;
    unsigned deferred = 0;
    uint64_t next_side = 0, next_plane = 0;
    for (uint64_t flat = 0; flat < a.n; ++flat) {
        if (flat == next_side) {
            if (a.side_bitoff) {
                a.side_bitoff[flat / a.interval] = pos;
                if (a.side_outl) a.side_outl[flat / a.interval] = (uint32_t)oi;
            }
            next_side += a.interval;
        }
        if (flat == next_plane) {
            if (a.plane_outl) a.plane_outl[flat / a.plane_size] = oi;
            next_plane += a.plane_size;
        }
        uint32_t sym = 0;
        const uint64_t p0 = pos;
        const uint32_t len = decode_one(br, pos, s_lut, s_ct, a.book_sym, &sym);
        if (len == 0) {
            // the reference reads up to 64 bits (or until the stream ends) without a match
            atomicOr(a.flags, (p0 + 64 > a.bit_length) ? kDecTruncated : kDecNoMatch);
            return;
        }
        if (pos > a.bit_length) {
            atomicOr(a.flags, kDecTruncated);
            return;
        }
        if (a.sym_out) a.sym_out[flat] = sym;
        if (sym == 0 && a.out_index) {
            if (oi >= a.n_outliers) deferred |= deferred ? 0u : kDecOutlierMissing;
            else if (a.out_index[oi] != flat) deferred |= deferred ? 0u : kDecOutlierIndex;
            ++oi;
        }
    }
    if (a.out_index && !deferred && oi != a.n_outliers) deferred = kDecOutlierUnused;
    if (deferred) atomicOr(a.flags, deferred);
}

__global__ void __launch_bounds__(128) k_chain_states(const uint32_t* __restrict__ sym,
                                                      const unsigned long long* plane_outl,
                                                      const float* __restrict__ out_value,
                                                      PlaneGeom g, double step, uint32_t radius,
                                                      uint64_t interval, float* side_state) {
    const uint64_t plane = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (plane >= g.planes) return;
    const uint64_t P = g.plane_size, base = plane * P;
    uint64_t oi = plane_outl[plane];
    const long long R = radius;
    float r = 0.0f;
    uint64_t to_side = base % interval;
    to_side = to_side == 0 ? 0 : interval - to_side;
    // the symbols of a plane are read 16 at a time ahead of the chain (independent loads in
    // flight instead of one memory round trip per step)
    constexpr int kAhead = 16;
    uint32_t sb[kAhead];
    for (uint64_t i = 0; i < P; ++i) {
        const uint64_t flat = base + i;
        const int slot = (int)(i % kAhead);
        if (slot == 0) {
#pragma unroll
            for (int k = 0; k < kAhead; ++k) sb[k] = i + k < P ? __ldg(sym + flat + k) : 0u;
        }
        if (to_side == 0) {
            side_state[flat / interval] = i == 0 ? 0.0f : r;
            to_side = interval;
        }
        --to_side;
        uint32_t s = sb[0];
#pragma unroll
        for (int k = 1; k < kAhead; ++k)
            if (slot == k) s = sb[k];
        float v;
        if (s == 0) {
            v = out_value[oi++];
        } else {
            const double pred = i == 0 ? 0.0 : (double)r;
            v = recon_value(pred, (double)((long long)s - R), step);
        }
        r = v;
    }
}

// ---- parallel foreign-stream scan (ref src/huffman.cpp:137-189 + src/codec.cpp:138-169) ----
// The bitstream is cut into subsequences of kPsBits bits; a thread decodes the codewords
// that START in its subsequence. The true start of subsequence i is the end of the last
// codeword that started in subsequence i-1, unknown up front: every thread first decodes from
// its nominal start, then starts are replaced by the predecessors' exits and the changed
// subsequences re-decoded until nothing changes. Canonical Huffman codes resynchronise within
// a few codewords, so a wrong start only perturbs the first few symbols of a subsequence and
// the fixed point is reached in a handful of passes (capped; the sequential scan is the
// fallback). A last pass decodes every subsequence from its true start at its global symbol
// index (a scan of the per-subsequence counts), writes what the sequential scan writes, and
// records the first error of each kind in flat order.
constexpr uint64_t kPsBits = 2048;
constexpr int kPsThreads = 256;

struct PsState {
    unsigned long long err_dec;   // (flat << 1 | nomatch) of the first decode error, or ~0
    unsigned long long err_out;   // (flat << 1 | index) of the first outlier error, or ~0
    unsigned long long esc_n;     // escapes among the first n symbols
    unsigned long long total;     // symbols in the stream (Σ counts)
    unsigned int changed;
};

__global__ void __launch_bounds__(kPsThreads) k_ps_sync(ScanArgs a, unsigned long long* starts,
                                                        unsigned long long* exits,
                                                        uint32_t* cnt, uint32_t* esc,
                                                        uint32_t* dirty, uint64_t M) {
    extern __shared__ uint32_t s_lut[];
    __shared__ CanonTables s_ct;
    load_tables(a.lut, a.canon, s_lut, &s_ct);
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= M || !dirty[i]) return;
    const uint64_t end = min((i + 1) * kPsBits, a.bit_length);
    uint64_t pos = starts[i];
    BitReader br;
    br.init(a.words, a.nwords, pos);
    uint32_t c = 0, e = 0;
    while (pos < end) {
        uint32_t sym = 0;
        const uint64_t p0 = pos;
        if (!decode_one(br, pos, s_lut, s_ct, a.book_sym, &sym)) {
            pos = p0;
            break;
        }
        ++c;
        e += sym == 0;
    }
    exits[i] = pos;
    cnt[i] = c;
    esc[i] = e;
    dirty[i] = 0;
}

__global__ void k_ps_fix(const unsigned long long* exits, unsigned long long* starts,
                         uint32_t* dirty, uint64_t M, PsState* st) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x + 1;
    if (i >= M) return;
    const unsigned long long e = exits[i - 1];
    if (starts[i] != e) {
        starts[i] = e;
        dirty[i] = 1;
        st->changed = 1;
    }
}

// exclusive scans of the counts (single CTA; a foreign-blob path, not the hot path)
__global__ void __launch_bounds__(1024) k_ps_scan(const uint32_t* cnt, const uint32_t* esc,
                                                  unsigned long long* base_sym,
                                                  unsigned long long* base_esc, uint64_t M,
                                                  PsState* st) {
    __shared__ unsigned long long s_a[32], s_b[32];
    __shared__ unsigned long long s_run_a, s_run_b;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        s_run_a = 0;
        s_run_b = 0;
    }
    __syncthreads();
    for (uint64_t c0 = 0; c0 < M; c0 += 1024) {
        const uint64_t i = c0 + tid;
        const unsigned long long va = i < M ? cnt[i] : 0, vb = i < M ? esc[i] : 0;
        unsigned long long ia = va, ib = vb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long xa = __shfl_up_sync(0xffffffffu, ia, o);
            const unsigned long long xb = __shfl_up_sync(0xffffffffu, ib, o);
            if (lane >= o) {
                ia += xa;
                ib += xb;
            }
        }
        if (lane == 31) {
            s_a[warp] = ia;
            s_b[warp] = ib;
        }
        __syncthreads();
        unsigned long long pa = s_run_a, pb = s_run_b, ta = 0, tb = 0;
        for (int w = 0; w < 32; ++w) {
            if (w < warp) {
                pa += s_a[w];
                pb += s_b[w];
            }
            ta += s_a[w];
            tb += s_b[w];
        }
        if (i < M) {
            base_sym[i] = pa + ia - va;
            base_esc[i] = pb + ib - vb;
        }
        __syncthreads();
        if (tid == 0) {
            s_run_a += ta;
            s_run_b += tb;
        }
        __syncthreads();
    }
    if (tid == 0) st->total = s_run_a;
}

__global__ void __launch_bounds__(kPsThreads) k_ps_final(ScanArgs a,
                                                         const unsigned long long* starts,
                                                         const unsigned long long* base_sym,
                                                         const unsigned long long* base_esc,
                                                         uint64_t M, PsState* st) {
    extern __shared__ uint32_t s_lut[];
    __shared__ CanonTables s_ct;
    load_tables(a.lut, a.canon, s_lut, &s_ct);
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    uint64_t g = base_sym[i];
    if (g >= a.n) return;
    uint64_t oi = base_esc[i];
    const uint64_t end = min((i + 1) * kPsBits, a.bit_length);
    uint64_t pos = starts[i];
    BitReader br;
    br.init(a.words, a.nwords, pos);
    while (pos < end && g < a.n) {
        if (g % a.interval == 0 && a.side_bitoff) {
            a.side_bitoff[g / a.interval] = pos;
            if (a.side_outl) a.side_outl[g / a.interval] = (uint32_t)oi;
        }
        if (a.plane_outl && g % a.plane_size == 0) a.plane_outl[g / a.plane_size] = oi;
        uint32_t sym = 0;
        const uint64_t p0 = pos;
        const uint32_t len = decode_one(br, pos, s_lut, s_ct, a.book_sym, &sym);
        if (len == 0) {
            atomicMin(&st->err_dec, ((unsigned long long)g << 1) | (p0 + 64 > a.bit_length ? 0ull : 1ull));
            return;
        }
        if (pos > a.bit_length) {
            atomicMin(&st->err_dec, (unsigned long long)g << 1);
            return;
        }
        if (a.sym_out) a.sym_out[g] = sym;
        if (sym == 0) {
            if (a.out_index) {
                if (oi >= a.n_outliers) atomicMin(&st->err_out, (unsigned long long)g << 1);
                else if (a.out_index[oi] != g)
                    atomicMin(&st->err_out, ((unsigned long long)g << 1) | 1ull);
            }
            ++oi;
        }
        ++g;
        if (g == a.n) st->esc_n = oi;
    }
}

// Flags exactly as the sequential scan would set them (first error in flat order).
__global__ void k_ps_flags(ScanArgs a, const PsState* st) {
    unsigned f = 0;
    if (st->err_dec != ~0ull) f = (st->err_dec & 1ull) ? kDecNoMatch : kDecTruncated;
    else if (st->total < a.n) f = kDecTruncated;
    else if (a.out_index && st->err_out != ~0ull)
        f = (st->err_out & 1ull) ? kDecOutlierIndex : kDecOutlierMissing;
    else if (a.out_index && st->esc_n != a.n_outliers) f = kDecOutlierUnused;
    if (f) atomicOr(a.flags, f);
}

__global__ void k_ps_init(unsigned long long* starts, uint32_t* dirty, uint64_t M, PsState* st) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < M) {
        starts[i] = i * kPsBits;
        dirty[i] = 1;
    }
    if (i == 0) {
        st->err_dec = ~0ull;
        st->err_out = ~0ull;
        st->esc_n = 0;
        st->total = 0;
        st->changed = 0;
    }
}

}  // namespace

cudaError_t set_decode_attrs() {
    static bool done = false;
    if (done) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(k_decode_prev, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kDecSmem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_ps_sync, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 4 * kLutSize);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_ps_final, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 4 * kLutSize);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_decode_lorenzo, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 4 * kLutSize);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_scan_decode, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 4 * kLutSize);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_lorenzo_syms, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 4 * kLutSize);
    done = e == cudaSuccess;
    return e;
}

cudaError_t launch_decode(const DecodeArgs& a, int sms, cudaStream_t s, uint64_t* launches) {
    cudaError_t e = set_decode_attrs();
    if (e != cudaSuccess) return e;
    const unsigned threads = 128;
    if (a.predictor == ACZ_PRED_PREV) {
        const uint64_t tasks = (a.nchunks + 31) / 32;
        uint64_t blocks = (tasks + kDW - 1) / kDW;
        if (blocks > (uint64_t)sms) blocks = sms;  // persistent: one CTA per SM
        k_decode_prev<<<(unsigned)blocks, kDW * 32, kDecSmem, s>>>(a);
    } else if (a.g.rows > 1 && a.g.rows <= kLorenzoWaveRows && a.sym_scratch) {
        const uint64_t blocks = (a.nchunks + threads - 1) / threads;
        k_lorenzo_syms<<<(unsigned)blocks, threads, 4 * kLutSize, s>>>(a, a.sym_scratch);
        k_decode_lorenzo_wave<<<(unsigned)a.g.planes, 32, 3 * 4 * a.g.rows, s>>>(a, a.sym_scratch);
        ++*launches;
    } else {
        const uint64_t blocks = (a.g.planes + threads - 1) / threads;
        k_decode_lorenzo<<<(unsigned)blocks, threads, 4 * kLutSize, s>>>(a);
    }
    ++*launches;
    return cudaGetLastError();
}

cudaError_t decode_stats(unsigned long long* out, bool reset) {
    cudaError_t e = cudaMemcpyFromSymbol(out, g_dclk, sizeof(g_dclk));
    if (e == cudaSuccess && reset) {
        unsigned long long z[4] = {0};
        e = cudaMemcpyToSymbol(g_dclk, z, sizeof(z));
    }
    return e;
}

size_t scan_decode_scratch_bytes(uint64_t bit_length) {
    const uint64_t M = (bit_length + kPsBits - 1) / kPsBits;
    return 256 + 8 * 4 * M + 4 * 3 * M + 1024;
}

cudaError_t launch_scan_decode(const ScanArgs& a, void* scratch, cudaStream_t s,
                               uint64_t* launches) {
    cudaError_t e = set_decode_attrs();
    if (e != cudaSuccess) return e;
    const uint64_t M = (a.bit_length + kPsBits - 1) / kPsBits;
    const bool force_seq = std::getenv("ACZ_SCAN_SEQUENTIAL") != nullptr;  // testing
    if (!scratch || M < 64 || force_seq) {  // short streams: one sequential pass
        k_scan_decode<<<1, 128, 4 * kLutSize, s>>>(a);
        ++*launches;
        return cudaGetLastError();
    }
    char* p = static_cast<char*>(scratch);
    PsState* st = reinterpret_cast<PsState*>(p);
    unsigned long long* starts = reinterpret_cast<unsigned long long*>(p + 256);
    unsigned long long* exits = starts + M;
    unsigned long long* base_sym = exits + M;
    unsigned long long* base_esc = base_sym + M;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(base_esc + M);
    uint32_t* esc = cnt + M;
    uint32_t* dirty = esc + M;
    const unsigned blocks = (unsigned)((M + kPsThreads - 1) / kPsThreads);
    k_ps_init<<<blocks, kPsThreads, 0, s>>>(starts, dirty, M, st);
    ++*launches;
    bool converged = false;
    for (int it = 0; it < 48 && !converged; ++it) {
        k_ps_sync<<<blocks, kPsThreads, 4 * kLutSize, s>>>(a, starts, exits, cnt, esc, dirty, M);
        e = cudaMemsetAsync(&st->changed, 0, sizeof(unsigned), s);
        if (e != cudaSuccess) return e;
        k_ps_fix<<<blocks, kPsThreads, 0, s>>>(exits, starts, dirty, M, st);
        *launches += 2;
        unsigned changed = 1;
        e = cudaMemcpyAsync(&changed, &st->changed, sizeof(unsigned), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return e;
        converged = changed == 0;
    }
    if (!converged) {  // no resynchronisation (adversarial stream): sequential scan
        k_scan_decode<<<1, 128, 4 * kLutSize, s>>>(a);
        ++*launches;
        return cudaGetLastError();
    }
    k_ps_scan<<<1, 1024, 0, s>>>(cnt, esc, base_sym, base_esc, M, st);
    k_ps_final<<<blocks, kPsThreads, 4 * kLutSize, s>>>(a, starts, base_sym, base_esc, M, st);
    k_ps_flags<<<1, 1, 0, s>>>(a, st);
    *launches += 3;
    return cudaGetLastError();
}

cudaError_t launch_chain_states(const uint32_t* sym, const unsigned long long* plane_outl,
                                const float* out_value, PlaneGeom g, double step,
                                uint32_t radius, uint64_t interval, float* side_state,
                                int sms, cudaStream_t s, uint64_t* launches) {
    (void)sms;
    const unsigned threads = 128;
    const uint64_t blocks = (g.planes + threads - 1) / threads;
    k_chain_states<<<(unsigned)blocks, threads, 0, s>>>(sym, plane_outl, out_value, g, step,
                                                        radius, interval, side_state);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace acz_b200
