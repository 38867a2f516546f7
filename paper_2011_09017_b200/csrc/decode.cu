// K6 Huffman decode + K7 reconstruction (ref src/huffman.cpp:137-189, src/codec.cpp:122-171).
//
// k_decode_prev   : one thread per sidecar chunk (`interval` symbols). The sidecar gives
//                   the chunk's bit offset, outlier prefix and the chain state before its
//                   first element, so every chunk decodes and reconstructs independently and
//                   bit-exactly. Canonical decode via a 4096-entry shared-memory LUT
//                   (codes <= 12 bits), per-length canonical ranges for longer codes.
// k_decode_lorenzo: Lorenzo2d, one thread per plane (sidecar interval = plane size).
// k_scan_decode   : sequential whole-stream decode used to (re)build the sidecar of a
//                   foreign ACZ1 blob and to validate it exactly like the reference
//                   (truncation / no-match DecodeError, outlier FormatErrors).
// k_chain_states  : thread-per-plane chain replay producing the sidecar chain states.
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
    __device__ __forceinline__ uint32_t peek12() const { return (uint32_t)(buf >> (64 - kLutBits)); }
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
    const uint32_t e = s_lut[br.peek12()];
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
    for (int i = threadIdx.x; i < kLutSize; i += blockDim.x) s_lut[i] = __ldg(lut + i);
    for (int i = threadIdx.x; i < 65; i += blockDim.x) {
        s_ct->first_code[i] = canon->first_code[i];
        s_ct->first_index[i] = canon->first_index[i];
        s_ct->count[i] = canon->count[i];
    }
    __syncthreads();
}

// Exact RN32 of a double kept in a double register (no F2F on the dependency chain):
// adding and subtracting 1.5 * 2^(e+29) rounds y to 24 significant bits, ties to even.
// Valid for y in the float normal range; other inputs take the conversion path.
__device__ __forceinline__ double rn32_in_double(double y) {
    const int hi = __double2hiint(y);
    const int ex = (hi >> 20) & 0x7FF;
    if (ex < 1023 - 126 || ex > 1023 + 127) return (double)__double2float_rn(y);
    const double M = __hiloint2double((ex << 20) + ((29 << 20) | (1 << 19)), 0);
    return __dsub_rn(__dadd_rn(y, M), M);
}

// Canonical decode limits (left-aligned): the code length of a 64-bit window w is the
// smallest l with (w >> (64 - l)) < limit[l]; codes of length l are [nc[l], limit[l]).
struct Limits {
    unsigned long long nc[65];
    unsigned long long lim[65];
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
            if (ct.count[l]) L->maxlen = l;
        }
    }
}

__global__ void __launch_bounds__(128) k_decode_prev(DecodeArgs a) {
    __shared__ uint32_t s_lut[kLutSize];
    __shared__ CanonTables s_ct;
    __shared__ Limits s_lim;
    load_tables(a.lut, a.canon, s_lut, &s_ct);
    build_limits(s_ct, &s_lim);
    __syncthreads();
    const uint64_t chunk = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (chunk >= a.nchunks) return;
    const uint64_t start = chunk * a.interval;
    const uint64_t end = min(a.g.n, start + a.interval);
    uint64_t pos = a.side_bitoff[chunk];
    uint32_t oi = a.side_outl[chunk];
    double r = (double)a.side_state[chunk];
    const uint64_t P = a.g.plane_size;
    uint64_t pin = start % P;
    const int R = (int)a.radius;
    const double step = a.step, eb = a.eb;
    const bool zf = a.zero_filter != 0;
    // bit reader: 64-bit MSB-aligned buffer; words are stored byte-swapped (ACZ1 order)
    const uint32_t* W = a.words;
    const bool short_codes = s_lim.maxlen <= 32;  // buffer always holds a whole code
    uint64_t wi = pos >> 5;
    const int off = (int)(pos & 31);
    unsigned long long buf =
        ((((unsigned long long)bswap32(__ldg(W + wi))) << 32) | bswap32(__ldg(W + wi + 1))) << off;
    int nb = 64 - off;
    wi += 2;
    float ob[8];
    uint64_t flat = start;
    while (flat < end) {
        // decode one symbol
        if (nb <= 32) {
            if ((wi & 31) == 0 && wi + 32 < a.nwords)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(W + wi + 32));
            buf |= (unsigned long long)bswap32(__ldg(W + wi)) << (32 - nb);
            ++wi;
            nb += 32;
        }
        const uint32_t e = s_lut[(uint32_t)(buf >> (64 - kLutBits))];
        uint32_t len = e & 31, sym;
        if (len) {
            sym = e >> 5;
        } else {
            // long code: canonical limit search (window has >= 33 valid bits; codes longer
            // than the buffer use an absolute 64-bit window)
            unsigned long long w = buf;
            if (!short_codes) {
                const uint64_t ap = (wi << 5) - (uint64_t)nb;  // absolute position of buf's MSB
                const uint64_t i = ap >> 5;
                const int o = (int)(ap & 31);
                const unsigned long long x0 = bswap32(__ldg(W + i)), x1 = bswap32(__ldg(W + i + 1)),
                                         x2 = bswap32(__ldg(W + i + 2));
                const unsigned long long h = (x0 << 32) | x1;
                w = o ? (h << o) | (x2 << o >> 32) : h;
            }
            len = kLutBits + 1;
            while (len < 64 && (w >> (64 - len)) >= s_lim.lim[len]) ++len;
            const unsigned long long c = w >> (64 - len);
            sym = __ldg(a.book_sym + s_ct.first_index[len] + (uint32_t)(c - s_lim.nc[len]));
        }
        if (len >= 64) {
            buf = 0;
        } else {
            buf <<= len;
        }
        nb -= (int)len;
        if (nb < 0) {
            // consumed beyond the buffer (code longer than the valid bits): re-sync
            const uint64_t ap = (wi << 5) - (uint64_t)(nb + (int)len) + len;
            wi = ap >> 5;
            const int o2 = (int)(ap & 31);
            buf = ((((unsigned long long)bswap32(__ldg(W + wi))) << 32) | bswap32(__ldg(W + wi + 1))) << o2;
            nb = 64 - o2;
            wi += 2;
        }
        // reconstruct (ref src/codec.cpp:143-164); r stays an exact float value in double
        float v;
        if (sym == 0) {
            v = __ldg(a.out_value + oi);
            ++oi;
            r = (double)v;
        } else {
            const double pred = pin == 0 ? 0.0 : r;
            const double y = __dadd_rn(pred, __dmul_rn((double)((int)sym - R), step));
            r = rn32_in_double(y);
            v = (float)r;
        }
        const float o = (zf && fabs(r) <= eb) ? 0.0f : v;
        const int slot = (int)(flat & 7);
        ob[slot] = o;
        ++flat;
        if (++pin == P) pin = 0;
        if (slot == 7) {
            float4* dst = reinterpret_cast<float4*>(a.out + flat - 8);
            dst[0] = make_float4(ob[0], ob[1], ob[2], ob[3]);
            dst[1] = make_float4(ob[4], ob[5], ob[6], ob[7]);
        }
    }
    // tail (chunk end not 8-aligned: only the tensor's last chunk)
    const int rem = (int)(flat & 7);
    for (int t = 0; t < rem; ++t) a.out[flat - rem + t] = ob[t];
}

__global__ void __launch_bounds__(128) k_decode_lorenzo(DecodeArgs a) {
    __shared__ uint32_t s_lut[kLutSize];
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

// Single-thread sequential decode of the whole stream (foreign blobs, generic Huffman).
__global__ void k_scan_decode(ScanArgs a) {
    __shared__ uint32_t s_lut[kLutSize];
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
                a.side_outl[flat / a.interval] = (uint32_t)oi;
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
    for (uint64_t i = 0; i < P; ++i) {
        const uint64_t flat = base + i;
        if (to_side == 0) {
            side_state[flat / interval] = i == 0 ? 0.0f : r;
            to_side = interval;
        }
        --to_side;
        const uint32_t s = sym[flat];
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

}  // namespace

cudaError_t launch_decode(const DecodeArgs& a, int sms, cudaStream_t s, uint64_t* launches) {
    (void)sms;
    const unsigned threads = 128;
    if (a.predictor == ACZ_PRED_PREV) {
        const uint64_t blocks = (a.nchunks + threads - 1) / threads;
        k_decode_prev<<<(unsigned)blocks, threads, 0, s>>>(a);
    } else {
        const uint64_t blocks = (a.g.planes + threads - 1) / threads;
        k_decode_lorenzo<<<(unsigned)blocks, threads, 0, s>>>(a);
    }
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_scan_decode(const ScanArgs& a, cudaStream_t s, uint64_t* launches) {
    k_scan_decode<<<1, 128, 0, s>>>(a);
    ++*launches;
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
