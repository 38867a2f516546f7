// K3 histogram, K4 codebook, K5 encode: the canonical Huffman coder of the reference
// (ref src/huffman.cpp:22-135), bit-exact.
//
// K3  k_histogram   : shared-memory privatised histogram over a window of 32768 bins
//                     centred on the zero-residual symbol (quant_radius; one 1024-thread CTA
//                     per SM), the zero-residual symbol itself counted in registers;
//                     out-of-window symbols go straight to global u64 atomics. The last CTA
//                     to finish builds the codebook (K4 fused).
// K4  k_codebook    : single 1024-thread CTA. Compaction of non-zero bins (ascending
//                     symbol order == the reference's std::map order, huffman.cpp:110),
//                     stable LSD radix sort of the leaves by frequency, two-queue merge
//                     (leaf wins frequency ties, internal nodes FIFO) which reproduces the
//                     reference heap's (freq, creation-index) pop order exactly
//                     (huffman.cpp:25-54), depths by pointer jumping, canonical
//                     (length, symbol) order by a stable counting sort (huffman.cpp:116-125),
//                     canonical codes (huffman.cpp:75-86), decode LUT.
// K5  k_encode_count: per-256-symbol-chunk bit / escape counts (persistent 1024-thread
//                     CTAs, one decoupled look-back across CTAs, CTA scan -> absolute chunk
//                     offsets); k_encode_write: a warp per chunk, bit concatenation in a
//                     per-warp shared stage, coalesced word stores (boundary words by
//                     atomicOr). Also writes the outlier list and the decode sidecar (bit
//                     offset / outlier prefix every `interval` symbols).
#include <algorithm>
#include <type_traits>

#include "internal.h"

namespace acz_b200 {

namespace {

// Shared-memory window of the histogram (bins centred on the zero-residual symbol): wide
// enough for error bounds down to 1e-4 on unit-scale activations (symbols spread over about
// +-5000 around the centre) so that out-of-window global atomics stay rare.
#ifndef ACZ_HIST_WINDOW
#define ACZ_HIST_WINDOW 32768
#endif
constexpr int kHistWindow = ACZ_HIST_WINDOW;
constexpr int kHistThreads = 1024;
#ifndef ACZ_HIST_LOADS
#define ACZ_HIST_LOADS 4
#endif
constexpr int kHistLoads = ACZ_HIST_LOADS;

// --------------------------------------------------------------------------- K3 ----
// The histogram buffer is self-cleaning: the codebook kernel zeroes every bin it reads and
// the `touched` bitmap, so no per-call memset of the 2R-bin table is needed.
__device__ __forceinline__ void codebook_fast_body(
    unsigned long long* __restrict__ hist, uint32_t* __restrict__ touched, uint32_t alphabet,
    uint32_t* __restrict__ book_sym, uint8_t* __restrict__ book_len,
    unsigned long long* __restrict__ enc, CanonTables* __restrict__ canon,
    uint32_t* __restrict__ lut, BookInfo* __restrict__ info);

// With cb.done set, the last histogram CTA to finish builds the codebook (K3+K4 fused): the
// single-CTA codebook then needs no SM of its own -- launched separately it waited for a
// whole SM to drain of other tensors' kernels (~20 us on the AlexNet critical path).
template <typename SymT>
__global__ void __launch_bounds__(kHistThreads) k_histogram(const SymT* __restrict__ sym, uint64_t n,
                                                   uint32_t alphabet, uint32_t win_lo,
                                                   uint32_t win_n, uint32_t center,
                                                   unsigned long long* __restrict__ hist,
                                                   uint32_t* __restrict__ touched, CbArgs cb) {
    extern __shared__ unsigned int bins[];  // kHistWindow
    for (uint32_t i = threadIdx.x; i < kHistWindow; i += blockDim.x) bins[i] = 0;
    __syncthreads();
    // the zero-residual symbol (about half of all ReLU activations) is counted in a register:
    // no shared-memory atomic contention on the hottest bin
    uint32_t c0 = 0;
    auto count = [&](uint32_t e) {
        if (e == center) {
            ++c0;
            return;
        }
        const uint32_t o = e - win_lo;
        if (o < win_n) {
            atomicAdd(&bins[o], 1u);
        } else if (e < alphabet) {
            atomicAdd(&hist[e], 1ull);
            atomicOr(&touched[e >> 5], 1u << (e & 31));
        }
    };
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    constexpr int V = 16 / sizeof(SymT);  // symbols per 128-bit load
    const uint64_t nv = ((reinterpret_cast<uintptr_t>(sym) & 15) == 0) ? n / V : 0;
    const uint4* s4 = reinterpret_cast<const uint4*>(sym);
    auto count4 = [&](const uint4 v) {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (sizeof(SymT) == 2) {
                count(w[k] & 0xFFFFu);
                count(w[k] >> 16);
            } else {
                count(w[k]);
            }
        }
    };
    // kHistLoads 128-bit loads per thread in flight before counting (one CTA per SM: the
    // loads in flight, not the counting, bound the pass)
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    for (; i + (kHistLoads - 1) * stride < nv; i += kHistLoads * stride) {
        uint4 v[kHistLoads];
#pragma unroll
        for (int u = 0; u < kHistLoads; ++u) v[u] = __ldcs(s4 + i + u * stride);
#pragma unroll
        for (int u = 0; u < kHistLoads; ++u) count4(v[u]);
    }
    for (; i < nv; i += stride) count4(__ldcs(s4 + i));
    for (uint64_t i = nv * V + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += stride)
        count((uint32_t)sym[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c0 += __shfl_xor_sync(0xffffffffu, c0, o);
    if ((threadIdx.x & 31) == 0 && c0) atomicAdd(&bins[center - win_lo], c0);
    __syncthreads();
    // flush: win_lo is a multiple of 32, so a warp's 32 consecutive bins are one bitmap word
    for (uint32_t i = threadIdx.x; i < kHistWindow; i += blockDim.x) {
        const uint32_t b = i < win_n ? bins[i] : 0u;
        if (b) atomicAdd(&hist[win_lo + i], (unsigned long long)b);
        const unsigned m = __ballot_sync(0xffffffffu, b != 0);
        if ((threadIdx.x & 31) == 0 && m) atomicOr(&touched[(win_lo + i) >> 5], m);
    }
    if (!cb.done) return;
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(cb.done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x == 0) *cb.done = 0;  // ready for the next call on this slot
    codebook_fast_body(hist, touched, alphabet, cb.book_sym, cb.book_len, cb.enc, cb.canon,
                       cb.lut, cb.info);
}

// --------------------------------------------------------------------------- K4 ----
constexpr int kCbThreads = 1024;
constexpr int kCbWarps = kCbThreads / 32;
constexpr int kRadixBits = 4;
constexpr int kRadixBuckets = 1 << kRadixBits;
constexpr uint64_t kSmemQueue = 16384;  // internal-node FIFO kept in shared memory

struct CbScratch {
    uint32_t* leaf_sym;           // k, ascending symbol
    unsigned long long* leaf_freq;
    unsigned long long* key_a;    // radix ping-pong (freq)
    unsigned long long* key_b;
    uint32_t* val_a;              // leaf ids
    uint32_t* val_b;
    unsigned long long* ifreq;    // internal-node frequencies (global fallback)
    uint32_t* anc_a;              // 2k-1 nodes
    uint32_t* anc_b;
    uint32_t* dist_a;
    uint32_t* dist_b;
};

__host__ __device__ inline size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

__host__ __device__ inline CbScratch carve(void* base, uint64_t k) {
    char* p = static_cast<char*>(base);
    CbScratch s;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char* r = p + off;
        off += align256(bytes);
        return r;
    };
    s.leaf_sym = reinterpret_cast<uint32_t*>(take(4 * k));
    s.leaf_freq = reinterpret_cast<unsigned long long*>(take(8 * k));
    s.key_a = reinterpret_cast<unsigned long long*>(take(8 * k));
    s.key_b = reinterpret_cast<unsigned long long*>(take(8 * k));
    s.val_a = reinterpret_cast<uint32_t*>(take(4 * k));
    s.val_b = reinterpret_cast<uint32_t*>(take(4 * k));
    s.ifreq = reinterpret_cast<unsigned long long*>(take(8 * k));
    s.anc_a = reinterpret_cast<uint32_t*>(take(4 * 2 * k));
    s.anc_b = reinterpret_cast<uint32_t*>(take(4 * 2 * k));
    s.dist_a = reinterpret_cast<uint32_t*>(take(4 * 2 * k));
    s.dist_b = reinterpret_cast<uint32_t*>(take(4 * 2 * k));
    return s;
}

// Block-wide exclusive scan of one u32 per thread (1024 threads). Returns the exclusive
// prefix; *total receives the block sum. `tmp` holds kCbWarps + 1 words.
__device__ __forceinline__ uint32_t block_scan_u32(uint32_t v, uint32_t* tmp, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) tmp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < kCbWarps ? tmp[lane] : 0;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < kCbWarps) tmp[lane] = wi - w;
        if (lane == kCbWarps - 1) tmp[kCbWarps] = wi;
    }
    __syncthreads();
    uint32_t res = tmp[warp] + inc - v;
    *total = tmp[kCbWarps];
    __syncthreads();
    return res;
}

// Canonical decode tables + LUT from per-length counts (shared by both codebook paths and
// the foreign-blob table builder). Canonical codes (ref src/huffman.cpp:75-86): the first
// code of length l is end(l-1) << 1, end(l) = first(l) + count(l). A LUT index v (the next
// kLutBits stream bits) decodes to the smallest l with v < end(l) << (kLutBits - l) -- a
// 4-step binary search over the left-justified limits; v beyond them is a long code (0).
__device__ void write_tables(const uint32_t* s_count, const unsigned long long* s_first_code,
                             const uint32_t* s_first_index, const uint32_t* book_sym,
                             CanonTables* canon, uint32_t* lut) {
    __shared__ uint32_t s_lj[kLutBits + 1];
    __shared__ uint32_t s_start[kLutBits + 1];
    const int tid = threadIdx.x;
    if (tid < 65) {
        canon->first_code[tid] = s_first_code[tid];
        canon->first_index[tid] = s_first_index[tid];
        canon->count[tid] = s_count[tid];
    }
    if (tid == 0) {
        unsigned long long end = 0;
        s_lj[0] = 0;
        for (int l = 1; l <= kLutBits; ++l) {
            const unsigned long long st = end << 1;
            end = st + s_count[l];
            s_start[l] = (uint32_t)st;
            s_lj[l] = (uint32_t)min(end << (kLutBits - l), (unsigned long long)kLutSize);
        }
    }
    // Long-code prefixes: a LUT index v past the short codes is the kLutBits-bit prefix of a
    // code longer than kLutBits; its length lies in [lmin(v), lmax(v)], lmin = the smallest l
    // with v < ceil(end(l) / 2^(l - kLutBits)), lmax = the smallest l with
    // v < floor(end(l) / 2^(l - kLutBits)) (every window with that prefix ends by then).
    // The entry keeps len = 0 (long) and carries lmin | lmax << 7 above the length field so
    // the sidecar decoder starts its limit search at lmin and stops at lmax.
    __shared__ uint32_t s_bc[65], s_bf[65];
    if (tid > kLutBits && tid <= 64) {  // one thread per length: end(l) = end(j) << (l - j),
        const int l = tid;               // j = the longest used length <= l
        int j = l;
        while (j > 0 && s_count[j] == 0) --j;
        const unsigned long long endj = j ? s_first_code[j] + s_count[j] : 0ull;
        const int sh = l - kLutBits;
        const unsigned long long hi = (endj << (l - j)) >> sh;  // l < 64: no overflow
        const bool big = l == 64 || hi >= (unsigned long long)kLutSize;
        const bool frac = ((endj << (l - j)) & ((1ull << sh) - 1)) != 0;
        s_bf[l] = big ? (uint32_t)kLutSize : (uint32_t)hi;
        s_bc[l] = big ? (uint32_t)kLutSize : (uint32_t)hi + (frac ? 1u : 0u);
    }
    __syncthreads();
    for (uint32_t v = tid; v < kLutSize; v += blockDim.x) {
        uint32_t e = 0;
        if (v >= s_lj[kLutBits]) {
            // both bounds are nondecreasing in l (end(l+1) >= 2 end(l)): binary searches
            uint32_t lo = kLutBits + 1, hi = 64;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (v < s_bc[mid]) hi = mid; else lo = mid + 1;
            }
            const uint32_t lmin = lo;
            hi = 64;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (v < s_bf[mid]) hi = mid; else lo = mid + 1;
            }
            e = (lmin << 5) | (lo << 12);
        }
        if (v < s_lj[kLutBits]) {
            int lo = 1, hi = kLutBits;  // smallest l with v < lj[l]
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (v < s_lj[mid]) hi = mid; else lo = mid + 1;
            }
            const uint32_t c = v >> (kLutBits - lo);
            e = (book_sym[s_first_index[lo] + (c - s_start[lo])] << 5) | (uint32_t)lo;
        }
        lut[v] = e;
    }
}

// Fast K4: every structure of the tree build lives in shared memory (books of up to
// kFastLeaves symbols -- all activation books at eb >= ~3e-4). Steps (ref
// src/huffman.cpp:22-86, 113-125):
//   1. compaction of the touched bins (bitmap written by K3), ascending symbol order
//      == the reference's std::map iteration order; the bins are zeroed on the way;
//   2. bitonic sort of the 64-bit keys (freq << 16 | leaf index): ascending frequency,
//      ties by symbol == the reference heap's (freq, creation index) order for leaves;
//   3. Huffman tree by parallel rounds (see k_codebook_slow, step 3) with S-positions
//      computed by binary search instead of a materialised merge;
//   4. depths by pointer jumping; 5. canonical (length, symbol) order; 6. decode tables.
constexpr int kFastLeaves = 8192;

// Block-wide bottom-up merge sort of n <= kPer * kCbThreads unique u64 keys in shared memory
// (ping-pong between a and b): every element finds its rank in the partner run by a
// fixed-step binary search, the kPer elements of a thread searching together (independent
// chains); one barrier per level. Returns the buffer that holds the sorted keys.
template <int kPer>
__device__ unsigned long long* block_merge_sort(unsigned long long* a, unsigned long long* b,
                                                uint32_t n) {
    const uint32_t tid = threadIdx.x;
    for (uint32_t run = 1; run < n; run <<= 1) {
        unsigned long long v[kPer];
        uint32_t lo[kPer], pe[kPer];
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const uint32_t i = tid + j * kCbThreads;
            v[j] = i < n ? a[i] : 0ull;
            const uint32_t base = i & ~(2 * run - 1);
            const uint32_t pb = (i & run) ? base : base + run;  // partner run
            lo[j] = pb;
            pe[j] = i < n ? min(pb + run, n) : pb;
        }
        for (uint32_t st = run; st > 0; st >>= 1) {
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                const uint32_t q = lo[j] + st - 1;
                if (q < pe[j] && a[q] < v[j]) lo[j] += st;
            }
        }
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const uint32_t i = tid + j * kCbThreads;
            if (i < n) {
                const uint32_t base = i & ~(2 * run - 1);
                const bool second = (i & run) != 0;
                const uint32_t own = i - (second ? base + run : base);
                const uint32_t pb = second ? base : base + run;
                b[base + own + (lo[j] - pb)] = v[j];
            }
        }
        __syncthreads();
        unsigned long long* t = a;
        a = b;
        b = t;
    }
    return a;
}
// phase timing of the fast codebook (debug; acz_gpu_debug_counters slots 8..15):
// compaction, sort, rounds, depths, canonical, tables (SM cycles), round count, calls
// Counted only in development builds (-DACZ_CB_STATS=1): the product build keeps no
// device-global mutable state.
#ifndef ACZ_CB_STATS
#define ACZ_CB_STATS 0
#endif
__device__ unsigned long long g_cbstats[8];
constexpr size_t kFastSmem = kFastLeaves * 8 /*keys*/ + kFastLeaves * 8 /*ifreq*/ +
                             2 * kFastLeaves * 2 /*parent*/ + 2 * kFastLeaves /*depth*/ +
                             kFastLeaves * 4 /*leaf symbols*/;

__device__ __forceinline__ void codebook_fast_body(
    unsigned long long* __restrict__ hist, uint32_t* __restrict__ touched, uint32_t alphabet,
    uint32_t* __restrict__ book_sym, uint8_t* __restrict__ book_len,
    unsigned long long* __restrict__ enc, CanonTables* __restrict__ canon,
    uint32_t* __restrict__ lut, BookInfo* __restrict__ info) {
    extern __shared__ unsigned long long dyn[];
    unsigned long long* key = dyn;                         // [kFastLeaves]
    unsigned long long* ifreq = dyn + kFastLeaves;         // [kFastLeaves]
    uint16_t* par = reinterpret_cast<uint16_t*>(dyn + 2 * kFastLeaves);  // [2*kFastLeaves]
    uint8_t* dep = reinterpret_cast<uint8_t*>(par + 2 * kFastLeaves);    // [2*kFastLeaves]
    __shared__ uint32_t scan_tmp[kCbWarps + 1];
    __shared__ unsigned long long s_first_code[65];
    __shared__ uint32_t s_count[65], s_first_index[65], s_base[65];
    __shared__ uint32_t s_wcnt[kCbWarps][65];
    __shared__ unsigned long long s_total_bits, s_esc;
    __shared__ uint32_t s_max_len, s_flags;
    __shared__ uint32_t sh_li, sh_ii, sh_nl;
    __shared__ unsigned long long sh_fx;
    const int tid = threadIdx.x;
    long long tclk = clock64();
    auto phase = [&](int slot) {
        if (tid == 0) {
            const long long t = clock64();
            if (ACZ_CB_STATS) atomicAdd(&g_cbstats[slot], (unsigned long long)(t - tclk));
            tclk = t;
        }
    };

    uint32_t* lsym = reinterpret_cast<uint32_t*>(dep + 2 * kFastLeaves);  // [kFastLeaves]
    const int lane = tid & 31, warp = tid >> 5;
    // (1) compaction -------------------------------------------------------------------
    // Thread t owns bitmap words [t*wpt, (t+1)*wpt): its touched-bin count, a block scan for
    // its first position (ascending symbol order == the reference's std::map order), then
    // every touched bin is fetched with an asynchronous 8-byte copy into its slot.
    const uint32_t nwords = (alphabet + 31) / 32;
    const uint32_t wpt = (nwords + kCbThreads - 1) / kCbThreads;
    const uint32_t w0 = min(nwords, (uint32_t)tid * wpt), w1 = min(nwords, w0 + wpt);
    uint32_t mine = 0;
    for (uint32_t w = w0; w < w1; ++w) mine += __popc(touched[w]);
    if (tid == 0) {
        s_flags = 0;
        s_total_bits = 0;
        s_max_len = 0;
        s_esc = 0;
    }
    uint32_t k;
    uint32_t pos = block_scan_u32(mine, scan_tmp, &k);
    if (k > kFastLeaves) {
        if (tid == 0) info->slow = 1;  // k_codebook_slow takes over (bins left intact)
        return;
    }
    for (uint32_t w = w0; w < w1; ++w) {
        for (uint32_t m = touched[w]; m; m &= m - 1) {
            const uint32_t sy = w * 32 + (__ffs(m) - 1);
            cp_async8(&key[pos], &hist[sy]);
            lsym[pos] = sy;
            ++pos;
        }
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    for (uint32_t p = tid; p < k; p += kCbThreads) {
        const unsigned long long f = key[p];
        if (lsym[p] == 0) s_esc = f;
        key[p] = (f << 16) | p;
    }
    // self-cleaning: zero the consumed bins and the bitmap (the copies above have landed)
    for (uint32_t w = w0; w < w1; ++w) {
        for (uint32_t m = touched[w]; m; m &= m - 1) hist[w * 32 + (__ffs(m) - 1)] = 0;
        touched[w] = 0;
    }
    __syncthreads();
    phase(0);
    if (k == 0) {
        if (tid == 0) {
            info->book_size = 0;
            info->total_bits = 0;
            info->n_escapes = 0;
            info->max_len = 0;
            info->flags = 0;
            info->slow = 0;
        }
        return;
    }

    // (2) stable LSD radix sort of the keys by frequency, 4-bit digits (keys are
    // freq << 16 | leaf with leaves in ascending symbol order, so a stable sort by frequency
    // gives the (freq, leaf) order). Thread t owns keys [8t, 8t+8); the 16 bucket counters
    // of a thread are packed as 16-bit fields in four u64 (sums <= 8192 never carry across
    // fields) and block-scanned together. The ifreq region is the ping-pong buffer.
    {
        constexpr int PER = kFastLeaves / kCbThreads;
        __shared__ unsigned long long s_wsum[kCbWarps][4];
        __shared__ unsigned long long s_wtot[4];
        __shared__ unsigned long long s_mx;
        unsigned long long mx = 0;
        for (uint32_t p = tid; p < k; p += kCbThreads) mx = max(mx, key[p] >> 16);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (tid == 0) s_mx = 0;
        __syncthreads();
        if (lane == 0) atomicMax(&s_mx, mx);
        __syncthreads();
        const int fbits = 64 - __clzll(s_mx | 1ull);
        const int passes = (fbits + 3) / 4;
        unsigned long long* src = key;
        unsigned long long* dst = ifreq;
        for (int ps = 0; ps < passes; ++ps) {
            const int sh = 16 + 4 * ps;
            unsigned long long kk[PER];
            uint32_t dg[PER];
            unsigned long long c[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const uint32_t idx = (uint32_t)tid * PER + j;
                kk[j] = idx < k ? src[idx] : 0ull;
                dg[j] = (uint32_t)(kk[j] >> sh) & 15u;
                const unsigned long long inc = idx < k ? 1ull << (16 * (dg[j] & 3)) : 0ull;
                const uint32_t q = dg[j] >> 2;
                c[0] += q == 0 ? inc : 0ull;
                c[1] += q == 1 ? inc : 0ull;
                c[2] += q == 2 ? inc : 0ull;
                c[3] += q == 3 ? inc : 0ull;
            }
            // block exclusive scan of the packed counters (thread order == key order)
            unsigned long long x[4] = {c[0], c[1], c[2], c[3]};
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const unsigned long long y = __shfl_up_sync(0xffffffffu, x[q], o);
                    if (lane >= o) x[q] += y;
                }
            }
            if (lane == 31)
#pragma unroll
                for (int q = 0; q < 4; ++q) s_wsum[warp][q] = x[q];
            __syncthreads();
            if (warp == 0) {  // exclusive scan of the 32 warp sums; row kCbWarps = totals
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const unsigned long long v = s_wsum[lane][q];
                    unsigned long long incl = v;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += y;
                    }
                    __syncwarp();
                    s_wsum[lane][q] = incl - v;
                    if (lane == 31) s_wtot[q] = incl;
                }
            }
            __syncthreads();
            unsigned long long wpre[4], tot[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                wpre[q] = s_wsum[warp][q];
                tot[q] = s_wtot[q];
            }
            // bucket bases: exclusive scan of the 16 totals, packed the same way
            unsigned long long base[4] = {0ull, 0ull, 0ull, 0ull};
            {
                unsigned long long run = 0;
#pragma unroll
                for (int d = 0; d < 16; ++d) {
                    base[d >> 2] |= run << (16 * (d & 3));
                    run += (tot[d >> 2] >> (16 * (d & 3))) & 0xFFFFull;
                }
            }
            unsigned long long cur[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) cur[q] = base[q] + wpre[q] + (x[q] - c[q]);
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const uint32_t idx = (uint32_t)tid * PER + j;
                if (idx < k) {
                    const uint32_t q = dg[j] >> 2, f = 16 * (dg[j] & 3);
                    const unsigned long long cq = q == 0 ? cur[0] : q == 1 ? cur[1] : q == 2 ? cur[2] : cur[3];
                    dst[(cq >> f) & 0xFFFFull] = kk[j];
                    const unsigned long long inc = 1ull << f;
                    cur[0] += q == 0 ? inc : 0ull;
                    cur[1] += q == 1 ? inc : 0ull;
                    cur[2] += q == 2 ? inc : 0ull;
                    cur[3] += q == 3 ? inc : 0ull;
                }
            }
            __syncthreads();
            unsigned long long* t = src;
            src = dst;
            dst = t;
        }
        if (src != key) {
            for (uint32_t p = tid; p < k; p += kCbThreads) key[p] = src[p];
            __syncthreads();
        }
    }

    unsigned long long* skey = key;
    unsigned long long* iq = ifreq;  // internal-node frequencies
    phase(1);
    // (3) tree by parallel rounds -------------------------------------------------------
    // node ids: leaf (symbol-order index) j -> j, internal t -> k + t; par[] = parent id.
    // Round: X = the two smallest (leaf wins frequency ties, internals FIFO: the reference
    // heap's (freq, creation index) order, huffman.cpp:42-54); every leaf with freq <= fx
    // and every queued internal (all <= fx) -- the set S -- precede X, and the pairs
    // S[2q], S[2q+1] are the next merges (each >= fx), an odd last element pairing with X.
    // Warp 0 forms X and counts S's leaves (32-way probes); then every thread places one S
    // element by binary search in the other list. Two barriers per round; the internal
    // frequencies accumulate by atomics into a pre-zeroed queue.
    const uint32_t root = k == 1 ? 0 : 2 * k - 2;
    if (k == 1) {
        if (tid == 0) par[0] = 0;
    }
    for (uint32_t i = tid; i < k; i += kCbThreads) iq[i] = 0;
    __syncthreads();
    {
        uint32_t li = 0, ii = 0, m = 0;  // queue state (uniform over the block)
        while (k > 1 && (k - li) + (m - ii) > 1) {
            if (tid < 32) {
                uint32_t l2 = li, i2 = ii;
                unsigned long long fx = 0;
                if (lane == 0) {
                    unsigned long long f2[2];
                    uint32_t id2[2];
                    for (int t = 0; t < 2; ++t) {
                        const unsigned long long fl = l2 < k ? (skey[l2] >> 16) : ~0ull;
                        if (l2 < k && (i2 >= m || fl <= iq[i2])) {  // leaf wins ties
                            f2[t] = fl;
                            id2[t] = (uint32_t)(skey[l2] & 0xFFFF);
                            ++l2;
                        } else {
                            f2[t] = iq[i2];
                            id2[t] = k + i2;
                            ++i2;
                        }
                    }
                    fx = f2[0] + f2[1];
                    if (ACZ_CB_STATS) atomicAdd(&g_cbstats[6], 1ull);
                    iq[m] = fx;
                    par[id2[0]] = (uint16_t)(k + m);
                    par[id2[1]] = (uint16_t)(k + m);
                }
                fx = __shfl_sync(0xffffffffu, fx, 0);
                l2 = __shfl_sync(0xffffffffu, l2, 0);
                i2 = __shfl_sync(0xffffffffu, i2, 0);
                // first leaf in [l2, k) with freq > fx: 32-way probes of strides 1024, 32, 1
                uint32_t lo = l2;
#pragma unroll
                for (int lev = 0; lev < 3; ++lev) {
                    const uint32_t st = lev == 0 ? 1024u : lev == 1 ? 32u : 1u;
                    const uint32_t q = lo + (uint32_t)lane * st + st - 1;  // last of block `lane`
                    const bool le = q < k && (skey[q] >> 16) <= fx;
                    lo += (uint32_t)__popc(__ballot_sync(0xffffffffu, le)) * st;
                }
                if (lane == 0) {
                    sh_li = l2;
                    sh_ii = i2;
                    sh_nl = min(lo, k) - l2;
                    sh_fx = fx;
                }
            }
            __syncthreads();
            const uint32_t l2 = sh_li, i2 = sh_ii, nl = sh_nl, xm = m;
            const unsigned long long fx = sh_fx;
            const uint32_t ni = xm - i2;  // queued internals (all precede X)
            const uint32_t ns = nl + ni, np = ns >> 1, m1 = xm + 1;
            const bool odd = ns & 1;
            for (uint32_t t = tid; t < ns; t += kCbThreads) {
                unsigned long long f;
                uint32_t node, p;
                if (t < nl) {
                    f = skey[l2 + t] >> 16;
                    node = (uint32_t)(skey[l2 + t] & 0xFFFF);
                    uint32_t lo = 0, hi = ni;  // internals with freq < f precede the leaf
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (iq[i2 + mid] < f) lo = mid + 1; else hi = mid;
                    }
                    p = t + lo;
                } else {
                    const uint32_t i = t - nl;
                    f = iq[i2 + i];
                    node = k + i2 + i;
                    uint32_t lo = 0, hi = nl;  // leaves with freq <= f precede the internal
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if ((skey[l2 + mid] >> 16) <= f) lo = mid + 1; else hi = mid;
                    }
                    p = i + lo;
                }
                const uint32_t q = p >> 1;  // p == ns - 1 with odd ns -> q == np (pairs with X)
                par[node] = (uint16_t)(k + m1 + q);
                if (odd && p == ns - 1) {
                    atomicAdd(&iq[m1 + q], f + fx);
                    par[k + xm] = (uint16_t)(k + m1 + q);
                } else {
                    atomicAdd(&iq[m1 + q], f);
                }
            }
            li = l2 + nl;
            ii = odd ? xm + 1 : xm;  // X is consumed, or stays at the queue front
            m = m1 + np + (odd ? 1u : 0u);
            __syncthreads();
        }
    }
    if (tid == 0 && k > 1) par[root] = (uint16_t)root;
    __syncthreads();
    phase(2);

    // (4) code lengths: every leaf walks its parent chain to the root (the kPer leaves of a
    // thread walk together), plus the per-length counts, total bits and the longest code --
    constexpr int kPer = kFastLeaves / kCbThreads;
    if (tid < 65) s_count[tid] = 0;
    __syncthreads();
    unsigned long long bits_part = 0;
    uint32_t maxl = 0;
    bool too_deep = false;
    {
        uint32_t nd[kPer], d[kPer];
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const uint32_t r = tid + j * kCbThreads;  // rank in frequency order
            nd[j] = r < k ? (uint32_t)(skey[r] & 0xFFFF) : root;
            d[j] = 0;
        }
        if (k > 1) {
            for (int it = 0; it < 65; ++it) {
                bool any = false;
#pragma unroll
                for (int j = 0; j < kPer; ++j) {
                    if (nd[j] != root) {
                        nd[j] = par[nd[j]];
                        ++d[j];
                        any = true;
                    }
                }
                if (!any) break;
            }
        }
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const uint32_t r = tid + j * kCbThreads;
            if (r < k) {
                const unsigned long long kk = skey[r];
                uint32_t l = k == 1 ? 1u : d[j];
                if (nd[j] != root || l > 64) {
                    too_deep = true;
                    l = 64;
                }
                dep[kk & 0xFFFF] = (uint8_t)l;
                atomicAdd(&s_count[l], 1u);
                bits_part += (kk >> 16) * l;
                maxl = max(maxl, l);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bits_part += __shfl_xor_sync(0xffffffffu, bits_part, o);
    maxl = __reduce_max_sync(0xffffffffu, maxl);
    if ((tid & 31) == 0) {
        atomicAdd(&s_total_bits, bits_part);
        atomicMax(&s_max_len, maxl);
    }
    if (too_deep) atomicOr(&s_flags, kFlagDepth64);
    phase(3);
    __syncthreads();
    if (tid == 0) {
        unsigned long long code = 0;
        uint32_t prev = 0, idx = 0;
        for (int l = 1; l <= 64; ++l) {
            s_first_index[l] = idx;
            if (s_count[l]) {
                code <<= (l - prev);
                s_first_code[l] = code;
                code += s_count[l];
                prev = l;
                idx += s_count[l];
            } else {
                s_first_code[l] = 0;
            }
        }
        s_first_code[0] = 0;
        s_first_index[0] = 0;
        if (s_max_len > 56) s_flags |= kFlagLenTooLong;
    }
    // (5) canonical order: stable counting sort by length over ascending symbols ---------
    if (tid < 65) s_base[tid] = 0;
    __syncthreads();
    const unsigned lanemask_lt = (1u << lane) - 1;
    uint32_t* s_book = reinterpret_cast<uint32_t*>(key);  // keys are dead from here on
    for (uint32_t base = 0; base < k; base += kCbThreads) {
        const uint32_t i = base + tid;
        const bool valid = i < k;
        const uint32_t l = valid ? min((uint32_t)dep[i], 64u) : 0xFFu;
        const unsigned same = __match_any_sync(0xffffffffu, l);
        const uint32_t rank_w = __popc(same & lanemask_lt);
        for (int j = lane; j < 65; j += 32) s_wcnt[warp][j] = 0;
        __syncwarp();
        if (valid && rank_w == 0) s_wcnt[warp][l] = __popc(same);
        __syncthreads();
        if (tid < 65) {
            uint32_t run = s_base[tid];
            for (int w = 0; w < kCbWarps; ++w) {
                const uint32_t c = s_wcnt[w][tid];
                s_wcnt[w][tid] = run;
                run += c;
            }
            s_base[tid] = run;
        }
        __syncthreads();
        if (valid) {
            const uint32_t rank = s_wcnt[warp][l] + rank_w;
            const uint32_t pos = s_first_index[l] + rank;
            const uint32_t sym = lsym[i];
            book_sym[pos] = sym;
            s_book[pos] = sym;
            book_len[pos] = (uint8_t)l;
            const unsigned long long code = s_first_code[l] + rank;
            enc[sym] = (code << 8) | l;
            // compact form for books with codes <= 27 bits: code | len << 27
            reinterpret_cast<uint32_t*>(enc + alphabet)[sym] =
                l <= 27 ? (uint32_t)code | ((uint32_t)l << 27) : 0u;
        }
        __syncthreads();
    }
    phase(4);
    // (6) decode tables ----------------------------------------------------------------
    write_tables(s_count, s_first_code, s_first_index, s_book, canon, lut);
    __syncthreads();
    phase(5);
    if (tid == 0) {
        if (ACZ_CB_STATS) atomicAdd(&g_cbstats[7], 1ull);
        info->book_size = k;
        info->total_bits = s_total_bits;
        info->n_escapes = s_esc;
        info->max_len = s_max_len;
        info->flags = s_flags;
        info->slow = 0;
    }
}

__global__ void __launch_bounds__(kCbThreads, 1) k_codebook_fast(
    unsigned long long* __restrict__ hist, uint32_t* __restrict__ touched, uint32_t alphabet,
    uint32_t* __restrict__ book_sym, uint8_t* __restrict__ book_len,
    unsigned long long* __restrict__ enc, CanonTables* __restrict__ canon,
    uint32_t* __restrict__ lut, BookInfo* __restrict__ info) {
    codebook_fast_body(hist, touched, alphabet, book_sym, book_len, enc, canon, lut, info);
}

// Slow K4 (books larger than kFastLeaves): global-memory scratch. Runs only when the fast
// kernel flagged info->slow; also cleans the histogram bins and the touched bitmap.
__global__ void __launch_bounds__(kCbThreads, 1) k_codebook_slow(
    unsigned long long* __restrict__ hist, uint32_t* __restrict__ touched, uint32_t alphabet,
    uint64_t max_leaves, void* scratch, uint32_t* __restrict__ book_sym,
    uint8_t* __restrict__ book_len, unsigned long long* __restrict__ enc,
    CanonTables* __restrict__ canon, uint32_t* __restrict__ lut, BookInfo* __restrict__ info) {
    if (!info->slow) return;
    extern __shared__ unsigned long long dyn[];  // radix table / internal FIFO
    __shared__ uint32_t scan_tmp[kCbWarps + 1];
    __shared__ unsigned long long s_first_code[65];
    __shared__ uint32_t s_count[65], s_first_index[65], s_base[65];
    __shared__ uint32_t s_wcnt[kCbWarps][65];
    __shared__ unsigned long long s_total_bits;
    __shared__ uint32_t s_max_len, s_flags;

    const int tid = threadIdx.x;
    CbScratch S = carve(scratch, max_leaves);

    // (1) compaction of non-zero bins, ascending symbol order --------------------------
    uint32_t k = 0;
    for (uint64_t base = 0; base < alphabet; base += kCbThreads) {
        const uint64_t s = base + tid;
        const unsigned long long f = s < alphabet ? hist[s] : 0ull;
        if (f) hist[s] = 0;  // self-cleaning histogram
        uint32_t tot;
        const uint32_t pos = block_scan_u32(f != 0, scan_tmp, &tot);
        if (f != 0 && k + pos < max_leaves) {
            S.leaf_sym[k + pos] = (uint32_t)s;
            S.leaf_freq[k + pos] = f;
        }
        k += tot;
    }
    for (uint32_t w = tid; w < (alphabet + 31) / 32; w += kCbThreads) touched[w] = 0;
    if (tid == 0) {
        s_flags = 0;
        s_total_bits = 0;
        s_max_len = 0;
    }
    __syncthreads();
    if (k == 0 || k > max_leaves) {
        if (tid == 0) {
            info->book_size = k;
            info->total_bits = 0;
            info->n_escapes = alphabet ? hist[0] : 0;
            info->max_len = 0;
            info->flags = k > max_leaves ? kFlagBookTooBig : 0;
            info->slow = 0;
        }
        return;
    }

    // (2) stable LSD radix sort of leaf ids by frequency ------------------------------
    unsigned long long maxf = 0;
    for (uint32_t i = tid; i < k; i += kCbThreads) {
        S.key_a[i] = S.leaf_freq[i];
        S.val_a[i] = i;
        maxf = max(maxf, S.leaf_freq[i]);
    }
    // block max via shared
    {
        __shared__ unsigned long long s_maxf;
        if (tid == 0) s_maxf = 0;
        __syncthreads();
        atomicMax(&s_maxf, maxf);
        __syncthreads();
        maxf = s_maxf;
    }
    const int key_bits = 64 - __clzll(maxf | 1ull);
    const int passes = (key_bits + kRadixBits - 1) / kRadixBits;
    uint32_t* table = reinterpret_cast<uint32_t*>(dyn);  // [kRadixBuckets][kCbThreads]
    unsigned long long *kin = S.key_a, *kout = S.key_b;
    uint32_t *vin = S.val_a, *vout = S.val_b;
    const uint32_t seg = (k + kCbThreads - 1) / kCbThreads;
    const uint32_t lo = min(k, tid * seg), hi = min(k, lo + seg);
    for (int p = 0; p < passes; ++p) {
        const int shift = p * kRadixBits;
        uint32_t cnt[kRadixBuckets];
#pragma unroll
        for (int d = 0; d < kRadixBuckets; ++d) cnt[d] = 0;
        for (uint32_t i = lo; i < hi; ++i) cnt[(kin[i] >> shift) & (kRadixBuckets - 1)]++;
#pragma unroll
        for (int d = 0; d < kRadixBuckets; ++d) table[d * kCbThreads + tid] = cnt[d];
        __syncthreads();
        // exclusive scan over the digit-major table: thread t scans 16 consecutive cells
        uint32_t local[kRadixBuckets];
        uint32_t run = 0;
#pragma unroll
        for (int j = 0; j < kRadixBuckets; ++j) {
            local[j] = table[tid * kRadixBuckets + j];
            run += local[j];
        }
        uint32_t tot;
        uint32_t pre = block_scan_u32(run, scan_tmp, &tot);
#pragma unroll
        for (int j = 0; j < kRadixBuckets; ++j) {
            table[tid * kRadixBuckets + j] = pre;
            pre += local[j];
        }
        __syncthreads();
#pragma unroll
        for (int d = 0; d < kRadixBuckets; ++d) cnt[d] = table[d * kCbThreads + tid];
        for (uint32_t i = lo; i < hi; ++i) {
            const int d = (kin[i] >> shift) & (kRadixBuckets - 1);
            const uint32_t o = cnt[d]++;
            kout[o] = kin[i];
            vout[o] = vin[i];
        }
        __syncthreads();
        unsigned long long* tk = kin;
        kin = kout;
        kout = tk;
        uint32_t* tv = vin;
        vin = vout;
        vout = tv;
        __threadfence_block();
        __syncthreads();
    }
    // sorted: kin (freq), vin (leaf id)

    // (3) Huffman tree by parallel rounds ----------------------------------------------
    //     Equivalent to the two-queue merge (leaf wins frequency ties, internals FIFO),
    //     itself equivalent to the reference heap order (ref src/huffman.cpp:42-54).
    //     A round pops the two smallest items a, b -> internal X; every pending item with
    //     key < key(X) (all queued internals, leaves with freq <= f(X)) is popped before X,
    //     in merged order, pairwise -> new internals Y_j (all > X); an odd leftover pairs
    //     with X. ~20 rounds for activation histograms instead of k-1 serial merges.
    //     node ids: leaf j -> j, internal t -> k + t; S.anc_a[] receives parents.
    const uint32_t root = k == 1 ? 0 : 2 * k - 2;
    {
        __shared__ uint32_t sh_li, sh_ii, sh_m, sh_nl, sh_ni, sh_xm, sh_done;
        unsigned long long* If = S.ifreq;               // internal freqs, creation order
        unsigned long long* Sf = kout;                  // merged S (freq)
        uint32_t* Sid = vout;                           // merged S (node id)
        if (tid == 0) {
            sh_li = 0;
            sh_ii = 0;
            sh_m = 0;
            sh_done = 0;
            if (k == 1) S.anc_a[0] = 0;
        }
        __syncthreads();
        while (k > 1) {
            if (tid == 0) {
                uint32_t li = sh_li, ii = sh_ii, m = sh_m;
                if ((k - li) + (m - ii) <= 1) {
                    sh_done = 1;
                } else {
                    unsigned long long f2[2];
                    uint32_t id2[2];
                    for (int t = 0; t < 2; ++t) {
                        if (li < k && (ii >= m || kin[li] <= If[ii])) {
                            f2[t] = kin[li];
                            id2[t] = vin[li++];
                        } else {
                            f2[t] = If[ii];
                            id2[t] = k + ii++;
                        }
                    }
                    const unsigned long long fx = f2[0] + f2[1];
                    If[m] = fx;
                    S.anc_a[id2[0]] = k + m;
                    S.anc_a[id2[1]] = k + m;
                    // leaves with freq <= fx
                    uint32_t lo = li, hi = k;
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (kin[mid] <= fx) lo = mid + 1; else hi = mid;
                    }
                    sh_nl = lo - li;
                    sh_ni = m - ii;
                    sh_xm = m;
                    sh_li = li;
                    sh_ii = ii;
                    sh_m = m + 1;
                }
            }
            __syncthreads();
            if (sh_done) break;
            const uint32_t li = sh_li, ii = sh_ii, nl = sh_nl, ni = sh_ni, xm = sh_xm;
            const uint32_t ns = nl + ni;
            const unsigned long long* A = kin + li;
            const uint32_t* Aid = vin + li;
            const unsigned long long* Bf = If + ii;
            // merge path: thread t writes outputs [d0, d1)
            const uint32_t per = (ns + kCbThreads - 1) / kCbThreads;
            const uint32_t d0 = min(ns, tid * per), d1 = min(ns, d0 + per);
            if (d0 < d1) {
                uint32_t lo = d0 > ni ? d0 - ni : 0, hi = min(d0, nl);
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (A[mid] <= Bf[d0 - mid - 1]) lo = mid + 1; else hi = mid;
                }
                uint32_t ia = lo, ib = d0 - lo;
                for (uint32_t d = d0; d < d1; ++d) {
                    if (ia < nl && (ib >= ni || A[ia] <= Bf[ib])) {
                        Sf[d] = A[ia];
                        Sid[d] = Aid[ia];
                        ++ia;
                    } else {
                        Sf[d] = Bf[ib];
                        Sid[d] = k + ii + ib;
                        ++ib;
                    }
                }
            }
            __syncthreads();
            const uint32_t m1 = xm + 1;  // first id slot after X
            const uint32_t np = ns >> 1;
            for (uint32_t q = tid; q < np; q += kCbThreads) {
                If[m1 + q] = Sf[2 * q] + Sf[2 * q + 1];
                S.anc_a[Sid[2 * q]] = k + m1 + q;
                S.anc_a[Sid[2 * q + 1]] = k + m1 + q;
            }
            __syncthreads();
            if (tid == 0) {
                uint32_t m = m1 + np;
                uint32_t iin = xm;  // X becomes the queue front
                if (ns & 1) {
                    // leftover pairs with X
                    If[m] = Sf[ns - 1] + If[xm];
                    S.anc_a[Sid[ns - 1]] = k + m;
                    S.anc_a[k + xm] = k + m;
                    ++m;
                    iin = xm + 1;
                }
                sh_li = li + nl;
                sh_ii = iin;
                sh_m = m;
            }
            __syncthreads();
        }
        if (tid == 0 && k > 1) S.anc_a[root] = root;
    }
    __syncthreads();

    // (4) depths by pointer jumping over 2k-1 nodes -------------------------------------
    const uint32_t nodes = k == 1 ? 1 : 2 * k - 1;
    uint32_t *ain = S.anc_a, *aout = S.anc_b, *din = S.dist_a, *dout = S.dist_b;
    for (uint32_t i = tid; i < nodes; i += kCbThreads) din[i] = (k == 1) ? 1 : (i == root ? 0 : 1);
    __syncthreads();
    if (k > 1) {
        for (int it = 0; it < 40; ++it) {
            int changed = 0;
            for (uint32_t i = tid; i < nodes; i += kCbThreads) {
                const uint32_t a = ain[i];
                if (a != root) {
                    dout[i] = din[i] + din[a];
                    aout[i] = ain[a];
                    changed = 1;
                } else {
                    dout[i] = din[i];
                    aout[i] = a;
                }
            }
            const int any = __syncthreads_or(changed);
            uint32_t* t = ain;
            ain = aout;
            aout = t;
            t = din;
            din = dout;
            dout = t;
            if (!any) break;
        }
    }
    // leaf j length = din[j]

    // (5) canonical order: stable counting sort by length over ascending symbols --------
    if (tid < 65) {
        s_count[tid] = 0;
        s_base[tid] = 0;
    }
    __syncthreads();
    unsigned long long bits_part = 0;
    uint32_t maxl = 0;
    bool too_deep = false;
    for (uint32_t i = tid; i < k; i += kCbThreads) {
        uint32_t l = din[i];
        if (l > 64) {
            too_deep = true;
            l = 64;
        }
        atomicAdd(&s_count[l], 1u);
        bits_part += S.leaf_freq[i] * l;
        maxl = max(maxl, l);
    }
    atomicAdd(&s_total_bits, bits_part);
    atomicMax(&s_max_len, maxl);
    if (too_deep) atomicOr(&s_flags, kFlagDepth64);
    __syncthreads();
    if (tid == 0) {
        unsigned long long code = 0;
        uint32_t prev = 0, idx = 0;
        for (int l = 1; l <= 64; ++l) {
            s_first_index[l] = idx;
            if (s_count[l]) {
                code <<= (l - prev);
                s_first_code[l] = code;
                code += s_count[l];
                prev = l;
                idx += s_count[l];
            } else {
                s_first_code[l] = 0;
            }
        }
        s_first_code[0] = 0;
        s_first_index[0] = 0;
        if (s_max_len > 56) s_flags |= kFlagLenTooLong;
    }
    __syncthreads();
    const int lane = tid & 31, warp = tid >> 5;
    const unsigned lanemask_lt = (1u << lane) - 1;
    for (uint32_t base = 0; base < k; base += kCbThreads) {
        const uint32_t i = base + tid;
        const bool valid = i < k;
        const uint32_t l = valid ? min(din[i], 64u) : 0xFFu;
        const unsigned same = __match_any_sync(0xffffffffu, l);
        const uint32_t rank_w = __popc(same & lanemask_lt);
        for (int j = lane; j < 65; j += 32) s_wcnt[warp][j] = 0;
        __syncwarp();
        if (valid && rank_w == 0) s_wcnt[warp][l] = __popc(same);
        __syncthreads();
        // prefix over warps per length (thread t < 65 handles length t)
        if (tid < 65) {
            uint32_t run = s_base[tid];
            for (int w = 0; w < kCbWarps; ++w) {
                const uint32_t c = s_wcnt[w][tid];
                s_wcnt[w][tid] = run;
                run += c;
            }
            s_base[tid] = run;
        }
        __syncthreads();
        if (valid) {
            const uint32_t rank = s_wcnt[warp][l] + rank_w;
            const uint32_t pos = s_first_index[l] + rank;
            const uint32_t sym = S.leaf_sym[i];
            book_sym[pos] = sym;
            book_len[pos] = (uint8_t)l;
            const unsigned long long code = s_first_code[l] + rank;
            enc[sym] = (code << 8) | l;
            // compact form for books with codes <= 27 bits: code | len << 27
            reinterpret_cast<uint32_t*>(enc + alphabet)[sym] =
                l <= 27 ? (uint32_t)code | ((uint32_t)l << 27) : 0u;
        }
        __syncthreads();
    }
    // (6) decode tables ----------------------------------------------------------------
    __syncthreads();
    write_tables(s_count, s_first_code, s_first_index, book_sym, canon, lut);
    if (tid == 0) {
        info->book_size = k;
        info->total_bits = s_total_bits;
        info->n_escapes = S.leaf_sym[0] == 0 ? S.leaf_freq[0] : 0;
        info->max_len = s_max_len;
        info->flags = s_flags | (k > kMaxBook ? kFlagBookTooBig : 0);
        info->slow = 0;
    }
}

// Builds the LUT + canonical tables for an existing canonical book (foreign blobs).
__global__ void __launch_bounds__(1024) k_build_tables(const uint32_t* __restrict__ book_sym,
                                                       const uint8_t* __restrict__ book_len,
                                                       uint32_t book_size,
                                                       CanonTables* __restrict__ canon,
                                                       uint32_t* __restrict__ lut,
                                                       unsigned int* flags) {
    __shared__ unsigned long long s_first_code[65];
    __shared__ uint32_t s_count[65], s_first_index[65];
    const int tid = threadIdx.x;
    if (tid < 65) s_count[tid] = 0;
    __syncthreads();
    for (uint32_t i = tid; i < book_size; i += blockDim.x) atomicAdd(&s_count[book_len[i]], 1u);
    __syncthreads();
    if (tid == 0) {
        // canonical order was validated on the host; codes follow ref huffman.cpp:75-86
        unsigned long long code = 0;
        uint32_t prev = 0, idx = 0;
        for (int l = 1; l <= 64; ++l) {
            s_first_index[l] = idx;
            s_first_code[l] = 0;
            if (s_count[l]) {
                code <<= (l - prev);
                s_first_code[l] = code;
                code += s_count[l];
                prev = l;
                idx += s_count[l];
            }
        }
        s_first_code[0] = 0;
        s_first_index[0] = 0;
    }
    __syncthreads();
    write_tables(s_count, s_first_code, s_first_index, book_sym, canon, lut);
    (void)flags;
}

// --------------------------------------------------------------------------- K5 ----
// Block-wide exclusive scan of two u32 per thread (kEncThreads threads). Returns the
// exclusive prefixes; *ta / *tb receive the block totals.
template <int NT>
__device__ __forceinline__ void block_scan2(uint32_t a, uint32_t b, uint32_t* ea, uint32_t* eb,
                                            uint32_t* ta, uint32_t* tb, uint32_t* sa,
                                            uint32_t* sb) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int W = NT / 32;
    uint32_t ia = a, ib = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t xa = __shfl_up_sync(0xffffffffu, ia, o);
        const uint32_t xb = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) {
            ia += xa;
            ib += xb;
        }
    }
    if (lane == 31) {
        sa[warp] = ia;
        sb[warp] = ib;
    }
    __syncthreads();
    uint32_t pa = 0, pb = 0, qa = 0, qb = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
        const uint32_t va = sa[w], vb = sb[w];
        if (w < warp) {
            pa += va;
            pb += vb;
        }
        qa += va;
        qb += vb;
    }
    *ea = pa + ia - a;
    *eb = pb + ib - b;
    *ta = qa;
    *tb = qb;
    __syncthreads();
}

// K5 encode (ref src/huffman.cpp:127-131 + BitWriter :88-103), two kernels over 256-symbol
// chunks (one warp, 8 symbols per lane):
//  K5a k_encode_count (persistent, CTA c owns a contiguous span of chunks): per-chunk bit and
//      escape counts, one decoupled look-back across CTAs for the span's global offsets, a
//      CTA scan turning the span's counts into absolute per-chunk offsets, and zeroing of the
//      words two chunks share (so no memset of the bitstream is needed).
//  K5b k_encode_write (one warp per chunk, no CTA-wide synchronisation): codes in registers,
//      warp scan of the lengths, MSB-first packing with a 64-bit accumulator into a per-warp
//      shared stage (OR only where two lanes share a word), coalesced word stores (the two
//      chunk-boundary words OR-ed), the outlier list and the decode sidecar.
constexpr int kChunk = 32 * kEncPer;  // symbols per chunk

// kLast: the second (last) read of the symbols, streamed (evict-first); the counting pass
// keeps them in L2 for it.
template <typename SymT, bool kLast>
__device__ __forceinline__ void load_chunk_syms(const SymT* __restrict__ symp, uint64_t n,
                                                uint64_t my0, bool vec_ok, uint32_t* sy) {
    if (vec_ok && my0 + kEncPer <= n) {
        const uint4* v4 = reinterpret_cast<const uint4*>(symp + my0);
        constexpr int per16 = 16 / (int)sizeof(SymT);
#pragma unroll
        for (int q = 0; q < kEncPer / per16; ++q) {
            const uint4 v = kLast ? __ldcs(v4 + q) : __ldg(v4 + q);
            const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (sizeof(SymT) == 2) {
                    sy[q * 8 + 2 * k] = w4[k] & 0xFFFFu;
                    sy[q * 8 + 2 * k + 1] = w4[k] >> 16;
                } else {
                    sy[q * 4 + k] = w4[k];
                }
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < kEncPer; ++i) sy[i] = my0 + i < n ? (uint32_t)symp[my0 + i] : 0u;
    }
}

constexpr int kCountThreads = 1024;  // counting CTAs of 1024 threads, ACZ_ENC_COUNT_CTAS per SM
#ifndef ACZ_ENC_COUNT_CTAS
#define ACZ_ENC_COUNT_CTAS 1
#endif

// code length of symbol v: the compact table when every code is <= 27 bits
template <bool kCompact>
__device__ __forceinline__ uint32_t code_len(const EncodeArgs& a, uint32_t v) {
    return kCompact ? __ldg(a.enc32 + v) >> 27 : (uint32_t)(__ldg(a.enc + v) & 0xFF);
}

template <typename SymT, bool kCompact>
__global__ void __launch_bounds__(kCountThreads) k_encode_count(EncodeArgs a) {
    const SymT* __restrict__ symp = static_cast<const SymT*>(a.sym);
    __shared__ uint32_t s_a[kCountThreads / 32], s_b[kCountThreads / 32];
    __shared__ unsigned long long s_red_bits[kCountThreads / 32], s_red_esc[kCountThreads / 32];
    __shared__ unsigned long long s_base_bits, s_base_esc;
    constexpr int W = kCountThreads / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t chunks = (a.n + kChunk - 1) / kChunk;
    const uint64_t span = (chunks + gridDim.x - 1) / gridDim.x;
    const uint64_t cb = (uint64_t)blockIdx.x * span, ce = min(chunks, cb + span);
    const bool vec_ok = (reinterpret_cast<uintptr_t>(symp) & 15) == 0;
    unsigned long long* coff = a.chunk_off;
    uint64_t nwords_dev = a.nwords;
    if (!encode_spec_ok(a, &nwords_dev)) return;  // speculative launch, book does not fit

    // ---- per-chunk counts (two chunks in flight per warp) -----------------------------
    unsigned long long wb = 0, we = 0;
    // the next pair of chunks is loaded while the current pair is counted (four chunks in
    // flight per warp: the loads, not the counting, bound this pass)
    uint32_t sy[kEncPer], sy2[kEncPer];
    {
        const uint64_t c = cb + warp;
        if (c < ce) load_chunk_syms<SymT, false>(symp, a.n, c * kChunk + (uint64_t)lane * kEncPer, vec_ok, sy);
        if (c + W < ce)
            load_chunk_syms<SymT, false>(symp, a.n, (c + W) * kChunk + (uint64_t)lane * kEncPer, vec_ok, sy2);
    }
    // Code lengths of the symbols around the centre, staged as bytes (while the first chunks
    // load): a warp's 32 lookups are then shared-memory reads instead of an L1 gather over
    // ~30 sectors (ncu: 29 sectors per request on AlexNet conv1).
    __shared__ uint32_t s_len4[kEncLenWindow / 4 + 1];
    const uint8_t* s_len = reinterpret_cast<const uint8_t*>(s_len4);
    for (uint32_t i = tid; i < (a.len_n + 3) / 4; i += kCountThreads) {
        uint32_t packed = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const uint32_t o = 4 * i + b;
            if (o < a.len_n) packed |= code_len<kCompact>(a, a.len_lo + o) << (8 * b);
        }
        s_len4[i] = packed;
    }
    __syncthreads();
    auto len_of = [&](uint32_t v) -> uint32_t {
        const uint32_t o = v - a.len_lo;
        return o < a.len_n ? (uint32_t)s_len[o] : code_len<kCompact>(a, v);
    };
    for (uint64_t c = cb + warp; c < ce; c += 2 * W) {
        const uint64_t c2 = c + W;
        uint32_t nx[kEncPer], nx2[kEncPer];
        const uint64_t cn = c + 2 * W;
        if (cn < ce)
            load_chunk_syms<SymT, false>(symp, a.n, cn * kChunk + (uint64_t)lane * kEncPer, vec_ok, nx);
        if (cn + W < ce)
            load_chunk_syms<SymT, false>(symp, a.n, (cn + W) * kChunk + (uint64_t)lane * kEncPer, vec_ok, nx2);
        uint32_t b1 = 0, e1 = 0, b2 = 0, e2 = 0;
        if (c2 < ce && (c2 + 1) * kChunk <= a.n) {
            // both chunks whole (every pair but the span's and the tensor's last): no bounds
#pragma unroll
            for (int i = 0; i < kEncPer; ++i) {
                b1 += len_of(sy[i]);
                e1 += sy[i] == 0;
                b2 += len_of(sy2[i]);
                e2 += sy2[i] == 0;
            }
        } else {
#pragma unroll
            for (int i = 0; i < kEncPer; ++i) {
                if (c * kChunk + (uint64_t)lane * kEncPer + i < a.n) {
                    b1 += len_of(sy[i]);
                    e1 += sy[i] == 0;
                }
                if (c2 < ce && c2 * kChunk + (uint64_t)lane * kEncPer + i < a.n) {
                    b2 += len_of(sy2[i]);
                    e2 += sy2[i] == 0;
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            b1 += __shfl_xor_sync(0xffffffffu, b1, o);
            e1 += __shfl_xor_sync(0xffffffffu, e1, o);
            b2 += __shfl_xor_sync(0xffffffffu, b2, o);
            e2 += __shfl_xor_sync(0xffffffffu, e2, o);
        }
        if (lane == 0) {
            coff[2 * c] = b1;
            coff[2 * c + 1] = e1;
            if (c2 < ce) {
                coff[2 * c2] = b2;
                coff[2 * c2 + 1] = e2;
            }
        }
        wb += b1 + (c2 < ce ? b2 : 0u);
        we += e1 + (c2 < ce ? e2 : 0u);
#pragma unroll
        for (int i = 0; i < kEncPer; ++i) {
            sy[i] = nx[i];
            sy2[i] = nx2[i];
        }
    }
    if (lane == 0) {
        s_red_bits[warp] = wb;
        s_red_esc[warp] = we;
    }
    __syncthreads();

    // ---- span offsets: decoupled look-back over the CTAs (warp 0) ----------------------
    if (warp == 0) {
        unsigned long long rb = lane < W ? s_red_bits[lane] : 0ull;
        unsigned long long re = lane < W ? s_red_esc[lane] : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            rb += __shfl_xor_sync(0xffffffffu, rb, o);
            re += __shfl_xor_sync(0xffffffffu, re, o);
        }
        const uint32_t c = blockIdx.x;
        TileStatus* st = a.status;
        volatile TileStatus* vst = st;
        unsigned long long pb = 0, pe = 0;
        if (lane == 0) {
            st[c].agg_bits = rb;
            st[c].agg_esc = re;
            if (c == 0) {
                st[c].incl_bits = rb;
                st[c].incl_esc = re;
            }
            __threadfence();
            atomicExch(&st[c].flag, c == 0 ? 2u : 1u);
        }
        if (c > 0) {
            int64_t base = (int64_t)c - 1;
            for (;;) {
                const int64_t j = base - lane;
                unsigned f = 2;
                unsigned long long vb = 0, ve = 0;
                if (j >= 0) {
                    unsigned long long spins = 0;
                    do {
                        f = vst[j].flag;
                    } while (f == 0 && ++spins < (1ull << 30));
                    if (f == 0 && a.sticky) {
                        // the predecessor never published: the offsets below would be wrong.
                        // Report it (the host checks the sticky word at every entry point)
                        atomicOr(a.sticky, kFlagInternal);
                        __threadfence_system();
                    }
                    __threadfence();
                    if (f == 2) {
                        vb = vst[j].incl_bits;
                        ve = vst[j].incl_esc;
                    } else {
                        vb = vst[j].agg_bits;
                        ve = vst[j].agg_esc;
                    }
                }
                const unsigned incl = __ballot_sync(0xffffffffu, f == 2);
                const int stop = incl ? __ffs(incl) - 1 : 31;  // nearest inclusive predecessor
                if (lane > stop) {
                    vb = 0;
                    ve = 0;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    vb += __shfl_xor_sync(0xffffffffu, vb, o);
                    ve += __shfl_xor_sync(0xffffffffu, ve, o);
                }
                pb += vb;
                pe += ve;
                if (incl) break;
                base -= 32;
            }
            if (lane == 0) {
                st[c].incl_bits = pb + rb;
                st[c].incl_esc = pe + re;
                __threadfence();
                atomicExch(&st[c].flag, 2u);
            }
        }
        if (lane == 0) {
            s_base_bits = pb;
            s_base_esc = pe;
        }
    }
    __syncthreads();

    // ---- absolute chunk offsets (CTA scan of the span's counts) ------------------------
    unsigned long long run_b = s_base_bits, run_e = s_base_esc;
    for (uint64_t c0 = cb; c0 < ce; c0 += kCountThreads) {
        const uint64_t c = c0 + tid;
        const uint32_t vb = c < ce ? (uint32_t)coff[2 * c] : 0u;
        const uint32_t ve = c < ce ? (uint32_t)coff[2 * c + 1] : 0u;
        uint32_t xb, xe, tb, te;
        block_scan2<kCountThreads>(vb, ve, &xb, &xe, &tb, &te, s_a, s_b);
        if (c < ce) {
            const unsigned long long off = run_b + xb;
            coff[2 * c] = off;
            coff[2 * c + 1] = run_e + xe;
            // a word shared with the previous chunk: zeroed here, OR-ed by both writers
            if ((off & 31) && c > 0) a.words[off >> 5] = 0u;
        }
        run_b += tb;
        run_e += te;
    }
    if (blockIdx.x == gridDim.x - 1) {
        // the stream's last partial word and the decoder's read-ahead padding
        const unsigned long long total = run_b;
        const uint64_t w0 = total >> 5;
        for (uint64_t w = w0 + tid; w < nwords_dev + 32; w += kCountThreads) a.words[w] = 0u;
    }
}

// kMode 0: every code <= 27 bits (compact u32 table); 1: <= 32 bits; 2: longer codes
// (appended in two pieces).
template <typename SymT, int kMode>
__global__ void __launch_bounds__(kEncThreads) k_encode_write(EncodeArgs a, uint32_t stage_words) {
    const SymT* __restrict__ symp = static_cast<const SymT*>(a.sym);
    extern __shared__ uint32_t stage_all[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* stage = stage_all + warp * stage_words;
    const uint64_t chunks = (a.n + kChunk - 1) / kChunk;
    const bool vec_ok = (reinterpret_cast<uintptr_t>(symp) & 15) == 0;
    {
        uint64_t nw;
        if (!encode_spec_ok(a, &nw)) return;  // speculative launch, book does not fit
    }
    // PrevValue sidecar intervals are powers of two >= kEncPer: at most one sidecar point per
    // lane, at its first symbol; other intervals (Lorenzo2d: the plane size) take the general
    // per-symbol path
    const bool ipow2 = (a.interval & (a.interval - 1)) == 0;
    const bool side_fast = ipow2 && a.interval >= (uint64_t)kEncPer;
    const uint64_t imask = a.interval - 1;
    const int ishift = __ffsll((long long)a.interval) - 1;
    for (uint64_t c = blockIdx.x * (uint64_t)(kEncThreads / 32) + warp; c < chunks;
         c += (uint64_t)gridDim.x * (kEncThreads / 32)) {
        const uint64_t my0 = c * kChunk + (uint64_t)lane * kEncPer;
        const int cnt = my0 >= a.n ? 0 : (a.n - my0 >= (uint64_t)kEncPer ? kEncPer : (int)(a.n - my0));
        uint32_t sy[kEncPer];
        load_chunk_syms<SymT, true>(symp, a.n, my0, vec_ok, sy);
        const unsigned long long cbit = a.chunk_off[2 * c];
        const unsigned long long cesc = a.chunk_off[2 * c + 1];
        // mode 0: the compact entry (code | len << 27, upper half zero); else (code << 8) | len
        unsigned long long code[kEncPer];
        auto clen = [&](int i) -> uint32_t {
            return kMode == 0 ? (uint32_t)code[i] >> 27 : (uint32_t)(code[i] & 0xFF);
        };
        auto cval = [&](int i) -> unsigned long long {
            return kMode == 0 ? (unsigned long long)((uint32_t)code[i] & 0x7FFFFFFu) : code[i] >> 8;
        };
        uint32_t my_bits = 0, escmask = 0;
#pragma unroll
        for (int i = 0; i < kEncPer; ++i) {
            if (kMode == 0) {
                code[i] = i < cnt ? __ldg(a.enc32 + sy[i]) : 0u;
            } else {
                code[i] = i < cnt ? __ldg(a.enc + sy[i]) : 0ull;
            }
            my_bits += clen(i);
            if (i < cnt && sy[i] == 0) escmask |= 1u << i;
        }
        const uint32_t my_esc = __popc(escmask);
        uint32_t ib = my_bits, ie = my_esc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t xb = __shfl_up_sync(0xffffffffu, ib, o);
            const uint32_t xe = __shfl_up_sync(0xffffffffu, ie, o);
            if (lane >= o) {
                ib += xb;
                ie += xe;
            }
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, ib, 31);
        const uint32_t ex_bits = ib - my_bits, ex_esc = ie - my_esc;
        const uint32_t s0 = (uint32_t)(cbit & 31);
        const uint32_t nw = (s0 + tot + 31) / 32;
        for (uint32_t i = lane; i < nw + 1; i += 32) stage[i] = 0;
        __syncwarp();
        // sidecar points and outliers (rare per symbol)
        if (a.side_bitoff && cnt) {
            if (side_fast) {
                if ((my0 & imask) == 0) {
                    const uint64_t si = my0 >> ishift;
                    a.side_bitoff[si] = cbit + ex_bits;
                    if (a.side_outl) a.side_outl[si] = (uint32_t)(cesc + ex_esc);
                }
            } else {
                uint32_t lb = 0, le = 0;
#pragma unroll
                for (int i = 0; i < kEncPer; ++i) {  // static indices: code[] stays in registers
                    if (i >= cnt) break;
                    const uint64_t g = my0 + i;
                    if ((ipow2 ? (g & imask) : g % a.interval) == 0) {
                        const uint64_t si = ipow2 ? (g >> ishift) : g / a.interval;
                        a.side_bitoff[si] = cbit + ex_bits + lb;
                        if (a.side_outl) a.side_outl[si] = (uint32_t)(cesc + ex_esc + le);
                    }
                    lb += clen(i);
                    le += (escmask >> i) & 1u;
                }
            }
        }
        if (escmask && a.x) {
            unsigned long long gesc = cesc + ex_esc;
            for (uint32_t m = escmask; m; m &= m - 1) {
                const int i = __ffs(m) - 1;
                a.out_index[gesc] = my0 + i;
                a.out_value[gesc] = a.x[my0 + i];
                ++gesc;
            }
        }
        // MSB-first packing: 64-bit accumulator, whole words stored, the lane's first word
        // (shared with the previous lane) and its trailing partial word OR-ed
        const uint32_t off = s0 + ex_bits;
        unsigned long long acc = 0;
        int nacc = (int)(off & 31);
        uint32_t wi = off >> 5;
        const uint32_t w_first = wi;
        auto emit = [&]() {
            const uint32_t word = (uint32_t)(acc >> 32);
            if (wi == w_first) {
                if (word) atomicOr(&stage[wi], word);
            } else {
                stage[wi] = word;
            }
            ++wi;
            acc <<= 32;
            nacc -= 32;
        };
#pragma unroll
        for (int i = 0; i < kEncPer; ++i) {
            const int len = (int)clen(i);
            if (kMode == 2 && len > 32) {
                const unsigned long long cv = code[i] >> 8;
                acc |= (cv >> 32) << (64 - nacc - (len - 32));
                nacc += len - 32;
                if (nacc >= 32) emit();
                acc |= (cv & 0xFFFFFFFFull) << (32 - nacc);
                nacc += 32;
                emit();
            } else {
                acc |= cval(i) << (64 - nacc - len);
                nacc += len;
                if (nacc >= 32) emit();
            }
        }
        if (nacc > 0) {
            const uint32_t word = (uint32_t)(acc >> 32);
            if (word) atomicOr(&stage[wi], word);
        }
        __syncwarp();
        const uint64_t gw0 = cbit >> 5;
        for (uint32_t i = lane; i < nw; i += 32) {
            const uint64_t gw = gw0 + i;
            const uint32_t v = bswap32(stage[i]);
            if ((i == 0 && s0) || (i == nw - 1 && ((s0 + tot) & 31))) {
                if (v) atomicOr(&a.words[gw], v);
            } else {
                a.words[gw] = v;
            }
        }
        __syncwarp();
    }
}

}  // namespace

cudaError_t launch_histogram(const void* sym, int sym16, uint64_t n, uint32_t alphabet,
                             uint32_t center, unsigned long long* hist, uint32_t* touched,
                             const CbArgs& cb, int sms, cudaStream_t s, uint64_t* launches) {
    const uint32_t win_lo = center > kHistWindow / 2 ? ((center - kHistWindow / 2) & ~31u) : 0u;
    const uint32_t win_n =
        alphabet - win_lo < (uint32_t)kHistWindow ? alphabet - win_lo : (uint32_t)kHistWindow;
    uint64_t blocks = (n / 4 + kHistThreads - 1) / kHistThreads;
#ifndef ACZ_HIST_BPS
#define ACZ_HIST_BPS 1  // blocks per SM (the window takes 128 KB of shared memory)
#endif
    const uint64_t cap = (uint64_t)sms * ACZ_HIST_BPS;
    if (blocks > cap) blocks = cap;
    if (blocks == 0) blocks = 1;
    const size_t smem = cb.done ? std::max<size_t>(4ull * kHistWindow, kFastSmem)
                                : 4ull * kHistWindow;
    static bool attr = false;
    if (!attr) {
        for (const void* f : {(const void*)k_histogram<uint16_t>, (const void*)k_histogram<uint32_t>}) {
            cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)std::max<size_t>(4ull * kHistWindow, kFastSmem));
            if (e != cudaSuccess) return e;
        }
        attr = true;
    }
    if (sym16)
        k_histogram<uint16_t><<<(unsigned)blocks, kHistThreads, smem, s>>>(
            static_cast<const uint16_t*>(sym), n, alphabet, win_lo, win_n, center, hist, touched, cb);
    else
        k_histogram<uint32_t><<<(unsigned)blocks, kHistThreads, smem, s>>>(
            static_cast<const uint32_t*>(sym), n, alphabet, win_lo, win_n, center, hist, touched, cb);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t codebook_stats(unsigned long long* out, bool reset) {
    cudaError_t e = cudaMemcpyFromSymbol(out, g_cbstats, sizeof(g_cbstats));
    if (e == cudaSuccess && reset) {
        unsigned long long z[8] = {0};
        e = cudaMemcpyToSymbol(g_cbstats, z, sizeof(z));
    }
    return e;
}

size_t codebook_scratch_bytes(uint64_t k) {
    return align256(4 * k) + 5 * align256(8 * k) + 2 * align256(4 * k) + 4 * align256(8 * k) +
           4096;
}

cudaError_t launch_codebook(unsigned long long* hist, uint32_t* touched, uint32_t alphabet,
                            uint64_t max_leaves, void* scratch, uint32_t* book_sym,
                            uint8_t* book_len, unsigned long long* enc, CanonTables* canon,
                            uint32_t* lut, BookInfo* info, bool slow_only, cudaStream_t s,
                            uint64_t* launches) {
    const size_t smem_slow = kSmemQueue * sizeof(unsigned long long);  // 128 KiB (>= radix table)
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_codebook_slow,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem_slow);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(k_codebook_fast, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kFastSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    if (!slow_only) {
        k_codebook_fast<<<1, kCbThreads, kFastSmem, s>>>(hist, touched, alphabet, book_sym,
                                                         book_len, enc, canon, lut, info);
        ++*launches;
    }
    if (max_leaves > (uint64_t)kFastLeaves) {
        k_codebook_slow<<<1, kCbThreads, smem_slow, s>>>(hist, touched, alphabet, max_leaves,
                                                         scratch, book_sym, book_len, enc, canon,
                                                         lut, info);
        ++*launches;
    }
    return cudaGetLastError();
}

cudaError_t launch_build_tables(const uint32_t* book_sym, const uint8_t* book_len,
                                uint32_t book_size, CanonTables* canon, uint32_t* lut,
                                unsigned int* flags, cudaStream_t s, uint64_t* launches) {
    k_build_tables<<<1, 1024, 0, s>>>(book_sym, book_len, book_size, canon, lut, flags);
    ++*launches;
    return cudaGetLastError();
}

size_t encode_scratch_bytes(uint64_t n, int sms) {
    const uint64_t chunks = (n + kChunk - 1) / kChunk;
    return align256(sizeof(TileStatus) * (uint64_t)sms * ACZ_ENC_COUNT_CTAS) + 16 * chunks + 256;
}

cudaError_t launch_encode(const EncodeArgs& a0, int sms, cudaStream_t s, uint64_t* launches) {
    EncodeArgs a = a0;
    const uint64_t chunks = (a.n + kChunk - 1) / kChunk;
    uint64_t grid = (uint64_t)sms * ACZ_ENC_COUNT_CTAS;  // persistent counting pass
    if (grid > chunks) grid = chunks;
    if (grid == 0) grid = 1;
    cudaError_t e = cudaMemsetAsync(a.status, 0, sizeof(TileStatus) * grid, s);
    if (e != cudaSuccess) return e;
    a.chunk_off = reinterpret_cast<unsigned long long*>(
        reinterpret_cast<char*>(a.status) + align256(sizeof(TileStatus) * (uint64_t)sms * ACZ_ENC_COUNT_CTAS));
    const int mode = a.max_len <= 27 ? 0 : a.max_len <= 32 ? 1 : 2;
    if (a.sym16) {
        if (mode == 0) k_encode_count<uint16_t, true><<<(unsigned)grid, kCountThreads, 0, s>>>(a);
        else k_encode_count<uint16_t, false><<<(unsigned)grid, kCountThreads, 0, s>>>(a);
    } else {
        if (mode == 0) k_encode_count<uint32_t, true><<<(unsigned)grid, kCountThreads, 0, s>>>(a);
        else k_encode_count<uint32_t, false><<<(unsigned)grid, kCountThreads, 0, s>>>(a);
    }
    ++*launches;
    const uint32_t stage_words = (uint32_t)((uint64_t)kChunk * (a.max_len ? a.max_len : 1) / 32 + 4);
    const size_t smem = (size_t)stage_words * 4 * (kEncThreads / 32);
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
        for (const void* f : {(const void*)k_encode_write<uint16_t, 0>,
                              (const void*)k_encode_write<uint16_t, 1>,
                              (const void*)k_encode_write<uint16_t, 2>,
                              (const void*)k_encode_write<uint32_t, 0>,
                              (const void*)k_encode_write<uint32_t, 1>,
                              (const void*)k_encode_write<uint32_t, 2>}) {
            e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
        }
        attr = smem;
    }
    const uint64_t wgrid = std::min<uint64_t>((chunks + kEncThreads / 32 - 1) / (kEncThreads / 32),
                                              (uint64_t)sms * 16);
#define ACZ_ENC_WRITE(T, M) k_encode_write<T, M><<<(unsigned)wgrid, kEncThreads, smem, s>>>(a, stage_words)
    if (a.sym16) {
        if (mode == 0) ACZ_ENC_WRITE(uint16_t, 0);
        else if (mode == 1) ACZ_ENC_WRITE(uint16_t, 1);
        else ACZ_ENC_WRITE(uint16_t, 2);
    } else {
        if (mode == 0) ACZ_ENC_WRITE(uint32_t, 0);
        else if (mode == 1) ACZ_ENC_WRITE(uint32_t, 1);
        else ACZ_ENC_WRITE(uint32_t, 2);
    }
#undef ACZ_ENC_WRITE
    ++*launches;
    return cudaGetLastError();
}

}  // namespace acz_b200
