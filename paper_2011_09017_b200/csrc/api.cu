// C-ABI implementation (include/acz_gpu.h): host orchestration of the device codec.
//
// compress  (ref src/codec.cpp:61-120):  K2 quant -> K3 histogram -> K4 codebook ->
//            [one stream sync: book size, total bits, outlier count, error flags] ->
//            blob allocation -> K5 encode (bitstream + outliers + decode sidecar).
// decompress (ref src/codec.cpp:122-171): K6+K7 fused chunk-parallel decode/reconstruct.
// ACZ1 (ref src/codec.cpp:177-262): header assembled on the host, bitstream copied
//            device->host straight into place (device bytes already are ACZ1 order).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "internal.h"

using namespace acz_b200;

// ------------------------------------------------------------------------- structs --
// Device block read back once per compress (codebook results + error flags).
struct SmallBlock {
    BookInfo info;
    unsigned int flags;
    unsigned int ticket;
    unsigned long long nnz;
    double sumabs;
    unsigned int maxsym;
    unsigned int hist_done;  // histogram CTA arrivals (fused codebook), zero between calls
    unsigned long long binding;  // sidecar binding computed on the device (sidecar export)
    unsigned int spec_fix;       // K2b planes the serial replay redid (read back with the book)
    CanonTables canon;
    uint32_t lut[kLutSize];
};

// Per-tensor workspace. A batched compress uses one slot per tensor so the tensors'
// kernels can run concurrently on the context's internal streams.
struct Slot {
    void* ws_sym = nullptr;
    size_t ws_sym_cap = 0;
    void* ws_hist = nullptr;  // u64 bins x alphabet + touched bitmap; kept zero between calls
    size_t ws_hist_cap = 0;
    bool hist_clean = false;
    void* ws_enc = nullptr;
    size_t ws_enc_cap = 0;
    uint32_t enc_alphabet = 0;
    uint32_t book_alphabet = 0;     // the last build_book's alphabet / leaf bound (book_wait)
    uint32_t book_center = 0;       // its centre symbol (the zero residual)
    uint64_t book_max_leaves = 0;
    bool book_pending = false;      // a build_book whose book_wait has not run (dirty bins)
    bool last_book_slow = false;    // the last book_wait ran the global-scratch codebook
    void* ws_cb = nullptr;
    size_t ws_cb_cap = 0;
    void* ws_status = nullptr;
    size_t ws_status_cap = 0;
    void* ws_row = nullptr;
    size_t ws_row_cap = 0;
    void* ws_book = nullptr;  // codebook output (sym u32 + len u8) before the blob exists
    size_t ws_book_cap = 0;
    void* ws_side = nullptr;  // sidecar chain states produced by K2
    size_t ws_side_cap = 0;
    void* ws_qs = nullptr;  // speculative quantiser scratch (look-back status, anchors)
    size_t ws_qs_cap = 0;
    void* ws_in = nullptr;  // device copy of a host input (host-buffer batched compress)
    size_t ws_in_cap = 0;
    void* ws_pack = nullptr;  // ACZ1 codebook + outliers serialised on the device
    size_t ws_pack_cap = 0;
    SmallBlock* d_small = nullptr;
    SmallBlock* h_small = nullptr;  // pinned mirror
    void* h_small_dev = nullptr;    // its device-side (mapped) address
    cudaEvent_t ev_book = nullptr;  // recorded after the codebook read-back
    cudaEvent_t ev_up = nullptr;    // host-input upload complete (serialises batch uploads)
    cudaEvent_t ev_dec = nullptr;   // host-batch decode complete (download may start)
    // Stream hand-over: the slot's workspaces are read by kernels still in flight on the
    // stream of its last call; a call on another stream waits for that work first.
    cudaEvent_t ev_last = nullptr;
    cudaStream_t last_stream = nullptr;
    bool has_last = false;
    uint64_t last_n = 0;
    bool last_sym16 = false;
};

struct acz_gpu_ctx {
    int device = 0;
    int sms = 148;
    std::string err;
    uint64_t launches = 0;
    cudaStream_t own = nullptr;  // stream used by the host-buffer entry points
    cudaStream_t io_up = nullptr, io_down = nullptr;  // copy streams of the host batches
    cudaEvent_t io_ev = nullptr;
    std::vector<Slot*> slots;    // slot 0 serves the single-tensor entry points
    std::vector<cudaStream_t> pool;     // internal streams of the batched entry points
    std::vector<cudaEvent_t> pool_ev;   // one per pool stream (join)
    cudaEvent_t ev_fork = nullptr;
    // Blob sizes of the last batched compress of each (shape, eb, radius, predictor): the
    // next one launches its encode before the codebook read-back reaches the host, into a
    // blob sized from these (see spec_encode).
    struct SizePred {
        uint32_t book;
        uint64_t bits, nout;
        uint32_t max_len;
    };
    std::unordered_map<std::string, SizePred> size_cache;
    // (shape, eb, radius) whose last K2b compress had to replay more than a quarter of its
    // planes serially (large error bounds defeat the walk): quantised by K2a from then on
    std::unordered_map<std::string, bool> spec_bad;
    // Asynchronous compresses awaiting their settle (acz_gpu_compress_async): a ring of
    // BookInfo + flags copies in mapped pinned memory (one entry per pending blob, written
    // by the device right behind the codebook) and its free list.
    void* async_host = nullptr;
    void* async_dev = nullptr;
    std::vector<uint32_t> async_free;
    // Sticky internal-error word in mapped pinned memory: kernels that detect an internal
    // consistency failure after the host has stopped waiting (the encoder's look-back) OR
    // kFlagInternal into it; every entry point reports it (ACZ_ERR_CUDA) and clears it.
    unsigned int* h_sticky = nullptr;
    unsigned int* d_sticky = nullptr;
    // K1 fixed-order reduction of sum|x| (deterministic mean_abs): per-CTA partials + ticket
    double* d_partials = nullptr;
    unsigned int* d_ticket = nullptr;
    void* ws_io = nullptr;  // host-API staging (input / output floats)
    size_t ws_io_cap = 0;
    void* ws_aux = nullptr;  // sequential-decode scratch (symbols, plane prefixes)
    size_t ws_aux_cap = 0;
    void* ws_scan = nullptr;  // parallel stream-scan scratch (subsequence starts / counts)
    size_t ws_scan_cap = 0;
    // profiling: events recorded around every launch when enabled
    bool prof = false;
    struct Pending {
        int cls;
        cudaEvent_t a, b;
    };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> event_pool;
    double prof_ms[ACZ_K_COUNT] = {0};
    uint64_t prof_n[ACZ_K_COUNT] = {0};
};

namespace {
cudaEvent_t take_event(acz_gpu_ctx* c) {
    if (!c->event_pool.empty()) {
        cudaEvent_t e = c->event_pool.back();
        c->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}
// RAII timer around one kernel launch (no-op unless profiling is on).
struct KTimer {
    acz_gpu_ctx* c;
    int cls;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    KTimer(acz_gpu_ctx* c_, int cls_, cudaStream_t s_) : c(c_), cls(cls_), s(s_) {
        if (c->prof) {
            a = take_event(c);
            cudaEventRecord(a, s);
        }
    }
    ~KTimer() {
        if (c->prof && a) {
            cudaEvent_t b = take_event(c);
            cudaEventRecord(b, s);
            c->pending.push_back({cls, a, b});
        }
    }
};
}  // namespace

struct acz_gpu_blob {
    acz_gpu_blob_info_t info{};
    uint64_t interval = 0, nchunks = 0, nwords = 0;
    uint32_t max_len = 0;
    // device arena
    void* arena = nullptr;
    size_t arena_bytes = 0;
    uint32_t* book_sym = nullptr;
    uint8_t* book_len = nullptr;
    uint32_t* words = nullptr;
    unsigned long long* out_index = nullptr;
    float* out_value = nullptr;
    unsigned long long* side_bitoff = nullptr;
    uint32_t* side_outl = nullptr;
    float* side_state = nullptr;
    uint32_t* lut = nullptr;
    CanonTables* canon = nullptr;
    cudaStream_t stream = nullptr;
    int invalid = 0;  // deferred decompress failure (foreign blobs), ACZ_ERR_*
    std::string invalid_msg;
    struct AsyncPending* async = nullptr;  // an unsettled acz_gpu_compress_async
};

namespace acz_b200 {
// Device memory held by live blobs (process-wide; arenas come from the stream-ordered pool):
// what a training step actually stashes in HBM, incl. decode sidecars and tables.
std::atomic<uint64_t> g_blob_live{0}, g_blob_peak{0};

void blob_bytes_add(uint64_t b) {
    const uint64_t v = g_blob_live.fetch_add(b) + b;
    uint64_t pk = g_blob_peak.load();
    while (v > pk && !g_blob_peak.compare_exchange_weak(pk, v)) {
    }
}

// Releases a blob's arena (stream-ordered) and its accounting.
void blob_arena_free(acz_gpu_blob* b, cudaStream_t s) {
    if (!b->arena) return;
    cudaFreeAsync(b->arena, s);
    g_blob_live.fetch_sub(b->arena_bytes);
    b->arena = nullptr;
}

PlaneGeom plane_geom(const uint64_t* shape, uint32_t rank) {
    PlaneGeom g{1, 1, 1, 1, 0};
    if (rank == 0) {
        g.n = 0;
        return g;
    }
    uint64_t n = 1;
    for (uint32_t i = 0; i < rank; ++i) n *= shape[i];
    g.n = n;
    if (rank == 1) {
        g.cols = shape[0];
    } else {
        g.rows = shape[rank - 2];
        g.cols = shape[rank - 1];
        for (uint32_t i = 0; i + 2 < rank; ++i) g.planes *= shape[i];
    }
    g.plane_size = g.rows * g.cols;
    return g;
}
}  // namespace acz_b200

namespace {

const char* kVersion = "acz-b200 0.1 (sm_100a)";

int fail(acz_gpu_ctx* c, int code, const std::string& msg) {
    if (c) c->err = msg;
    return code;
}

// No exception crosses the C-ABI: host allocation failures (std::bad_alloc from the
// per-call vectors, e.g. sized by an untrusted blob) map to ACZ_ERR_NOMEM.
template <class F>
int guarded(acz_gpu_ctx* c, F&& f) {
    try {
        return f();
    } catch (const std::bad_alloc&) {
        return fail(c, ACZ_ERR_NOMEM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(c, ACZ_ERR_INVALID, std::string("unexpected exception: ") + e.what());
    } catch (...) {
        return fail(c, ACZ_ERR_INVALID, "unexpected exception");
    }
}

int cuda_fail(acz_gpu_ctx* c, cudaError_t e, const char* where) {
    return fail(c, ACZ_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(expr)                                                   \
    do {                                                           \
        cudaError_t _e = (expr);                                   \
        if (_e != cudaSuccess) return cuda_fail(ctx, _e, #expr);   \
    } while (0)

cudaError_t grow(void** p, size_t* cap, size_t need) {
    if (need <= *cap && *p) return cudaSuccess;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    size_t want = std::max<size_t>(need, 256);
    cudaError_t e = cudaMalloc(p, want);
    if (e == cudaSuccess) *cap = want;
    return e;
}

bool params_ok(double eb, uint32_t radius) {
    // ref src/codec.cpp:54-59
    return (eb > 0.0) && std::isfinite(eb) && radius >= 2 && radius <= (1u << 24) &&
           (radius & (radius - 1)) == 0;
}

const char* param_msg(double eb) {
    return (!(eb > 0.0) || !std::isfinite(eb)) ? "error bound must be positive"
                                               : "quant_radius must be a power of two in [2, 2^24]";
}

uint64_t sidecar_interval_default() {
    static uint64_t v = [] {
        const char* s = std::getenv("ACZ_SIDECAR_INTERVAL");
        uint64_t x = s ? std::strtoull(s, nullptr, 10) : 0;
        if (x < 32) x = 128;  // the decoder's output tiles need a multiple of 32
        uint64_t p2 = 1;
        while (p2 * 2 <= x) p2 *= 2;  // power of two (mask arithmetic in the kernels)
        return p2;
    }();
    return v;
}

// Sidecar interval of a tensor: PrevValue and the Lorenzo2d wavefront path use fixed-size
// chunks (chunk-parallel symbol decode); row-major Lorenzo2d (single-row or very tall planes)
// one chunk per plane.
bool lorenzo_wave(const PlaneGeom& g) { return g.rows > 1 && g.rows <= kLorenzoWaveRows; }
uint64_t sidecar_interval_for(uint32_t pred, const PlaneGeom& g) {
    return (pred == ACZ_PRED_PREV || lorenzo_wave(g)) ? sidecar_interval_default() : g.plane_size;
}

uint64_t acz1_size(uint32_t rank, uint32_t book, uint64_t bits, uint64_t nout) {
    // ref src/codec.cpp:177-199
    return 4 + 1 + 1 + 1 + 8ull * rank + 8 + 4 + 4 + 2 + 5ull * book + 8 + (bits + 7) / 8 +
           12ull * nout;
}

size_t al(size_t v) { return (v + 255) & ~size_t(255); }

// Allocates the blob arena for the given sizes and carves the pointers.
cudaError_t blob_alloc(acz_gpu_blob* b, uint32_t book, uint64_t nwords, uint64_t nout,
                       uint64_t nchunks, bool with_outl, cudaStream_t s) {
    size_t off = 0;
    const size_t o_sym = off; off += al(4ull * std::max<uint32_t>(book, 1));
    const size_t o_len = off; off += al(std::max<uint32_t>(book, 1));
    const size_t o_words = off; off += al(4ull * (nwords + 32));  // decoder reads 3 blocks ahead
    const size_t o_oidx = off; off += al(8ull * std::max<uint64_t>(nout, 1));
    const size_t o_oval = off; off += al(4ull * std::max<uint64_t>(nout, 1));
    const size_t o_sb = off; off += al(8ull * std::max<uint64_t>(nchunks, 1));
    const size_t o_so = off; off += with_outl ? al(4ull * std::max<uint64_t>(nchunks, 1)) : 0;
    const size_t o_ss = off; off += al(4ull * std::max<uint64_t>(nchunks, 1));
    const size_t o_lut = off; off += al(4ull * kLutSize);
    const size_t o_canon = off; off += al(sizeof(CanonTables));
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, off, s);
    if (e != cudaSuccess) return e;
    char* c = static_cast<char*>(p);
    b->arena = p;
    b->arena_bytes = off;
    blob_bytes_add(off);
    b->book_sym = reinterpret_cast<uint32_t*>(c + o_sym);
    b->book_len = reinterpret_cast<uint8_t*>(c + o_len);
    b->words = reinterpret_cast<uint32_t*>(c + o_words);
    b->out_index = reinterpret_cast<unsigned long long*>(c + o_oidx);
    b->out_value = reinterpret_cast<float*>(c + o_oval);
    b->side_bitoff = reinterpret_cast<unsigned long long*>(c + o_sb);
    b->side_outl = with_outl ? reinterpret_cast<uint32_t*>(c + o_so) : nullptr;
    b->side_state = reinterpret_cast<float*>(c + o_ss);
    b->lut = reinterpret_cast<uint32_t*>(c + o_lut);
    b->canon = reinterpret_cast<CanonTables*>(c + o_canon);
    b->stream = s;
    return cudaSuccess;
}

// ACZS v3: "ACZS" u32 version, u64 {count, bit_length, interval, nchunks, binding, has_outl},
// u64 bit offset x nchunks, [u32 outlier prefix x nchunks if has_outl], f32 state x nchunks.
uint64_t sidecar_bytes(uint64_t nchunks, bool has_outl) {
    return 4 + 4 + 8 * 6 + nchunks * (8 + (has_outl ? 4 : 0) + 4);
}

uint64_t fnv1a(const uint8_t* p, size_t n, uint64_t h = 1469598103934665603ull) {
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

constexpr uint32_t kSidecarVersion = 3;

// Header part of the sidecar binding (acz_binding in common.cuh adds the codebook and a
// sampled bitstream digest): rank, extents, eb, radius, predictor, sizes.
uint64_t blob_binding_h0(const acz_gpu_blob_info_t& in) {
    uint64_t h = fnv1a(reinterpret_cast<const uint8_t*>(&in.rank), sizeof(in.rank));
    h = fnv1a(reinterpret_cast<const uint8_t*>(in.shape), 8ull * in.rank, h);
    h = fnv1a(reinterpret_cast<const uint8_t*>(&in.eb), 8, h);
    h = fnv1a(reinterpret_cast<const uint8_t*>(&in.quant_radius), 4, h);
    h = fnv1a(reinterpret_cast<const uint8_t*>(&in.predictor), 4, h);
    h = fnv1a(reinterpret_cast<const uint8_t*>(&in.codebook_size), 4, h);
    h = fnv1a(reinterpret_cast<const uint8_t*>(&in.bit_length), 8, h);
    h = fnv1a(reinterpret_cast<const uint8_t*>(&in.outlier_count), 8, h);
    return h;
}

int ensure_small(acz_gpu_ctx* ctx, Slot* sl) {
    if (sl->d_small) return ACZ_OK;
    CK(cudaMalloc(&sl->d_small, sizeof(SmallBlock)));
    CK(cudaMemset(sl->d_small, 0, sizeof(SmallBlock)));
    CK(cudaHostAlloc(&sl->h_small, sizeof(SmallBlock), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(&sl->h_small_dev, sl->h_small, 0));
    CK(cudaEventCreateWithFlags(&sl->ev_book, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&sl->ev_up, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&sl->ev_dec, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&sl->ev_last, cudaEventDisableTiming));
    return ACZ_OK;
}

// Orders a call's use of slot sl on stream s after the slot's previous call when that one
// ran on another stream (single-tensor entry points share slot 0 whatever the stream).
int slot_enter(acz_gpu_ctx* ctx, Slot* sl, cudaStream_t s) {
    if (sl->has_last && sl->last_stream != s) CK(cudaStreamWaitEvent(s, sl->ev_last, 0));
    return ACZ_OK;
}
// Marks the end of the work a call enqueued on s for slot sl.
int slot_leave(acz_gpu_ctx* ctx, Slot* sl, cudaStream_t s) {
    CK(cudaEventRecord(sl->ev_last, s));
    sl->last_stream = s;
    sl->has_last = true;
    return ACZ_OK;
}

// Reports (and clears) an internal failure a kernel recorded after the host stopped
// waiting for it (see acz_gpu_ctx::h_sticky).
int check_sticky(acz_gpu_ctx* ctx) {
    if (!ctx->h_sticky) return ACZ_OK;
    const unsigned v = *(volatile unsigned*)ctx->h_sticky;
    if (!v) return ACZ_OK;
    *(volatile unsigned*)ctx->h_sticky = 0;
    return fail(ctx, ACZ_ERR_CUDA, "internal: encoder look-back timeout (a previous blob on "
                                   "this context may be corrupt)");
}

// Slot i (created on first use).
Slot* get_slot(acz_gpu_ctx* ctx, size_t i) {
    while (ctx->slots.size() <= i) ctx->slots.push_back(new (std::nothrow) Slot());
    return ctx->slots[i];
}

void free_slot(Slot* sl) {
    if (!sl) return;
    for (void* p : {sl->ws_sym, sl->ws_hist, sl->ws_enc, sl->ws_cb, sl->ws_status, sl->ws_row,
                    sl->ws_book, sl->ws_side, sl->ws_qs, sl->ws_in, sl->ws_pack})
        if (p) cudaFree(p);
    if (sl->ev_last) cudaEventDestroy(sl->ev_last);
    if (sl->d_small) cudaFree(sl->d_small);
    if (sl->h_small) cudaFreeHost(sl->h_small);
    if (sl->ev_book) cudaEventDestroy(sl->ev_book);
    if (sl->ev_up) cudaEventDestroy(sl->ev_up);
    if (sl->ev_dec) cudaEventDestroy(sl->ev_dec);
    delete sl;
}

// Runs the fused stats pass and returns non-finite / nnz / sum|x|.
int run_stats(acz_gpu_ctx* ctx, const float* d_in, uint64_t n, uint32_t* d_bitmap,
              cudaStream_t s, unsigned* flags, uint64_t* nnz, double* sumabs) {
    Slot* sl = get_slot(ctx, 0);
    int rc = ensure_small(ctx, sl);
    if (rc) return rc;
    if ((rc = slot_enter(ctx, sl, s))) return rc;
    CK(cudaMemsetAsync(&sl->d_small->flags, 0, sizeof(unsigned), s));
    CK(cudaMemsetAsync(&sl->d_small->nnz, 0, sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(&sl->d_small->sumabs, 0, sizeof(double), s));
    {
        KTimer kt(ctx, ACZ_K_STATS, s);
        CK(launch_stats(d_in, n, d_bitmap, &sl->d_small->nnz, &sl->d_small->flags,
                        sumabs ? &sl->d_small->sumabs : nullptr, ctx->d_partials, ctx->d_ticket,
                        ctx->sms, s, &ctx->launches));
    }
    if ((rc = slot_leave(ctx, sl, s))) return rc;
    CK(cudaMemcpyAsync(sl->h_small, sl->d_small, offsetof(SmallBlock, canon),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (flags) *flags = sl->h_small->flags;
    if (nnz) *nnz = sl->h_small->nnz;
    if (sumabs) *sumabs = sl->h_small->sumabs;
    return ACZ_OK;
}

int validate_shape(acz_gpu_ctx* ctx, const uint64_t* shape, uint32_t rank, uint64_t* n) {
    if (rank > ACZ_MAX_RANK) return fail(ctx, ACZ_ERR_SHAPE, "rank exceeds ACZ_MAX_RANK");
    if (rank && !shape) return fail(ctx, ACZ_ERR_INVALID, "null shape");
    uint64_t v = rank ? 1 : 0;
    for (uint32_t i = 0; i < rank; ++i) {
        if (shape[i] == 0) return fail(ctx, ACZ_ERR_SHAPE, "tensor extents must be positive");
        v *= shape[i];
    }
    *n = v;
    return ACZ_OK;
}

}  // namespace

// ------------------------------------------------------------------------ context --
extern "C" {

const char* acz_gpu_version(void) { return kVersion; }

int acz_gpu_ctx_create(int device, acz_gpu_ctx** out) {
    if (!out) return ACZ_ERR_INVALID;
    *out = nullptr;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return ACZ_ERR_CUDA;
    acz_gpu_ctx* ctx = new (std::nothrow) acz_gpu_ctx();
    if (!ctx) return ACZ_ERR_NOMEM;
    ctx->device = device;
    cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
    // keep freed blob memory cached in the stream-ordered pool
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    e = cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete ctx;
        return ACZ_ERR_CUDA;
    }
    void* sticky_dev = nullptr;
    if (ensure_small(ctx, get_slot(ctx, 0)) != ACZ_OK ||
        cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaHostAlloc(&ctx->h_sticky, sizeof(unsigned), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(&sticky_dev, ctx->h_sticky, 0) != cudaSuccess ||
        cudaMalloc(&ctx->d_partials, sizeof(double) * stats_partials(ctx->sms) + 256) !=
            cudaSuccess) {
        acz_gpu_ctx_destroy(ctx);
        return ACZ_ERR_CUDA;
    }
    *ctx->h_sticky = 0;
    ctx->d_sticky = static_cast<unsigned*>(sticky_dev);
    ctx->d_ticket = reinterpret_cast<unsigned*>(ctx->d_partials + stats_partials(ctx->sms));
    if (cudaMemset(ctx->d_ticket, 0, sizeof(unsigned)) != cudaSuccess) {
        acz_gpu_ctx_destroy(ctx);
        return ACZ_ERR_CUDA;
    }
    *out = ctx;
    return ACZ_OK;
}

int acz_gpu_ctx_destroy(acz_gpu_ctx* ctx) {
    if (!ctx) return ACZ_ERR_INVALID;
    cudaDeviceSynchronize();
    for (void* p : {ctx->ws_io, ctx->ws_aux, ctx->ws_scan, (void*)ctx->d_partials})
        if (p) cudaFree(p);
    if (ctx->h_sticky) cudaFreeHost(ctx->h_sticky);
    if (ctx->async_host) cudaFreeHost(ctx->async_host);
    for (Slot* sl : ctx->slots) free_slot(sl);
    for (auto st : ctx->pool) cudaStreamDestroy(st);
    for (auto e : ctx->pool_ev) cudaEventDestroy(e);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    if (ctx->io_up) cudaStreamDestroy(ctx->io_up);
    if (ctx->io_down) cudaStreamDestroy(ctx->io_down);
    if (ctx->io_ev) cudaEventDestroy(ctx->io_ev);
    for (auto& p : ctx->pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (auto e : ctx->event_pool) cudaEventDestroy(e);
    delete ctx;
    return ACZ_OK;
}

const char* acz_gpu_last_error(const acz_gpu_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

uint64_t acz_gpu_launch_count(const acz_gpu_ctx* ctx) { return ctx ? ctx->launches : 0; }

int acz_gpu_memory_info(const acz_gpu_ctx* ctx, uint64_t* workspace_bytes,
                        uint64_t* blob_live_bytes, uint64_t* blob_peak_bytes, int reset_peak) {
    if (!ctx) return ACZ_ERR_INVALID;
    uint64_t ws = ctx->ws_io_cap + ctx->ws_aux_cap + ctx->ws_scan_cap;
    for (const Slot* sl : ctx->slots) {
        if (!sl) continue;
        ws += sl->ws_sym_cap + sl->ws_hist_cap + sl->ws_enc_cap + sl->ws_cb_cap +
              sl->ws_status_cap + sl->ws_row_cap + sl->ws_book_cap + sl->ws_side_cap +
              sl->ws_qs_cap + sl->ws_in_cap + sl->ws_pack_cap + (sl->d_small ? sizeof(SmallBlock) : 0);
    }
    if (workspace_bytes) *workspace_bytes = ws;
    if (blob_live_bytes) *blob_live_bytes = g_blob_live.load();
    if (blob_peak_bytes) *blob_peak_bytes = g_blob_peak.load();
    if (reset_peak) g_blob_peak.store(g_blob_live.load());
    return ACZ_OK;
}

int acz_gpu_memory_breakdown(const acz_gpu_ctx* ctx, uint64_t* out, uint32_t n) {
    if (!ctx || !out) return ACZ_ERR_INVALID;
    uint64_t v[ACZ_MEM_COUNT] = {0};
    for (const Slot* sl : ctx->slots) {
        if (!sl) continue;
        v[ACZ_MEM_SYMBOLS] += sl->ws_sym_cap;
        v[ACZ_MEM_TABLES] += sl->ws_hist_cap + sl->ws_enc_cap + sl->ws_cb_cap + sl->ws_book_cap;
        v[ACZ_MEM_QUANT] += sl->ws_side_cap + sl->ws_qs_cap + sl->ws_row_cap;
        v[ACZ_MEM_ENCODE] += sl->ws_status_cap + sl->ws_pack_cap;
        v[ACZ_MEM_STAGING] += sl->ws_in_cap;
    }
    v[ACZ_MEM_STAGING] += ctx->ws_io_cap;
    v[ACZ_MEM_DECODE] += ctx->ws_aux_cap + ctx->ws_scan_cap;
    for (uint32_t i = 0; i < n && i < ACZ_MEM_COUNT; ++i) out[i] = v[i];
    return ACZ_OK;
}

int acz_gpu_ctx_trim(acz_gpu_ctx* ctx) {
    if (!ctx) return ACZ_ERR_INVALID;
    return guarded(ctx, [&]() -> int {
    ctx->err.clear();
    CK(cudaSetDevice(ctx->device));
    CK(cudaDeviceSynchronize());  // nothing of this context may still read its workspaces
    for (Slot*& sl : ctx->slots) {
        free_slot(sl);
        sl = new (std::nothrow) Slot();  // recreated lazily (events, small block, buffers)
        if (!sl) return fail(ctx, ACZ_ERR_NOMEM, "slot");
    }
    for (void** p : {&ctx->ws_io, &ctx->ws_aux, &ctx->ws_scan}) {
        if (*p) cudaFree(*p);
        *p = nullptr;
    }
    ctx->ws_io_cap = ctx->ws_aux_cap = ctx->ws_scan_cap = 0;
    // hand the freed blob arenas of the stream-ordered pool back to the device
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, ctx->device) == cudaSuccess)
        CK(cudaMemPoolTrimTo(pool, 0));
    return check_sticky(ctx);
    });
}

}  // extern "C"

// ----------------------------------------------------------------------- compress --
namespace {

// Symbols whose code lengths the counting pass stages in shared memory: kEncLenWindow
// symbols centred on the book's centre symbol (every symbol of a book at eb >= ~1e-4 on
// unit-scale data; the rest are looked up in the global tables).
void set_len_window(EncodeArgs& ea, const Slot* sl) {
    const uint32_t a = sl->enc_alphabet, half = (uint32_t)kEncLenWindow / 2;
    ea.len_lo = sl->book_center > half ? sl->book_center - half : 0u;
    ea.len_n = ea.len_lo < a ? std::min<uint32_t>((uint32_t)kEncLenWindow, a - ea.len_lo) : 0u;
}

// Blob-side finalisation shared by compress and the generic Huffman encoder: after the
// codebook sync, allocates the blob, copies the tables and runs K5.
int finish_encode(acz_gpu_ctx* ctx, Slot* sl, acz_gpu_blob* b, const void* d_sym, int sym16,
                  uint64_t n, const float* d_x, uint64_t interval, bool with_outl,
                  cudaStream_t s) {
    const BookInfo& bi = sl->h_small->info;
    const uint64_t nwords = (bi.total_bits + 31) / 32;
    const uint64_t nout = d_x ? bi.n_escapes : 0;
    const uint64_t nchunks = interval ? (n + interval - 1) / interval : 0;
    CK(blob_alloc(b, bi.book_size, nwords, nout, nchunks, with_outl, s));
    b->nwords = nwords;
    b->interval = interval;
    b->nchunks = nchunks;
    b->max_len = bi.max_len;
    // the encoder writes every word of the stream and zeroes the padding (no memset)
    const uint32_t* wb_sym = static_cast<const uint32_t*>(sl->ws_book);
    const uint8_t* wb_len =
        reinterpret_cast<const uint8_t*>(wb_sym + std::max<uint64_t>(sl->ws_book_cap / 5, 1));
    CopyRegions cr{};
    auto add = [&](const void* src, void* dst, uint64_t bytes) {
        cr.src[cr.n] = src;
        cr.dst[cr.n] = dst;
        cr.bytes[cr.n] = bytes;
        ++cr.n;
    };
    add(wb_sym, b->book_sym, 4ull * bi.book_size);
    add(wb_len, b->book_len, bi.book_size);
    add(sl->d_small->lut, b->lut, 4ull * kLutSize);
    add(&sl->d_small->canon, b->canon, sizeof(CanonTables));
    if (nchunks && d_x) add(sl->ws_side, b->side_state, 4ull * nchunks);
    CK(launch_copy_regions(cr, ctx->sms, s, &ctx->launches));
    EncodeArgs ea;
    ea.sym = d_sym;
    ea.sym16 = sym16;
    ea.n = n;
    ea.enc = static_cast<const unsigned long long*>(sl->ws_enc);
    ea.enc32 = reinterpret_cast<const uint32_t*>(ea.enc + sl->enc_alphabet);
    set_len_window(ea, sl);
    ea.x = d_x;
    ea.words = b->words;
    ea.nwords = nwords;
    ea.out_index = b->out_index;
    ea.out_value = b->out_value;
    ea.side_bitoff = nchunks ? b->side_bitoff : nullptr;
    ea.side_outl = b->side_outl;
    ea.interval = interval ? interval : 1;
    ea.max_len = bi.max_len;
    ea.status = static_cast<TileStatus*>(sl->ws_status);
    ea.sticky = ctx->d_sticky;
    {
        KTimer kt(ctx, ACZ_K_ENCODE, s);
        CK(launch_encode(ea, ctx->sms, s, &ctx->launches));
    }
    return ACZ_OK;
}

// Histogram + codebook + the BookInfo read-back, recorded on sl->ev_book (the caller waits
// for it before sizing the blob: the single host synchronisation of a compress).
int build_book(acz_gpu_ctx* ctx, Slot* sl, const void* d_sym, int sym16, uint64_t n,
               uint32_t alphabet, uint32_t center, cudaStream_t s) {
    const uint64_t max_leaves = std::min<uint64_t>(alphabet, n);
    const size_t hist_bytes = 8ull * alphabet + 4ull * ((alphabet + 31) / 32);
    if (hist_bytes > sl->ws_hist_cap || sl->book_pending) sl->hist_clean = false;
    CK(grow(&sl->ws_hist, &sl->ws_hist_cap, hist_bytes));
    if (!sl->hist_clean) {
        CK(cudaMemsetAsync(sl->ws_hist, 0, sl->ws_hist_cap, s));
        sl->hist_clean = true;
    }
    unsigned long long* hist = static_cast<unsigned long long*>(sl->ws_hist);
    uint32_t* touched = reinterpret_cast<uint32_t*>(hist + alphabet);
    CK(grow(&sl->ws_enc, &sl->ws_enc_cap, 12ull * alphabet));  // u64 table + u32 compact table
    sl->enc_alphabet = alphabet;
    sl->book_center = center;
    CK(grow(&sl->ws_cb, &sl->ws_cb_cap, codebook_scratch_bytes(max_leaves)));
    CK(grow(&sl->ws_book, &sl->ws_book_cap, 5ull * max_leaves + 64));
    CK(grow(&sl->ws_status, &sl->ws_status_cap, encode_scratch_bytes(n, ctx->sms)));
    uint32_t* wb_sym = static_cast<uint32_t*>(sl->ws_book);
    uint8_t* wb_len = reinterpret_cast<uint8_t*>(wb_sym + std::max<uint64_t>(sl->ws_book_cap / 5, 1));
    unsigned long long* enc = static_cast<unsigned long long*>(sl->ws_enc);
    // K3 + K4 fused (the last histogram CTA builds books of <= 8192 symbols); larger books
    // set info.slow and the host runs the global-scratch codebook (book_wait). ACZ_BOOK_UNFUSED=1
    // launches the separate kernels (development A/B).
    static const bool unfused = [] {
        const char* e = std::getenv("ACZ_BOOK_UNFUSED");
        return e && e[0] == '1';
    }();
    CbArgs cb{};
    if (!unfused) {
        cb.done = &sl->d_small->hist_done;
        cb.book_sym = wb_sym;
        cb.book_len = wb_len;
        cb.enc = enc;
        cb.canon = &sl->d_small->canon;
        cb.lut = sl->d_small->lut;
        cb.info = &sl->d_small->info;
    }
    sl->book_alphabet = alphabet;
    sl->book_max_leaves = max_leaves;
    sl->book_pending = true;
    {
    KTimer kt(ctx, ACZ_K_HIST, s);
    sl->hist_clean = false;  // until the codebook kernels have consumed the bins
    CK(launch_histogram(d_sym, sym16, n, alphabet, center, hist, touched, cb, ctx->sms, s,
                        &ctx->launches));
    }
    if (unfused) {
    KTimer kt(ctx, ACZ_K_BOOK, s);
    CK(launch_codebook(hist, touched, alphabet, max_leaves, sl->ws_cb, wb_sym, wb_len, enc,
                       &sl->d_small->canon, sl->d_small->lut, &sl->d_small->info, false, s,
                       &ctx->launches));
    }
    sl->hist_clean = true;
    // BookInfo + flags straight into the mapped pinned mirror (no copy-engine queueing)
    CopyRegions cr{};
    cr.src[0] = sl->d_small;
    cr.dst[0] = sl->h_small_dev;
    cr.bytes[0] = offsetof(SmallBlock, canon);
    cr.n = 1;
    cr.to_host = 1;
    CK(launch_copy_regions(cr, ctx->sms, s, &ctx->launches));
    CK(cudaEventRecord(sl->ev_book, s));
    return ACZ_OK;
}

int decompress_on(acz_gpu_ctx* ctx, Slot* sl, const acz_gpu_blob* b, int zero_filter,
                  float* d_out, cudaStream_t s) {
    if (!b || !d_out || !sl) return ACZ_ERR_INVALID;
    if (b->invalid) return fail(ctx, b->invalid, b->invalid_msg);
    if (int rc = check_sticky(ctx)) return rc;
    if (int rc = slot_enter(ctx, sl, s)) return rc;
    const acz_gpu_blob_info_t& in = b->info;
    const PlaneGeom g = plane_geom(in.shape, in.rank);
    if (in.predictor == ACZ_PRED_LORENZO2D)
        CK(grow(&sl->ws_row, &sl->ws_row_cap, 4ull * std::max(g.planes * g.cols, in.element_count)));
    DecodeArgs a;
    a.words = b->words;
    a.nwords = b->nwords;
    a.bit_length = in.bit_length;
    a.lut = b->lut;
    a.canon = b->canon;
    a.book_sym = b->book_sym;
    a.book_size = in.codebook_size;
    a.side_bitoff = b->side_bitoff;
    a.side_outl = b->side_outl;
    a.side_state = b->side_state;
    a.interval = b->interval;
    a.nchunks = b->nchunks;
    a.out_index = b->out_index;
    a.out_value = b->out_value;
    a.n_outliers = in.outlier_count;
    a.g = g;
    a.eb = in.eb;
    a.step = 2.0 * in.eb;
    a.radius = in.quant_radius;
    a.predictor = in.predictor;
    a.zero_filter = zero_filter;
    a.out = d_out;
    a.row_scratch = static_cast<float*>(sl->ws_row);
    a.sym_scratch = static_cast<uint32_t*>(sl->ws_row);  // (the two Lorenzo paths exclusive)
    {
        KTimer kt(ctx, ACZ_K_DECODE, s);
        CK(launch_decode(a, ctx->sms, s, &ctx->launches));
    }
    return slot_leave(ctx, sl, s);
}


// Key of a compress's (shape, eb, radius, predictor): size predictions and the K2b record.
std::string params_key(const uint64_t* shape, uint32_t rank, double eb, uint32_t radius,
                       uint32_t predictor) {
    std::string k(reinterpret_cast<const char*>(shape), 8 * rank);
    k.append(reinterpret_cast<const char*>(&eb), 8);
    k.append(reinterpret_cast<const char*>(&radius), 4);
    k.append(reinterpret_cast<const char*>(&predictor), 4);
    return k;
}

// K2b (the speculative quantiser) unless this context saw it replay more than a quarter of
// the planes of the same (shape, eb, radius) serially -- large error bounds (e.g. eb = 0.1
// on unit-scale data, the controller's default eb_max) defeat its walk, and the serial
// replay after it costs more than K2a alone (128x3x224x224 at eb = 0.1: K2b 2.9 ms + replay
// 3.7 ms). ACZ_SPEC_QUANT=1 (tests) always takes K2b.
bool use_k2b(acz_gpu_ctx* ctx, const std::string& key, uint32_t predictor, const PlaneGeom& g) {
    if (!quant_spec_applicable(predictor, g.plane_size, g.planes, ctx->sms)) return false;
    if (std::getenv("ACZ_SPEC_QUANT")) return true;
    auto it = ctx->spec_bad.find(key);
    return it == ctx->spec_bad.end() || !it->second;
}

// State of a compress between its asynchronous first half (quantiser, histogram, codebook)
// and its second half (blob sizing after the BookInfo read-back, encode).
struct Plan {
    uint64_t n = 0;
    PlaneGeom g{};
    uint32_t rank = 0;
    uint64_t shape[ACZ_MAX_RANK] = {0};
    double eb = 0;
    uint32_t radius = 0, predictor = 0;
    uint64_t interval = 0;
    int sym16 = 0;
    const float* d_in = nullptr;
    bool k2b = false;  // quantised by K2b (its serial-replay count is read with the book)
    // speculative encode (spec_encode): the pre-sized blob and its capacities
    acz_gpu_blob* spec = nullptr;
    unsigned long long cap_bits = 0;
    uint64_t cap_out = 0;
    uint32_t cap_book = 0, cap_len = 0;
};

int compress_begin(acz_gpu_ctx* ctx, Slot* sl, const float* d_in, const uint64_t* shape,
                   uint32_t rank, double eb, uint32_t quant_radius, uint32_t predictor,
                   cudaStream_t s, Plan* pl) {
    uint64_t n = 0;
    int rc = validate_shape(ctx, shape, rank, &n);
    if (rc) return rc;
    if (n && !d_in) return fail(ctx, ACZ_ERR_INVALID, "null input");
    if (predictor > 1) return fail(ctx, ACZ_ERR_PARAM, "unknown predictor");
    if (!params_ok(eb, quant_radius)) {
        // The reference builds the Tensor (finiteness check) before compress validates.
        if (n) {
            unsigned fl = 0;
            rc = run_stats(ctx, d_in, n, nullptr, s, &fl, nullptr, nullptr);
            if (rc) return rc;
            if (fl & kFlagNonFinite) return fail(ctx, ACZ_ERR_DOMAIN, "tensor element is not finite");
        }
        return fail(ctx, ACZ_ERR_PARAM, param_msg(eb));
    }
    if (n == 0) return fail(ctx, ACZ_ERR_DOMAIN, "compress: empty tensor");
    rc = ensure_small(ctx, sl);
    if (rc) return rc;
    if ((rc = slot_enter(ctx, sl, s))) return rc;
    const PlaneGeom g = plane_geom(shape, rank);
    const uint32_t alphabet = 2u * quant_radius;
    const uint64_t interval = sidecar_interval_for(predictor, g);
    const uint64_t nchunks = (n + interval - 1) / interval;

    const int sym16 = (predictor == ACZ_PRED_PREV && quant_radius <= 32768) ? 1 : 0;
    // u16 symbols take 2 bytes per element (+16: the encoder's vector loads of the tail)
    CK(grow(&sl->ws_sym, &sl->ws_sym_cap, (sym16 ? 2ull : 4ull) * n + 16));
    CK(grow(&sl->ws_side, &sl->ws_side_cap, 4ull * nchunks));
    if (predictor == ACZ_PRED_LORENZO2D)
        CK(grow(&sl->ws_row, &sl->ws_row_cap, 4ull * g.planes * g.cols));
    sl->last_n = n;
    sl->last_book_slow = false;

    SmallBlock* sm = sl->d_small;
    CK(cudaMemsetAsync(&sm->flags, 0, sizeof(unsigned), s));
    QuantArgs qa;
    qa.x = d_in;
    qa.g = g;
    qa.eb = eb;
    qa.step = 2.0 * eb;
    qa.radius = quant_radius;
    qa.predictor = predictor;
    sl->last_sym16 = sym16 != 0;
    qa.sym = sym16 ? nullptr : static_cast<uint32_t*>(sl->ws_sym);
    qa.sym16 = sym16 ? static_cast<uint16_t*>(sl->ws_sym) : nullptr;
    qa.side_state = static_cast<float*>(sl->ws_side);
    qa.interval = interval;
    qa.row_scratch = static_cast<float*>(sl->ws_row);
    qa.flags = &sm->flags;
    const bool k2b = use_k2b(ctx, params_key(shape, rank, eb, quant_radius, predictor),
                             predictor, g);
    {
        KTimer kt(ctx, ACZ_K_QUANT, s);
        if (k2b) {
            CK(grow(&sl->ws_qs, &sl->ws_qs_cap, quant_spec_scratch_bytes(g.planes, g.plane_size)));
            CK(cudaMemsetAsync(&sm->spec_fix, 0, sizeof(unsigned), s));
            qa.spec_fix = &sm->spec_fix;
            CK(launch_quant_spec(qa, sl->ws_qs, s, &ctx->launches));
        } else {
            CK(launch_quant(qa, ctx->sms, s, &ctx->launches));
        }
    }
    rc = build_book(ctx, sl, sl->ws_sym, sym16, n, alphabet, quant_radius, s);
    if (const int lr = slot_leave(ctx, sl, s)) return lr;
    if (rc) return rc;
    pl->n = n;
    pl->g = g;
    pl->rank = rank;
    for (uint32_t i = 0; i < rank; ++i) pl->shape[i] = shape[i];
    pl->eb = eb;
    pl->radius = quant_radius;
    pl->predictor = predictor;
    pl->interval = interval;
    pl->sym16 = sym16;
    pl->d_in = d_in;
    pl->k2b = k2b;
    return ACZ_OK;
}

// Waits for the codebook (ev_book). A book of more than 8192 symbols leaves info.slow set
// by the fused kernel: the global-scratch codebook then runs here, followed by a second
// BookInfo read-back (small error bounds only).
int book_wait(acz_gpu_ctx* ctx, Slot* sl, cudaStream_t s) {
    CK(cudaEventSynchronize(sl->ev_book));
    sl->book_pending = false;
    if (!sl->h_small->info.slow) return ACZ_OK;
    sl->last_book_slow = true;
    sl->book_pending = true;
    unsigned long long* hist = static_cast<unsigned long long*>(sl->ws_hist);
    uint32_t* touched = reinterpret_cast<uint32_t*>(hist + sl->book_alphabet);
    uint32_t* wb_sym = static_cast<uint32_t*>(sl->ws_book);
    uint8_t* wb_len = reinterpret_cast<uint8_t*>(wb_sym + std::max<uint64_t>(sl->ws_book_cap / 5, 1));
    {
    KTimer kt(ctx, ACZ_K_BOOK, s);
    CK(launch_codebook(hist, touched, sl->book_alphabet, sl->book_max_leaves, sl->ws_cb, wb_sym,
                       wb_len, static_cast<unsigned long long*>(sl->ws_enc), &sl->d_small->canon,
                       sl->d_small->lut, &sl->d_small->info, true, s, &ctx->launches));
    }
    CopyRegions cr{};
    cr.src[0] = sl->d_small;
    cr.dst[0] = sl->h_small_dev;
    cr.bytes[0] = offsetof(SmallBlock, canon);
    cr.n = 1;
    cr.to_host = 1;
    CK(launch_copy_regions(cr, ctx->sms, s, &ctx->launches));
    CK(cudaEventRecord(sl->ev_book, s));
    CK(cudaEventSynchronize(sl->ev_book));
    sl->book_pending = false;
    return ACZ_OK;
}

int compress_end(acz_gpu_ctx* ctx, Slot* sl, const Plan& pl, cudaStream_t s, acz_gpu_blob** out) {
    if (int rc = book_wait(ctx, sl, s)) return rc;
    if (pl.k2b)
        ctx->spec_bad[params_key(pl.shape, pl.rank, pl.eb, pl.radius, pl.predictor)] =
            4ull * sl->h_small->spec_fix > pl.g.planes;
    if (int rc = check_sticky(ctx)) return rc;
    const BookInfo bi = sl->h_small->info;
    const unsigned flags = sl->h_small->flags | bi.flags;
    // precedence follows the reference: Tensor ctor (DomainError), huffman_encode
    // (DecodeError), then the codebook limit in compress (FormatError).
    if (flags & kFlagNonFinite) return fail(ctx, ACZ_ERR_DOMAIN, "tensor element is not finite");
    if (flags & kFlagInternal) return fail(ctx, ACZ_ERR_CUDA, "internal: look-back timeout");
    if (flags & kFlagDepth64) return fail(ctx, ACZ_ERR_DECODE, "huffman code length exceeds 64 bits");
    if (bi.book_size > kMaxBook)
        return fail(ctx, ACZ_ERR_FORMAT, "codebook exceeds the 65535-entry limit of the blob format");
    if (flags & kFlagLenTooLong) return fail(ctx, ACZ_ERR_FORMAT, "code length > 56 bits unsupported");

    acz_gpu_blob* b = new (std::nothrow) acz_gpu_blob();
    if (!b) return fail(ctx, ACZ_ERR_NOMEM, "blob");
    int rc = finish_encode(ctx, sl, b, sl->ws_sym, pl.sym16, pl.n, pl.d_in, pl.interval,
                           pl.predictor == ACZ_PRED_LORENZO2D, s);
    if (const int lr = slot_leave(ctx, sl, s)) rc = rc ? rc : lr;
    if (rc) {
        blob_arena_free(b, s);
        delete b;
        return rc;
    }
    acz_gpu_blob_info_t& in = b->info;
    in.rank = pl.rank;
    for (uint32_t i = 0; i < pl.rank; ++i) in.shape[i] = pl.shape[i];
    in.eb = pl.eb;
    in.quant_radius = pl.radius;
    in.predictor = pl.predictor;
    in.element_count = pl.n;
    in.codebook_size = bi.book_size;
    in.bit_length = bi.total_bits;
    in.outlier_count = bi.n_escapes;
    in.uncompressed_bytes = 4ull * pl.n;
    in.compressed_bytes = acz1_size(pl.rank, bi.book_size, bi.total_bits, bi.n_escapes);
    in.device_bytes = b->arena_bytes;
    in.sidecar_bytes = sidecar_bytes(b->nchunks, b->side_outl != nullptr);
    in.max_code_length = bi.max_len;
    *out = b;
    return ACZ_OK;
}

// Speculative encode (batched compress, PrevValue): the encode is enqueued right behind the
// codebook on the tensor's stream, into a blob sized from the same tensor shape's previous
// compress with margins (+6.25 % + 32 KB of bitstream, 2x + 4096 outliers, +1024 book
// entries, the code-length class of the previous book). The kernels read the sizes from
// the device BookInfo and write nothing if the book does not fit (or needed the global
// codebook, or flagged an error); the host, which still reads every book back, then
// re-encodes that tensor into an exactly sized blob (spec_finish). The GPU thus never waits
// for the host between a tensor's codebook and its encode.
std::string size_key(const Plan& pl) {
    return params_key(pl.shape, pl.rank, pl.eb, pl.radius, pl.predictor);
}

// Opt-in (ACZ_SPEC_ENCODE=1, read per batch): measured neutral on the AlexNet step and
// 4 % slower on ResNet-18 B128 (20 tensors: the early encodes contend with the other
// tensors' quantisers and histograms), at +6 % device bytes per blob.
bool spec_encode_enabled() {
    const char* e = std::getenv("ACZ_SPEC_ENCODE");
    return e && e[0] == '1';
}

int spec_encode(acz_gpu_ctx* ctx, Slot* sl, Plan* pl, const acz_gpu_ctx::SizePred& pr,
                cudaStream_t s) {
    const uint64_t n = pl->n, interval = pl->interval;
    const uint64_t nchunks = (n + interval - 1) / interval;
    pl->cap_book = (uint32_t)std::min<uint64_t>(std::min<uint64_t>(sl->book_max_leaves, kMaxBook),
                                                 (uint64_t)pr.book + 1024);
    pl->cap_bits = pr.bits + pr.bits / 16 + 262144;
    pl->cap_out = pr.nout * 2 + 4096;
    pl->cap_len = pr.max_len <= 27 ? 27u : pr.max_len <= 32 ? 32u : 56u;
    const uint64_t nwords = (pl->cap_bits + 31) / 32;
    acz_gpu_blob* b = new (std::nothrow) acz_gpu_blob();
    if (!b) return fail(ctx, ACZ_ERR_NOMEM, "blob");
    if (cudaError_t e = blob_alloc(b, pl->cap_book, nwords, pl->cap_out, nchunks, false, s)) {
        delete b;
        return cuda_fail(ctx, e, "spec blob");
    }
    b->interval = interval;
    b->nchunks = nchunks;
    const uint32_t* wb_sym = static_cast<const uint32_t*>(sl->ws_book);
    const uint8_t* wb_len =
        reinterpret_cast<const uint8_t*>(wb_sym + std::max<uint64_t>(sl->ws_book_cap / 5, 1));
    CopyRegions cr{};
    auto add = [&](const void* src, void* dst, uint64_t bytes) {
        cr.src[cr.n] = src;
        cr.dst[cr.n] = dst;
        cr.bytes[cr.n] = bytes;
        ++cr.n;
    };
    add(wb_sym, b->book_sym, 4ull * pl->cap_book);
    add(wb_len, b->book_len, pl->cap_book);
    add(sl->d_small->lut, b->lut, 4ull * kLutSize);
    add(&sl->d_small->canon, b->canon, sizeof(CanonTables));
    add(sl->ws_side, b->side_state, 4ull * nchunks);
    int rc = ACZ_OK;
    if (cudaError_t e = launch_copy_regions(cr, ctx->sms, s, &ctx->launches)) rc = cuda_fail(ctx, e, "spec copy");
    EncodeArgs ea;
    ea.sym = sl->ws_sym;
    ea.sym16 = pl->sym16;
    ea.n = n;
    ea.enc = static_cast<const unsigned long long*>(sl->ws_enc);
    ea.enc32 = reinterpret_cast<const uint32_t*>(ea.enc + sl->enc_alphabet);
    set_len_window(ea, sl);
    ea.x = pl->d_in;
    ea.words = b->words;
    ea.nwords = nwords;
    ea.out_index = b->out_index;
    ea.out_value = b->out_value;
    ea.side_bitoff = b->side_bitoff;
    ea.side_outl = nullptr;
    ea.interval = interval;
    ea.max_len = pl->cap_len;
    ea.status = static_cast<TileStatus*>(sl->ws_status);
    ea.sticky = ctx->d_sticky;
    ea.spec_info = &sl->d_small->info;
    ea.cap_bits = pl->cap_bits;
    ea.cap_out = pl->cap_out;
    ea.cap_book = pl->cap_book;
    ea.cap_len = pl->cap_len;
    if (!rc) {
        KTimer kt(ctx, ACZ_K_ENCODE, s);
        if (cudaError_t e = launch_encode(ea, ctx->sms, s, &ctx->launches)) rc = cuda_fail(ctx, e, "spec encode");
    }
    if (const int lr = slot_leave(ctx, sl, s)) rc = rc ? rc : lr;
    if (rc) {
        blob_arena_free(b, s);
        delete b;
        return rc;
    }
    pl->spec = b;
    return ACZ_OK;
}

// Second half of a speculatively encoded tensor: the book read-back decides whether the
// blob holds the encode (fill in its sizes) or the tensor is re-encoded exactly.
int spec_finish(acz_gpu_ctx* ctx, Slot* sl, Plan& pl, cudaStream_t s, acz_gpu_blob** out) {
    acz_gpu_blob* b = pl.spec;
    pl.spec = nullptr;
    int rc = book_wait(ctx, sl, s);
    if (!rc) rc = check_sticky(ctx);
    const BookInfo bi = sl->h_small->info;
    const unsigned flags = sl->h_small->flags | bi.flags;
    const bool fits = !rc && !flags && !sl->last_book_slow && bi.book_size >= 1 &&
                      bi.total_bits <= pl.cap_bits && bi.n_escapes <= pl.cap_out &&
                      bi.book_size <= pl.cap_book && bi.max_len <= pl.cap_len;
    if (!fits) {
        blob_arena_free(b, s);
        delete b;
        return rc ? rc : compress_end(ctx, sl, pl, s, out);
    }
    b->nwords = (bi.total_bits + 31) / 32;
    b->max_len = bi.max_len;
    acz_gpu_blob_info_t& in = b->info;
    in.rank = pl.rank;
    for (uint32_t i = 0; i < pl.rank; ++i) in.shape[i] = pl.shape[i];
    in.eb = pl.eb;
    in.quant_radius = pl.radius;
    in.predictor = pl.predictor;
    in.element_count = pl.n;
    in.codebook_size = bi.book_size;
    in.bit_length = bi.total_bits;
    in.outlier_count = bi.n_escapes;
    in.uncompressed_bytes = 4ull * pl.n;
    in.compressed_bytes = acz1_size(pl.rank, bi.book_size, bi.total_bits, bi.n_escapes);
    in.device_bytes = b->arena_bytes;
    in.sidecar_bytes = sidecar_bytes(b->nchunks, false);
    in.max_code_length = bi.max_len;
    *out = b;
    return ACZ_OK;
}

// ACZ1 bytes of a blob into host memory dst (ref src/codec.cpp:177-199 blob_to_bytes): the
// header is written here, the codebook and outliers are serialised on the device into the
// slot's pack buffer, and every device part goes out as an async copy on s. The caller
// synchronises s before reading dst (the batch entry point once, at the end).
int blob_to_host_enqueue(acz_gpu_ctx* ctx, Slot* sl, const acz_gpu_blob* b, uint8_t* dst,
                         uint64_t cap, cudaStream_t s) {
    const acz_gpu_blob_info_t& in = b->info;
    if (cap < in.compressed_bytes) return fail(ctx, ACZ_ERR_INVALID, "destination too small");
    if (!sl) return fail(ctx, ACZ_ERR_NOMEM, "slot");
    const uint32_t k = in.codebook_size;
    const uint64_t nout = in.outlier_count;
    uint8_t* p = dst;
    auto put = [&](uint64_t v, int bytes) {
        for (int i = 0; i < bytes; ++i) *p++ = (uint8_t)(v >> (8 * i));
    };
    std::memcpy(p, "ACZ1", 4);
    p += 4;
    put(1, 1);
    put(in.predictor, 1);
    put(in.rank, 1);
    for (uint32_t i = 0; i < in.rank; ++i) put(in.shape[i], 8);
    uint64_t ebits;
    std::memcpy(&ebits, &in.eb, 8);
    put(ebits, 8);
    put(in.quant_radius, 4);
    put(nout, 4);
    put(k, 2);
    uint8_t* book_at = p;
    p += 5ull * k;
    put(in.bit_length, 8);
    const uint64_t nbytes = (in.bit_length + 7) / 8;
    CK(cudaMemcpyAsync(p, b->words, nbytes, cudaMemcpyDeviceToHost, s));
    p += nbytes;
    uint8_t* outl_at = p;
    p += 12ull * nout;
    if ((uint64_t)(p - dst) != in.compressed_bytes)
        return fail(ctx, ACZ_ERR_FORMAT, "internal: ACZ1 size mismatch");
    if (k || nout) {
        const size_t need = 5ull * k + 12ull * nout;
        if (int rc = slot_enter(ctx, sl, s)) return rc;
        CK(grow(&sl->ws_pack, &sl->ws_pack_cap, need));
        uint8_t* pk = static_cast<uint8_t*>(sl->ws_pack);
        CK(launch_pack_acz1(b->book_sym, b->book_len, k, b->out_index, b->out_value, nout, pk,
                            pk + 5ull * k, ctx->sms, s, &ctx->launches));
        if (k) CK(cudaMemcpyAsync(book_at, pk, 5ull * k, cudaMemcpyDeviceToHost, s));
        if (nout) CK(cudaMemcpyAsync(outl_at, pk + 5ull * k, 12ull * nout, cudaMemcpyDeviceToHost, s));
        return slot_leave(ctx, sl, s);
    }
    return ACZ_OK;
}

// Decode sidecar ("ACZS" v3) into host memory dst, async on s (see blob_to_host_enqueue).
// The binding is computed on the device from the blob's codebook and bitstream.
int sidecar_to_host_enqueue(acz_gpu_ctx* ctx, Slot* sl, const acz_gpu_blob* b, uint8_t* dst,
                            uint64_t cap, cudaStream_t s) {
    const bool has_outl = b->side_outl != nullptr;
    const uint64_t need = sidecar_bytes(b->nchunks, has_outl);
    if (cap < need) return fail(ctx, ACZ_ERR_INVALID, "destination too small");
    uint8_t* p = dst;
    if (!sl) return fail(ctx, ACZ_ERR_NOMEM, "slot");
    if (int rc = ensure_small(ctx, sl)) return rc;
    if (int rc = slot_enter(ctx, sl, s)) return rc;
    std::memcpy(p, "ACZS", 4);
    p += 4;
    std::memcpy(p, &kSidecarVersion, 4);
    p += 4;
    const uint64_t hdr[6] = {b->info.element_count, b->info.bit_length, b->interval, b->nchunks,
                             0ull, has_outl ? 1ull : 0ull};
    std::memcpy(p, hdr, sizeof(hdr));
    CK(launch_blob_digest(b->book_sym, b->book_len, b->info.codebook_size,
                          reinterpret_cast<const uint8_t*>(b->words), (b->info.bit_length + 7) / 8,
                          blob_binding_h0(b->info), &sl->d_small->binding, s, &ctx->launches));
    CK(cudaMemcpyAsync(p + 4 * 8, &sl->d_small->binding, 8, cudaMemcpyDeviceToHost, s));
    p += sizeof(hdr);
    CK(cudaMemcpyAsync(p, b->side_bitoff, 8ull * b->nchunks, cudaMemcpyDeviceToHost, s));
    p += 8ull * b->nchunks;
    if (has_outl) {
        CK(cudaMemcpyAsync(p, b->side_outl, 4ull * b->nchunks, cudaMemcpyDeviceToHost, s));
        p += 4ull * b->nchunks;
    }
    CK(cudaMemcpyAsync(p, b->side_state, 4ull * b->nchunks, cudaMemcpyDeviceToHost, s));
    return slot_leave(ctx, sl, s);
}

constexpr size_t kPoolStreams = 8;

// Internal streams for the batched entry points, forked from the caller's stream: pool[i]
// (i < kPoolStreams) run at the device's lowest priority, pool[kPoolStreams + i] at the
// highest. A tensor whose quantiser is the long speculative kernel (the step's critical
// path) goes to a high-priority stream: its CTAs keep the SMs, and the other tensors'
// short kernels fill its tail and run alongside its histogram/codebook/encode (measured on
// AlexNet: 2.61 vs 2.87 ms per step with the priorities the other way round).
int pool_fork(acz_gpu_ctx* ctx, size_t k, cudaStream_t user) {
    if (ctx->pool.empty()) {
        int least = 0, greatest = 0;
        CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        for (size_t i = 0; i < 2 * kPoolStreams; ++i) {
            cudaStream_t st = nullptr;
            cudaEvent_t ev = nullptr;
            CK(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking,
                                            i < kPoolStreams ? least : greatest));
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            ctx->pool.push_back(st);
            ctx->pool_ev.push_back(ev);
        }
    }
    CK(cudaEventRecord(ctx->ev_fork, user));
    for (size_t i = 0; i < k; ++i) {
        CK(cudaStreamWaitEvent(ctx->pool[i], ctx->ev_fork, 0));
        CK(cudaStreamWaitEvent(ctx->pool[kPoolStreams + i], ctx->ev_fork, 0));
    }
    return ACZ_OK;
}

// Join: the caller's stream waits for the first k internal streams of both priorities.
int pool_join(acz_gpu_ctx* ctx, size_t k, cudaStream_t user) {
    for (size_t i = 0; i < k; ++i)
        for (size_t j : {i, kPoolStreams + i}) {
            CK(cudaEventRecord(ctx->pool_ev[j], ctx->pool[j]));
            CK(cudaStreamWaitEvent(user, ctx->pool_ev[j], 0));
        }
    return ACZ_OK;
}

// Stream of tensor i of a batch (see pool_fork).
cudaStream_t tensor_stream(acz_gpu_ctx* ctx, uint32_t i, size_t k, const uint64_t* shape,
                           uint32_t rank, uint32_t predictor) {
    const PlaneGeom g = plane_geom(shape, rank);
    const bool bulk = g.n && quant_spec_applicable(predictor, g.plane_size, g.planes, ctx->sms);
    return ctx->pool[(bulk ? kPoolStreams : 0) + i % k];
}

}  // namespace

extern "C" {

int acz_gpu_compress(acz_gpu_ctx* ctx, const float* d_in, const uint64_t* shape, uint32_t rank,
                     double eb, uint32_t quant_radius, uint32_t predictor, void* stream,
                     acz_gpu_blob** out) {
    return guarded(ctx, [&]() -> int {
    if (!ctx || !out) return ACZ_ERR_INVALID;
    *out = nullptr;
    ctx->err.clear();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Slot* sl = get_slot(ctx, 0);
    Plan pl;
    int rc = compress_begin(ctx, sl, d_in, shape, rank, eb, quant_radius, predictor, s, &pl);
    if (rc) return rc;
    return compress_end(ctx, sl, pl, s, out);
    });
}

// ---------------------------------------------------- asynchronous compress (hooks) --
// The training hooks compress one conv input at a time while the forward pass is still
// being enqueued; a host wait per layer for its codebook drains the GPU's queue every
// layer. acz_gpu_compress_async enqueues the whole compress (quantiser, histogram,
// codebook, encode) with no host wait, into a blob sized from the previous compress of the
// same (shape, eb, radius, predictor) -- the speculative encode of the batched path, whose
// kernels write nothing unless the book fits -- and a copy of the BookInfo into a mapped
// ring entry of the context, behind an event. acz_gpu_compress_settle later reads that
// entry: the blob is complete (bit-identical to acz_gpu_compress), or it did not fit and
// the caller compresses the tensor again synchronously.
struct AsyncHead {  // the leading fields of SmallBlock
    acz_b200::BookInfo info;
    unsigned int flags;
};
static_assert(offsetof(AsyncHead, flags) == offsetof(SmallBlock, flags),
              "AsyncHead must mirror SmallBlock's leading fields");
constexpr uint32_t kAsyncRing = 1024;
constexpr size_t kAsyncStride = (sizeof(AsyncHead) + 63) & ~size_t(63);

struct AsyncPending {
    acz_gpu_ctx* ctx = nullptr;
    uint32_t ring = 0;
    cudaEvent_t ev = nullptr;
    Plan pl;
    std::string key;
};

namespace {
void async_release(acz_gpu_blob* b) {
    AsyncPending* p = b->async;
    if (!p) return;
    // an unsettled blob being freed: its BookInfo copy may still be in flight, and the ring
    // entry must not be handed to another compress (possibly on another stream) before it
    // has landed
    if (p->ev) cudaEventSynchronize(p->ev);
    if (p->ev) cudaEventDestroy(p->ev);
    p->ctx->async_free.push_back(p->ring);
    delete p;
    b->async = nullptr;
}
}  // namespace

int acz_gpu_compress_async(acz_gpu_ctx* ctx, const float* d_in, const uint64_t* shape,
                           uint32_t rank, double eb, uint32_t quant_radius, uint32_t predictor,
                           uint64_t size_tag, void* stream, acz_gpu_blob** out, int* pending) {
    return guarded(ctx, [&]() -> int {
    if (!ctx || !out || !pending) return ACZ_ERR_INVALID;
    *out = nullptr;
    *pending = 0;
    ctx->err.clear();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Slot* sl = get_slot(ctx, 0);
    if (!sl) return fail(ctx, ACZ_ERR_NOMEM, "slot");
    Plan pl;
    int rc = compress_begin(ctx, sl, d_in, shape, rank, eb, quant_radius, predictor, s, &pl);
    if (rc) return rc;
    // the prediction comes from the last compress with the same parameters AND tag (the
    // controller tags by layer: layers with equal input shapes compress to different sizes)
    std::string key = size_key(pl);
    key.append(reinterpret_cast<const char*>(&size_tag), 8);
    auto it = ctx->size_cache.find(key);
    if (predictor == ACZ_PRED_PREV && it != ctx->size_cache.end()) {
        if (!ctx->async_host) {
            CK(cudaHostAlloc(&ctx->async_host, kAsyncStride * kAsyncRing, cudaHostAllocMapped));
            CK(cudaHostGetDevicePointer(&ctx->async_dev, ctx->async_host, 0));
            for (uint32_t i = kAsyncRing; i-- > 0;) ctx->async_free.push_back(i);
        }
        if (!ctx->async_free.empty()) {
            if ((rc = spec_encode(ctx, sl, &pl, it->second, s))) return rc;
            acz_gpu_blob* b = pl.spec;
            pl.spec = nullptr;
            AsyncPending* ap = new (std::nothrow) AsyncPending();
            cudaEvent_t ev = nullptr;
            cudaError_t e = ap ? cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)
                               : cudaErrorMemoryAllocation;
            const uint32_t ring = ctx->async_free.back();
            CopyRegions cr{};
            cr.src[0] = sl->d_small;
            cr.dst[0] = static_cast<char*>(ctx->async_dev) + kAsyncStride * ring;
            cr.bytes[0] = sizeof(AsyncHead);
            cr.n = 1;
            cr.to_host = 1;
            if (e == cudaSuccess) e = launch_copy_regions(cr, ctx->sms, s, &ctx->launches);
            if (e == cudaSuccess) e = cudaEventRecord(ev, s);
            if (e != cudaSuccess) {
                if (ev) cudaEventDestroy(ev);
                delete ap;
                blob_arena_free(b, s);
                delete b;
                return cuda_fail(ctx, e, "async compress");
            }
            ctx->async_free.pop_back();
            ap->ctx = ctx;
            ap->ring = ring;
            ap->ev = ev;
            ap->pl = pl;
            ap->key = key;
            b->async = ap;
            b->invalid = ACZ_ERR_INVALID;
            b->invalid_msg = "blob of an unsettled asynchronous compress";
            *out = b;
            *pending = 1;
            return ACZ_OK;
        }
    }
    rc = compress_end(ctx, sl, pl, s, out);
    if (rc == ACZ_OK && predictor == ACZ_PRED_PREV) {
        const acz_gpu_blob_info_t& in = (*out)->info;
        ctx->size_cache[key] = {in.codebook_size, in.bit_length, in.outlier_count,
                                in.max_code_length};
    }
    return rc;
    });
}

int acz_gpu_compress_settle(acz_gpu_ctx* ctx, acz_gpu_blob* b, int wait, int* state) {
    return guarded(ctx, [&]() -> int {
    if (!ctx || !b || !state) return ACZ_ERR_INVALID;
    ctx->err.clear();
    AsyncPending* ap = b->async;
    if (!ap) {
        *state = b->invalid ? ACZ_ASYNC_REFIT : ACZ_ASYNC_DONE;
        return ACZ_OK;
    }
    if (ap->ctx != ctx) return fail(ctx, ACZ_ERR_INVALID, "blob of another context");
    if (!wait) {
        const cudaError_t q = cudaEventQuery(ap->ev);
        if (q == cudaErrorNotReady) {
            *state = ACZ_ASYNC_PENDING;
            return ACZ_OK;
        }
        if (q != cudaSuccess) return cuda_fail(ctx, q, "async settle");
    }
    CK(cudaEventSynchronize(ap->ev));
    AsyncHead h;
    std::memcpy(&h, static_cast<const char*>(ctx->async_host) + kAsyncStride * ap->ring,
                sizeof(AsyncHead));
    const BookInfo& bi = h.info;
    const Plan& pl = ap->pl;
    const unsigned flags = h.flags | bi.flags;
    const bool fits = !flags && !bi.slow && bi.book_size >= 1 && bi.total_bits <= pl.cap_bits &&
                      bi.n_escapes <= pl.cap_out && bi.book_size <= pl.cap_book &&
                      bi.max_len <= pl.cap_len;
    if (!flags && !bi.slow && bi.book_size >= 1)  // the next prediction: this book's sizes
        ctx->size_cache[ap->key] = {bi.book_size, bi.total_bits, bi.n_escapes, bi.max_len};
    if (fits) {
        b->nwords = (bi.total_bits + 31) / 32;
        b->max_len = bi.max_len;
        acz_gpu_blob_info_t& in = b->info;
        in.rank = pl.rank;
        for (uint32_t i = 0; i < pl.rank; ++i) in.shape[i] = pl.shape[i];
        in.eb = pl.eb;
        in.quant_radius = pl.radius;
        in.predictor = pl.predictor;
        in.element_count = pl.n;
        in.codebook_size = bi.book_size;
        in.bit_length = bi.total_bits;
        in.outlier_count = bi.n_escapes;
        in.uncompressed_bytes = 4ull * pl.n;
        in.compressed_bytes = acz1_size(pl.rank, bi.book_size, bi.total_bits, bi.n_escapes);
        in.device_bytes = b->arena_bytes;
        in.sidecar_bytes = sidecar_bytes(b->nchunks, false);
        in.max_code_length = bi.max_len;
        b->invalid = 0;
        b->invalid_msg.clear();
    }
    async_release(b);
    *state = fits ? ACZ_ASYNC_DONE : ACZ_ASYNC_REFIT;
    if (!fits) {  // why (acz_gpu_last_error; not an error)
        char why[160];
        std::snprintf(why, sizeof why,
                      "refit: flags %u slow %u book %u/%u bits %llu/%llu outliers %llu/%llu "
                      "len %u/%u", flags, (unsigned)bi.slow, bi.book_size, pl.cap_book,
                      (unsigned long long)bi.total_bits, (unsigned long long)pl.cap_bits,
                      (unsigned long long)bi.n_escapes, (unsigned long long)pl.cap_out,
                      bi.max_len, pl.cap_len);
        ctx->err = why;
    }
    return check_sticky(ctx);
    });
}

int acz_gpu_compress_batch(acz_gpu_ctx* ctx, uint32_t count, const float* const* d_in,
                           const uint64_t* shapes, const uint32_t* ranks, double eb,
                           uint32_t quant_radius, uint32_t predictor, void* stream,
                           acz_gpu_blob** out, int* status) {
    return guarded(ctx, [&]() -> int {
    if (!ctx || !out || (count && (!d_in || !shapes || !ranks))) return ACZ_ERR_INVALID;
    ctx->err.clear();
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    for (uint32_t i = 0; i < count; ++i) {
        out[i] = nullptr;
        if (status) status[i] = ACZ_OK;
    }
    if (count == 0) return ACZ_OK;
    const size_t k = std::min<size_t>(count, kPoolStreams);
    int rc = pool_fork(ctx, k, user);
    if (rc) return rc;
    std::vector<Plan> plans(count);
    std::vector<int> st(count, ACZ_OK);
    std::vector<size_t> off(count);
    std::vector<cudaStream_t> ts(count);
    size_t o = 0;
    for (uint32_t i = 0; i < count; ++i) {
        off[i] = o;
        o += ranks[i];
        ts[i] = tensor_stream(ctx, i, k, shapes + off[i], ranks[i], predictor);
    }
    // first halves: every tensor's quantiser/histogram/codebook, round-robin over streams
    for (uint32_t i = 0; i < count; ++i) {
        Slot* sl = get_slot(ctx, i);
        if (!sl) {
            st[i] = ACZ_ERR_NOMEM;
            continue;
        }
        st[i] = compress_begin(ctx, sl, d_in[i], shapes + off[i], ranks[i], eb, quant_radius,
                               predictor, ts[i], &plans[i]);
        if (st[i] == ACZ_OK && predictor == ACZ_PRED_PREV && spec_encode_enabled()) {
            auto it = ctx->size_cache.find(size_key(plans[i]));
            if (it != ctx->size_cache.end()) st[i] = spec_encode(ctx, sl, &plans[i], it->second, ts[i]);
        }
    }
    // second halves in completion order: a tensor's encode is launched as soon as its own
    // codebook read-back has landed, so short tensors do not queue behind a long quantiser
    int first_err = ACZ_OK;
    std::string first_msg;
    std::vector<char> done(count, 0);
    uint32_t remaining = count;
    auto finish = [&](uint32_t i) {
        if (st[i] == ACZ_OK) {
            Slot* sl = get_slot(ctx, i);
            st[i] = plans[i].spec ? spec_finish(ctx, sl, plans[i], ts[i], &out[i])
                                  : compress_end(ctx, sl, plans[i], ts[i], &out[i]);
            if (st[i] == ACZ_OK && predictor == ACZ_PRED_PREV) {
                const acz_gpu_blob_info_t& in = out[i]->info;
                ctx->size_cache[size_key(plans[i])] = {in.codebook_size, in.bit_length,
                                                       in.outlier_count, in.max_code_length};
            }
        }
        if (st[i] != ACZ_OK && first_err == ACZ_OK) {
            first_err = st[i];
            first_msg = ctx->err;
        }
        if (status) status[i] = st[i];
        done[i] = 1;
        --remaining;
    };
    // Poll in priority order (tensors on the high-priority stream first: their encode is on
    // the critical path) and rescan from the top after every finish, so a critical tensor
    // whose codebook lands while others are being finished waits for at most one of them.
    std::vector<uint32_t> prio(count);
    for (uint32_t i = 0; i < count; ++i) prio[i] = i;
    std::stable_partition(prio.begin(), prio.end(), [&](uint32_t i) {
        return ts[i] != ctx->pool[i % k];  // on a high-priority stream
    });
    while (remaining) {
        bool progressed = false;
        for (uint32_t i : prio) {
            if (done[i]) continue;
            if (st[i] != ACZ_OK || cudaEventQuery(get_slot(ctx, i)->ev_book) != cudaErrorNotReady) {
                finish(i);
                progressed = true;
                break;
            }
        }
        // nothing ready: poll again (blocking on one tensor would hold back the others, whose
        // completion order depends on the stream priorities and the scheduler)
        if (!progressed) std::this_thread::yield();
    }
    rc = pool_join(ctx, k, user);
    if (rc) return rc;
    if (first_err) ctx->err = first_msg;
    return first_err;
    });
}

int acz_gpu_compress_host_batch(acz_gpu_ctx* ctx, uint32_t count, const float* const* h_in,
                                const uint64_t* shapes, const uint32_t* ranks, double eb,
                                uint32_t quant_radius, uint32_t predictor, uint8_t* const* acz1,
                                const uint64_t* acz1_cap, uint64_t* acz1_size,
                                uint8_t* const* sidecar, const uint64_t* sidecar_cap,
                                uint64_t* sidecar_size, int* status) {
    return guarded(ctx, [&]() -> int {
    if (!ctx || (count && (!h_in || !shapes || !ranks || !acz1 || !acz1_cap || !acz1_size)))
        return ACZ_ERR_INVALID;
    ctx->err.clear();
    if (count == 0) return ACZ_OK;
    const size_t k = std::min<size_t>(count, kPoolStreams);
    int rc = pool_fork(ctx, k, ctx->own);
    if (rc) return rc;
    std::vector<Plan> plans(count);
    std::vector<int> st(count, ACZ_OK);
    std::vector<const uint64_t*> shp(count);
    std::vector<uint64_t> nel(count, 0);
    std::vector<cudaStream_t> ts(count);
    for (uint32_t i = 0, o = 0; i < count; o += ranks[i], ++i) {
        shp[i] = shapes + o;
        st[i] = validate_shape(ctx, shp[i], ranks[i], &nel[i]);
        ts[i] = st[i] == ACZ_OK ? tensor_stream(ctx, i, k, shp[i], ranks[i], predictor)
                                : ctx->pool[i % k];
    }
    // Uploads go one at a time, largest tensor first (an event chain across the pool
    // streams): concurrent copies would share PCIe and all land together at the end, while
    // in sequence the big tensor's kernels run under the remaining uploads and the tail after
    // the last upload is the smallest tensor's work. Each tensor's kernels start on its own
    // stream as soon as its own input has landed.
    std::vector<uint32_t> order(count);
    for (uint32_t i = 0; i < count; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(),
                     [&](uint32_t a, uint32_t b) { return nel[a] > nel[b]; });
    cudaEvent_t prev_up = nullptr;
    for (uint32_t i : order) {
        Slot* sl = get_slot(ctx, i);
        cudaStream_t s = ts[i];
        const uint64_t n = nel[i];
        if (!sl) st[i] = ACZ_ERR_NOMEM;
        if (st[i] == ACZ_OK) st[i] = ensure_small(ctx, sl);
        if (st[i] == ACZ_OK && n) {
            cudaError_t e = grow(&sl->ws_in, &sl->ws_in_cap, 4ull * n);
            if (e == cudaSuccess && prev_up) e = cudaStreamWaitEvent(s, prev_up, 0);
            if (e == cudaSuccess) e = cudaMemcpyAsync(sl->ws_in, h_in[i], 4ull * n,
                                                      cudaMemcpyHostToDevice, s);
            if (e == cudaSuccess) e = cudaEventRecord(sl->ev_up, s);
            if (e != cudaSuccess) st[i] = cuda_fail(ctx, e, "host input upload");
            else prev_up = sl->ev_up;
        }
        if (st[i] == ACZ_OK)
            st[i] = compress_begin(ctx, sl, static_cast<const float*>(sl->ws_in), shp[i], ranks[i],
                                   eb, quant_radius, predictor, s, &plans[i]);
    }
    // second halves in completion order, then the bytes back to the host
    int first_err = ACZ_OK;
    std::string first_msg;
    std::vector<char> done(count, 0);
    uint32_t remaining = count;
    auto finish = [&](uint32_t i) {
        cudaStream_t s = ts[i];
        acz_gpu_blob* b = nullptr;
        if (st[i] == ACZ_OK) st[i] = compress_end(ctx, get_slot(ctx, i), plans[i], s, &b);
        if (st[i] == ACZ_OK) {
            acz1_size[i] = b->info.compressed_bytes;  // the needed size, also on failure
            if (sidecar_size) sidecar_size[i] = b->info.sidecar_bytes;
            if (acz1_cap[i] < b->info.compressed_bytes)
                st[i] = fail(ctx, ACZ_ERR_INVALID, "ACZ1 destination too small");
            else
                st[i] = blob_to_host_enqueue(ctx, get_slot(ctx, i), b, acz1[i], acz1_cap[i], s);
            if (st[i] == ACZ_OK) acz1_size[i] = b->info.compressed_bytes;
        }
        if (st[i] == ACZ_OK && sidecar && sidecar[i]) {
            if (!sidecar_cap || sidecar_cap[i] < b->info.sidecar_bytes)
                st[i] = fail(ctx, ACZ_ERR_INVALID, "sidecar destination too small");
            else
                st[i] = sidecar_to_host_enqueue(ctx, get_slot(ctx, i), b, sidecar[i],
                                                sidecar_cap[i], s);
            if (st[i] == ACZ_OK && sidecar_size) sidecar_size[i] = b->info.sidecar_bytes;
        }
        if (b) acz_gpu_blob_free(b);  // stream-ordered: the copies above complete first
        if (st[i] != ACZ_OK && first_err == ACZ_OK) {
            first_err = st[i];
            first_msg = ctx->err;
        }
        if (status) status[i] = st[i];
        done[i] = 1;
        --remaining;
    };
    std::vector<uint32_t> prio(count);
    for (uint32_t i = 0; i < count; ++i) prio[i] = i;
    std::stable_partition(prio.begin(), prio.end(),
                          [&](uint32_t i) { return ts[i] != ctx->pool[i % k]; });
    while (remaining) {  // see acz_gpu_compress_batch
        bool progressed = false;
        for (uint32_t i : prio) {
            if (done[i]) continue;
            if (st[i] != ACZ_OK || cudaEventQuery(get_slot(ctx, i)->ev_book) != cudaErrorNotReady) {
                finish(i);
                progressed = true;
                break;
            }
        }
        if (!progressed) std::this_thread::yield();
    }
    rc = pool_join(ctx, k, ctx->own);
    if (rc) return rc;
    CK(cudaStreamSynchronize(ctx->own));  // every ACZ1 / sidecar byte is in host memory
    if (first_err) ctx->err = first_msg;
    if (!first_err) first_err = check_sticky(ctx);
    return first_err;
    });
}

int acz_gpu_decompress_batch(acz_gpu_ctx* ctx, uint32_t count, const acz_gpu_blob* const* blobs,
                             int zero_filter, float* const* d_out, void* stream) {
    return guarded(ctx, [&]() -> int {
    if (!ctx || (count && (!blobs || !d_out))) return ACZ_ERR_INVALID;
    ctx->err.clear();
    if (count == 0) return ACZ_OK;
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    const size_t k = std::min<size_t>(count, kPoolStreams);
    int rc = pool_fork(ctx, k, user);
    if (rc) return rc;
    int first_err = ACZ_OK;
    for (uint32_t i = 0; i < count; ++i) {
        rc = decompress_on(ctx, get_slot(ctx, i), blobs[i], zero_filter, d_out[i],
                           ctx->pool[i % k]);
        if (rc && first_err == ACZ_OK) first_err = rc;
    }
    rc = pool_join(ctx, k, user);
    if (rc) return rc;
    return first_err;
    });
}

int acz_gpu_decompress(acz_gpu_ctx* ctx, const acz_gpu_blob* b, int zero_filter, float* d_out,
                       void* stream) {
    return guarded(ctx, [&]() -> int {
    if (!ctx || !b || !d_out) return ACZ_ERR_INVALID;
    ctx->err.clear();
    return decompress_on(ctx, get_slot(ctx, 0), b, zero_filter, d_out,
                         static_cast<cudaStream_t>(stream));
    });
}

int acz_gpu_blob_info(const acz_gpu_blob* b, acz_gpu_blob_info_t* info) {
    if (!b || !info) return ACZ_ERR_INVALID;
    *info = b->info;
    return ACZ_OK;
}

int acz_gpu_blob_free(acz_gpu_blob* b) {
    if (!b) return ACZ_ERR_INVALID;
    async_release(b);
    blob_arena_free(b, b->stream);
    delete b;
    return ACZ_OK;
}

// ------------------------------------------------------------------ serialisation --
int acz_gpu_blob_to_host(acz_gpu_ctx* ctx, const acz_gpu_blob* b, uint8_t* dst, uint64_t cap,
                         uint64_t* written, void* stream) {
    return guarded(ctx, [&]() -> int {
    if (!ctx || !b || !dst) return ACZ_ERR_INVALID;
    ctx->err.clear();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int rc = blob_to_host_enqueue(ctx, get_slot(ctx, 0), b, dst, cap, s);
    if (rc) return rc;
    CK(cudaStreamSynchronize(s));
    if (int sr = check_sticky(ctx)) return sr;
    if (written) *written = b->info.compressed_bytes;
    return ACZ_OK;
    });
}

int acz_gpu_sidecar_to_host(acz_gpu_ctx* ctx, const acz_gpu_blob* b, uint8_t* dst, uint64_t cap,
                            uint64_t* written, void* stream) {
    return guarded(ctx, [&]() -> int {
    if (!ctx || !b || !dst) return ACZ_ERR_INVALID;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int rc = sidecar_to_host_enqueue(ctx, get_slot(ctx, 0), b, dst, cap, s);
    if (rc) return rc;
    CK(cudaStreamSynchronize(s));
    if (written) *written = sidecar_bytes(b->nchunks, b->side_outl != nullptr);
    return ACZ_OK;
    });
}

// Sidecar arrays the decoders index with (bit offsets, outlier prefixes) must be in range:
// offsets start at 0, never decrease, advance at most 64 bits per symbol and stay within the
// stream; prefixes start at 0, never decrease and stay within the outlier list; chain states
// are finite (reference chain values always are). Anything else falls back to the rebuild.
bool sidecar_arrays_ok(const uint8_t* p, uint64_t nchunks, uint64_t interval, bool has_outl,
                       uint64_t bit_length, uint64_t nout) {
    uint64_t prev = 0;
    for (uint64_t c = 0; c < nchunks; ++c) {
        uint64_t v;
        std::memcpy(&v, p + 8 * c, 8);
        if ((c == 0 && v != 0) || v < prev || v > bit_length || v - prev > 64 * interval)
            return false;
        prev = v;
    }
    p += 8 * nchunks;
    if (has_outl) {
        uint32_t po = 0;
        for (uint64_t c = 0; c < nchunks; ++c) {
            uint32_t v;
            std::memcpy(&v, p + 4 * c, 4);
            if ((c == 0 && v != 0) || v < po || v > nout) return false;
            po = v;
        }
        p += 4 * nchunks;
    }
    for (uint64_t c = 0; c < nchunks; ++c) {
        float f;
        std::memcpy(&f, p + 4 * c, 4);
        if (!std::isfinite(f)) return false;
    }
    return true;
}

// ACZ1 bytes (+ optional ACZS sidecar) in host memory -> device blob on stream s, with the
// reference's blob_from_bytes checks on the host. The bitstream, the raw codebook/outlier
// sections and the sidecar are copied straight from the caller's buffers (async when they
// are page-locked); the codebook and outliers are de-interleaved on the device. async: do
// not synchronise s when a valid sidecar was supplied (the caller keeps src/sidecar alive
// and orders its own work after s).
static int blob_from_host_body(acz_gpu_ctx* ctx, Slot* sl, const uint8_t* src, uint64_t size,
                               const uint8_t* sidecar, uint64_t sidecar_size, cudaStream_t s,
                               acz_gpu_blob** out, bool async) {
    if (!ctx || !out || (!src && size)) return ACZ_ERR_INVALID;
    if (!sl) return fail(ctx, ACZ_ERR_NOMEM, "slot");
    *out = nullptr;
    {
        const int rc = ensure_small(ctx, sl);
        if (rc) return rc;
    }
    // ---- ref src/codec.cpp:201-262 (blob_from_bytes), same checks and order ----
    uint64_t pos = 0;
    bool trunc = false;
    auto get = [&](int bytes) -> uint64_t {
        if (trunc || pos + (uint64_t)bytes > size) {
            trunc = true;
            return 0;
        }
        uint64_t v = 0;
        for (int i = 0; i < bytes; ++i) v |= (uint64_t)src[pos + i] << (8 * i);
        pos += (uint64_t)bytes;
        return v;
    };
#define NEED()                                                                       \
    do {                                                                             \
        if (trunc) return fail(ctx, ACZ_ERR_FORMAT, "unexpected end of stream");     \
    } while (0)
    if (size < 4) return fail(ctx, ACZ_ERR_FORMAT, "unexpected end of stream at offset 0");
    if (std::memcmp(src, "ACZ1", 4) != 0)
        return fail(ctx, ACZ_ERR_FORMAT, "bad blob magic at offset 0 (expected \"ACZ1\")");
    pos = 4;
    const uint64_t version = get(1);
    NEED();
    if (version != 1) return fail(ctx, ACZ_ERR_FORMAT, "unsupported blob version");
    const uint64_t pred = get(1);
    NEED();
    if (pred > 1) return fail(ctx, ACZ_ERR_FORMAT, "unknown predictor id");
    const uint64_t rank = get(1);
    NEED();
    if (rank == 0) return fail(ctx, ACZ_ERR_FORMAT, "blob rank must be >= 1");
    if (rank > ACZ_MAX_RANK) return fail(ctx, ACZ_ERR_FORMAT, "blob rank exceeds ACZ_MAX_RANK");
    acz_gpu_blob_info_t in{};
    in.rank = (uint32_t)rank;
    in.predictor = (uint32_t)pred;
    uint64_t count = 1;
    for (uint64_t i = 0; i < rank; ++i) {
        in.shape[i] = get(8);
        NEED();
        if (in.shape[i] == 0) return fail(ctx, ACZ_ERR_FORMAT, "zero extent in blob header");
        count *= in.shape[i];
    }
    const uint64_t ebits = get(8);
    in.quant_radius = (uint32_t)get(4);
    NEED();
    std::memcpy(&in.eb, &ebits, 8);
    if (!params_ok(in.eb, in.quant_radius)) return fail(ctx, ACZ_ERR_PARAM, param_msg(in.eb));
    const uint64_t nout = get(4);
    const uint64_t k = get(2);
    NEED();
    if (k == 0) return fail(ctx, ACZ_ERR_FORMAT, "empty codebook");
    const uint64_t book_off = pos;
    std::vector<uint32_t> bsym(k);
    std::vector<uint8_t> blen(k);
    for (uint64_t i = 0; i < k; ++i) {
        bsym[i] = (uint32_t)get(4);
        blen[i] = (uint8_t)get(1);
    }
    const uint64_t bit_length = get(8);
    NEED();
    const uint64_t nbytes = bit_length / 8 + ((bit_length & 7) ? 1 : 0);
    if (nbytes > size - pos) return fail(ctx, ACZ_ERR_FORMAT, "unexpected end of stream");
    const uint8_t* bits = src + pos;
    pos += nbytes;
    const uint64_t outl_off = pos;
    // the count is untrusted: parse record by record (the reference's error order), but
    // never allocate for more records than the remaining bytes can hold
    const uint64_t nfit = std::min<uint64_t>(nout, (size - pos) / 12 + 1);
    std::vector<unsigned long long> oidx(nfit);
    std::vector<float> oval(nfit);
    for (uint64_t i = 0; i < nout; ++i) {
        if (i >= nfit) return fail(ctx, ACZ_ERR_FORMAT, "unexpected end of stream");
        oidx[i] = get(8);
        const uint32_t vb = (uint32_t)get(4);
        NEED();
        std::memcpy(&oval[i], &vb, 4);
        if (oidx[i] >= count) return fail(ctx, ACZ_ERR_FORMAT, "outlier index out of range");
        if (i > 0 && oidx[i] <= oidx[i - 1])
            return fail(ctx, ACZ_ERR_FORMAT, "outlier indices are not strictly increasing");
    }
    if (pos != size) return fail(ctx, ACZ_ERR_FORMAT, "trailing bytes after blob");
#undef NEED
    in.element_count = count;
    in.codebook_size = (uint32_t)k;
    in.bit_length = bit_length;
    in.outlier_count = nout;
    in.uncompressed_bytes = 4ull * count;
    in.compressed_bytes = size;
    uint32_t maxl = 0;
    for (uint64_t i = 0; i < k; ++i) maxl = std::max<uint32_t>(maxl, blen[i]);
    in.max_code_length = maxl;

    // deferred (decompress-time) checks of the reference: huffman_decode book validation
    int deferred = 0;
    std::string dmsg;
    for (uint64_t i = 1; i < k && !deferred; ++i)
        if (blen[i - 1] > blen[i] || (blen[i - 1] == blen[i] && bsym[i - 1] >= bsym[i])) {
            deferred = ACZ_ERR_DECODE;
            dmsg = "codebook entries are not in canonical order";
        }
    for (uint64_t i = 0; i < k && !deferred; ++i)
        if (blen[i] == 0 || blen[i] > 64) {
            deferred = ACZ_ERR_DECODE;
            dmsg = "invalid code length in codebook";
        }
    const PlaneGeom g = plane_geom(in.shape, in.rank);
    const uint64_t interval = sidecar_interval_for((uint32_t)pred, g);
    // sidecar supplied?
    bool have_side = false;
    uint64_t side_interval = interval, side_chunks = (count + interval - 1) / interval;
    const bool want_outl = pred == ACZ_PRED_LORENZO2D;
    uint32_t sver = 0;
    if (sidecar && sidecar_size >= 56) std::memcpy(&sver, sidecar + 4, 4);
    if (sidecar && sidecar_size >= 56 && std::memcmp(sidecar, "ACZS", 4) == 0 &&
        sver == kSidecarVersion) {
        uint64_t hdr[6];
        std::memcpy(hdr, sidecar + 8, sizeof(hdr));
        if (hdr[0] == count && hdr[1] == bit_length && hdr[2] > 0 &&
            (pred != ACZ_PRED_PREV || (hdr[2] % 32 == 0 && (hdr[2] & (hdr[2] - 1)) == 0)) &&
            hdr[3] == (count + hdr[2] - 1) / hdr[2] && hdr[5] == (want_outl ? 1ull : 0ull) &&
            sidecar_size == sidecar_bytes(hdr[3], want_outl) &&
            (pred == ACZ_PRED_PREV || hdr[2] == sidecar_interval_for((uint32_t)pred, g))) {
            uint64_t book_sum = 0;
            for (uint64_t i = 0; i < k; ++i) book_sum += acz_book_term(bsym[i], blen[i], i);
            const uint64_t want = acz_binding(blob_binding_h0(in), book_sum,
                                              acz_bits_digest(bits, nbytes));
            if (hdr[4] == want && sidecar_arrays_ok(sidecar + 56, hdr[3], hdr[2], want_outl,
                                                    bit_length, nout)) {
                have_side = true;
                side_interval = hdr[2];
                side_chunks = hdr[3];
            }
        }
    }
    acz_gpu_blob* b = new (std::nothrow) acz_gpu_blob();
    if (!b) return fail(ctx, ACZ_ERR_NOMEM, "blob");
    b->info = in;
    const uint64_t nwords = (bit_length + 31) / 32;
    cudaError_t e = blob_alloc(b, (uint32_t)k, nwords, nout, side_chunks, want_outl, s);
    if (e != cudaSuccess) {
        delete b;
        return cuda_fail(ctx, e, "blob_alloc");
    }
    b->nwords = nwords;
    b->interval = side_interval;
    b->nchunks = side_chunks;
    b->max_len = maxl;
    b->info.device_bytes = b->arena_bytes;
    b->info.sidecar_bytes = sidecar_bytes(side_chunks, want_outl);
    auto cleanup = [&](int rc) {
        blob_arena_free(b, s);
        delete b;
        return rc;
    };
#define CKB(expr)                                                                  \
    do {                                                                           \
        cudaError_t _e = (expr);                                                   \
        if (_e != cudaSuccess) return cleanup(cuda_fail(ctx, _e, #expr));          \
    } while (0)
    // the bitstream's byte image == the words array; zero only the tail and the padding
    CKB(cudaMemsetAsync(reinterpret_cast<uint8_t*>(b->words) + nbytes, 0,
                        4ull * (nwords + 32) - nbytes, s));
    CKB(cudaMemcpyAsync(b->words, bits, nbytes, cudaMemcpyHostToDevice, s));
    {
        const size_t raw = 5ull * k + 12ull * nout;
        CKB(grow(&sl->ws_pack, &sl->ws_pack_cap, raw));
        uint8_t* rp = static_cast<uint8_t*>(sl->ws_pack);
        CKB(cudaMemcpyAsync(rp, src + book_off, 5ull * k, cudaMemcpyHostToDevice, s));
        if (nout) CKB(cudaMemcpyAsync(rp + 5ull * k, src + outl_off, 12ull * nout,
                                      cudaMemcpyHostToDevice, s));
        CKB(launch_unpack_acz1(rp, (uint32_t)k, nout, b->book_sym, b->book_len, b->out_index,
                               b->out_value, ctx->sms, s, &ctx->launches));
    }
    if (deferred) {
        CKB(cudaStreamSynchronize(s));
        b->invalid = deferred;
        b->invalid_msg = dmsg;
        *out = b;
        return ACZ_OK;
    }
    CKB(launch_build_tables(b->book_sym, b->book_len, (uint32_t)k, b->canon, b->lut, nullptr, s,
                            &ctx->launches));
    if (have_side) {
        const uint8_t* p = sidecar + 56;
        CKB(cudaMemcpyAsync(b->side_bitoff, p, 8ull * side_chunks, cudaMemcpyHostToDevice, s));
        p += 8ull * side_chunks;
        if (want_outl) {
            CKB(cudaMemcpyAsync(b->side_outl, p, 4ull * side_chunks, cudaMemcpyHostToDevice, s));
            p += 4ull * side_chunks;
        }
        CKB(cudaMemcpyAsync(b->side_state, p, 4ull * side_chunks, cudaMemcpyHostToDevice, s));
        if (!async) CKB(cudaStreamSynchronize(s));  // the caller may release src / sidecar
        *out = b;
        return ACZ_OK;
    }
    // rebuild the sidecar on the GPU: sequential decode + validation, then chain states
    const bool prev = pred == ACZ_PRED_PREV;
    const size_t aux = (prev ? 4ull * count : 0) + 8ull * (g.planes + 1) + 256;
    CKB(grow(&ctx->ws_aux, &ctx->ws_aux_cap, aux));
    unsigned long long* plane_outl = static_cast<unsigned long long*>(ctx->ws_aux);
    uint32_t* syms = prev ? reinterpret_cast<uint32_t*>(plane_outl + g.planes + 1) : nullptr;
    CKB(cudaMemsetAsync(&sl->d_small->flags, 0, sizeof(unsigned), s));
    ScanArgs sa;
    sa.words = b->words;
    sa.nwords = nwords;
    sa.bit_length = bit_length;
    sa.n = count;
    sa.lut = b->lut;
    sa.canon = b->canon;
    sa.book_sym = b->book_sym;
    sa.out_index = b->out_index;
    sa.n_outliers = nout;
    sa.interval = side_interval;
    sa.side_bitoff = b->side_bitoff;
    sa.side_outl = b->side_outl;
    sa.sym_out = syms;
    sa.plane_outl = plane_outl;
    sa.plane_size = g.plane_size;
    sa.flags = &sl->d_small->flags;
    {
        KTimer kt(ctx, ACZ_K_SCAN, s);
        CKB(grow(&ctx->ws_scan, &ctx->ws_scan_cap, scan_decode_scratch_bytes(bit_length)));
        CKB(launch_scan_decode(sa, ctx->ws_scan, s, &ctx->launches));
    }
    CKB(cudaMemcpyAsync(&sl->h_small->flags, &sl->d_small->flags, sizeof(unsigned),
                        cudaMemcpyDeviceToHost, s));
    CKB(cudaStreamSynchronize(s));
    const unsigned fl = sl->h_small->flags;
    if (fl) {
        b->invalid = (fl & (kDecTruncated | kDecNoMatch)) ? ACZ_ERR_DECODE : ACZ_ERR_FORMAT;
        b->invalid_msg = (fl & kDecTruncated)        ? "truncated bitstream"
                         : (fl & kDecNoMatch)        ? "no codeword matches bitstream"
                         : (fl & kDecOutlierMissing) ? "escape symbol without a matching outlier record"
                         : (fl & kDecOutlierIndex)   ? "outlier index does not match scan position"
                                                     : "blob contains unused outlier records";
        *out = b;
        return ACZ_OK;
    }
    if (prev) {
        CKB(launch_chain_states(syms, plane_outl, b->out_value, g, 2.0 * in.eb, in.quant_radius,
                                side_interval, b->side_state, ctx->sms, s, &ctx->launches));
    }
    CKB(cudaStreamSynchronize(s));
#undef CKB
    *out = b;
    return ACZ_OK;
}

static int blob_from_host_on(acz_gpu_ctx* ctx, Slot* sl, const uint8_t* src, uint64_t size,
                             const uint8_t* sidecar, uint64_t sidecar_size, cudaStream_t s,
                             acz_gpu_blob** out, bool async) {
    if (!ctx || !out || (!src && size)) return ACZ_ERR_INVALID;
    if (!sl) return fail(ctx, ACZ_ERR_NOMEM, "slot");
    if (int rc = ensure_small(ctx, sl)) return rc;
    if (int rc = slot_enter(ctx, sl, s)) return rc;
    const int rc = blob_from_host_body(ctx, sl, src, size, sidecar, sidecar_size, s, out, async);
    const int lr = slot_leave(ctx, sl, s);
    return rc ? rc : lr;
}

extern "C" int acz_gpu_blob_from_host(acz_gpu_ctx* ctx, const uint8_t* src, uint64_t size,
                                      const uint8_t* sidecar, uint64_t sidecar_size, void* stream,
                                      acz_gpu_blob** out) {
    return guarded(ctx, [&]() -> int {
    if (!ctx || !out || (!src && size)) return ACZ_ERR_INVALID;
    ctx->err.clear();
    return blob_from_host_on(ctx, get_slot(ctx, 0), src, size, sidecar, sidecar_size,
                             static_cast<cudaStream_t>(stream), out, false);
    });
}

int acz_gpu_decompress_host_batch(acz_gpu_ctx* ctx, uint32_t count, const uint8_t* const* acz1,
                                  const uint64_t* acz1_size, const uint8_t* const* sidecar,
                                  const uint64_t* sidecar_size, int zero_filter,
                                  float* const* h_out, const uint64_t* out_cap, int* status) {
    return guarded(ctx, [&]() -> int {
    if (!ctx || (count && (!acz1 || !acz1_size || !h_out || !out_cap))) return ACZ_ERR_INVALID;
    ctx->err.clear();
    if (count == 0) return ACZ_OK;
    const size_t k = std::min<size_t>(count, kPoolStreams);
    int rc = pool_fork(ctx, k, ctx->own);
    if (rc) return rc;
    if (!ctx->io_up) {
        CK(cudaStreamCreateWithFlags(&ctx->io_up, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&ctx->io_down, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ctx->io_ev, cudaEventDisableTiming));
    }
    CK(cudaStreamWaitEvent(ctx->io_up, ctx->ev_fork, 0));
    CK(cudaStreamWaitEvent(ctx->io_down, ctx->ev_fork, 0));
    // smallest blob first: the download stream (the bound: outputs are ~3x the blobs) starts
    // after one short upload + decode and then stays fed while the larger blobs upload
    std::vector<uint32_t> order(count);
    for (uint32_t i = 0; i < count; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(),
                     [&](uint32_t a, uint32_t b) { return acz1_size[a] < acz1_size[b]; });
    int first_err = ACZ_OK;
    std::string first_msg;
    for (uint32_t i : order) {
        Slot* sl = get_slot(ctx, i);
        cudaStream_t s = ctx->pool[i % k];
        acz_gpu_blob* b = nullptr;
        int st = sl ? ACZ_OK : ACZ_ERR_NOMEM;
        if (st == ACZ_OK)
            st = blob_from_host_on(ctx, sl, acz1[i], acz1_size[i], sidecar ? sidecar[i] : nullptr,
                                   sidecar && sidecar_size ? sidecar_size[i] : 0, ctx->io_up, &b,
                                   true);
        uint64_t n = 0;
        if (st == ACZ_OK) {
            n = b->info.element_count;
            if (out_cap[i] < n) st = fail(ctx, ACZ_ERR_SHAPE, "output buffer too small for the blob");
        }
        if (st == ACZ_OK) {
            cudaError_t e = cudaEventRecord(sl->ev_up, ctx->io_up);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(s, sl->ev_up, 0);
            if (e == cudaSuccess) e = grow(&sl->ws_in, &sl->ws_in_cap, 4ull * n);
            st = e == cudaSuccess ? ACZ_OK : cuda_fail(ctx, e, "host batch decompress");
        }
        if (st == ACZ_OK)
            st = decompress_on(ctx, sl, b, zero_filter, static_cast<float*>(sl->ws_in), s);
        if (st == ACZ_OK) {
            cudaError_t e = cudaEventRecord(sl->ev_dec, s);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->io_down, sl->ev_dec, 0);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(h_out[i], sl->ws_in, 4ull * n, cudaMemcpyDeviceToHost,
                                    ctx->io_down);
            if (e != cudaSuccess) st = cuda_fail(ctx, e, "host batch download");
        }
        if (b) {
            b->stream = s;  // freed after its decode (stream order on s)
            acz_gpu_blob_free(b);
        }
        if (status) status[i] = st;
        if (st != ACZ_OK && first_err == ACZ_OK) {
            first_err = st;
            first_msg = ctx->err;
        }
    }
    rc = pool_join(ctx, k, ctx->own);
    if (rc) return rc;
    CK(cudaEventRecord(ctx->io_ev, ctx->io_up));
    CK(cudaStreamWaitEvent(ctx->own, ctx->io_ev, 0));
    CK(cudaEventRecord(ctx->io_ev, ctx->io_down));
    CK(cudaStreamWaitEvent(ctx->own, ctx->io_ev, 0));
    CK(cudaStreamSynchronize(ctx->own));
    if (first_err) ctx->err = first_msg;
    if (!first_err) first_err = check_sticky(ctx);
    return first_err;
    });
}

// ------------------------------------------------------------------- host buffers --
void acz_gpu_host_free(void* p) { std::free(p); }

int acz_gpu_compress_host(acz_gpu_ctx* ctx, const float* h_in, const uint64_t* shape,
                          uint32_t rank, double eb, uint32_t quant_radius, uint32_t predictor,
                          uint8_t** acz1, uint64_t* acz1_size, uint8_t** sidecar,
                          uint64_t* sidecar_size) {
    return guarded(ctx, [&]() -> int {
    if (!ctx || !acz1 || !acz1_size) return ACZ_ERR_INVALID;
    *acz1 = nullptr;
    if (sidecar) *sidecar = nullptr;
    uint64_t n = 0;
    int rc = validate_shape(ctx, shape, rank, &n);
    if (rc) return rc;
    cudaStream_t s = ctx->own;
    if (n) {
        CK(grow(&ctx->ws_io, &ctx->ws_io_cap, 4ull * n));
        CK(cudaMemcpyAsync(ctx->ws_io, h_in, 4ull * n, cudaMemcpyHostToDevice, s));
    }
    acz_gpu_blob* b = nullptr;
    rc = acz_gpu_compress(ctx, static_cast<const float*>(ctx->ws_io), shape, rank, eb,
                          quant_radius, predictor, s, &b);
    if (rc) return rc;
    const uint64_t sz = b->info.compressed_bytes;
    uint8_t* buf = static_cast<uint8_t*>(std::malloc(sz));
    if (!buf) {
        acz_gpu_blob_free(b);
        return fail(ctx, ACZ_ERR_NOMEM, "host buffer");
    }
    rc = acz_gpu_blob_to_host(ctx, b, buf, sz, nullptr, s);
    if (!rc && sidecar) {
        const uint64_t ss = b->info.sidecar_bytes;
        *sidecar = static_cast<uint8_t*>(std::malloc(ss));
        if (!*sidecar) rc = fail(ctx, ACZ_ERR_NOMEM, "host buffer");
        else rc = acz_gpu_sidecar_to_host(ctx, b, *sidecar, ss, sidecar_size, s);
    }
    acz_gpu_blob_free(b);
    if (rc) {
        std::free(buf);
        if (sidecar && *sidecar) {
            std::free(*sidecar);
            *sidecar = nullptr;
        }
        return rc;
    }
    *acz1 = buf;
    *acz1_size = sz;
    return ACZ_OK;
    });
}

int acz_gpu_decompress_host(acz_gpu_ctx* ctx, const uint8_t* acz1, uint64_t acz1_size,
                            const uint8_t* sidecar, uint64_t sidecar_size, int zero_filter,
                            float* h_out, uint64_t n) {
    return guarded(ctx, [&]() -> int {
    if (!ctx || !h_out) return ACZ_ERR_INVALID;
    cudaStream_t s = ctx->own;
    acz_gpu_blob* b = nullptr;
    int rc = acz_gpu_blob_from_host(ctx, acz1, acz1_size, sidecar, sidecar_size, s, &b);
    if (rc) return rc;
    if (b->info.element_count != n) {
        acz_gpu_blob_free(b);
        return fail(ctx, ACZ_ERR_SHAPE, "output size mismatch");
    }
    int grc = (int)grow(&ctx->ws_io, &ctx->ws_io_cap, 4ull * n);
    if (grc != cudaSuccess) {
        acz_gpu_blob_free(b);
        return cuda_fail(ctx, (cudaError_t)grc, "grow");
    }
    rc = acz_gpu_decompress(ctx, b, zero_filter, static_cast<float*>(ctx->ws_io), s);
    if (!rc) {
        cudaError_t e = cudaMemcpyAsync(h_out, ctx->ws_io, 4ull * n, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) rc = cuda_fail(ctx, e, "d2h");
    }
    acz_gpu_blob_free(b);
    return rc;
    });
}

// ---------------------------------------------------------------------- statistics --
int acz_gpu_zero_bitmap(acz_gpu_ctx* ctx, const float* d_in, uint64_t n, uint32_t* d_bitmap,
                        uint64_t* nonzero, void* stream) {
    return guarded(ctx, [&]() -> int {
    if (!ctx || (!d_in && n)) return ACZ_ERR_INVALID;
    ctx->err.clear();
    if (n == 0) return fail(ctx, ACZ_ERR_DOMAIN, "nonzero_ratio: empty tensor");
    unsigned fl = 0;
    uint64_t nz = 0;
    int rc = run_stats(ctx, d_in, n, d_bitmap, static_cast<cudaStream_t>(stream), &fl, &nz, nullptr);
    if (rc) return rc;
    if (nonzero) *nonzero = nz;
    if (fl & kFlagNonFinite) return fail(ctx, ACZ_ERR_DOMAIN, "tensor element is not finite");
    return ACZ_OK;
    });
}

int acz_gpu_nonzero_ratio(acz_gpu_ctx* ctx, const float* d_in, uint64_t n, void* stream,
                          double* ratio) {
    uint64_t nz = 0;
    int rc = acz_gpu_zero_bitmap(ctx, d_in, n, nullptr, &nz, stream);
    if (rc) return rc;
    if (ratio) *ratio = (double)nz / (double)n;  // ref include/acz/tensor.hpp:98
    return ACZ_OK;
}

int acz_gpu_mean_abs(acz_gpu_ctx* ctx, const float* d_in, uint64_t n, void* stream,
                     double* mean) {
    return guarded(ctx, [&]() -> int {
    if (!ctx || (!d_in && n)) return ACZ_ERR_INVALID;
    ctx->err.clear();
    if (n == 0) return fail(ctx, ACZ_ERR_DOMAIN, "mean_abs: empty tensor");
    unsigned fl = 0;
    double sa = 0;
    int rc = run_stats(ctx, d_in, n, nullptr, static_cast<cudaStream_t>(stream), &fl, nullptr, &sa);
    if (rc) return rc;
    if (fl & kFlagNonFinite) return fail(ctx, ACZ_ERR_DOMAIN, "tensor element is not finite");
    if (mean) *mean = sa / (double)n;
    return ACZ_OK;
    });
}

// ------------------------------------------------------------------------- Huffman --
int acz_gpu_huffman_encode(acz_gpu_ctx* ctx, const uint32_t* d_symbols, uint64_t n,
                           uint32_t* book_sym, uint8_t* book_len, uint32_t book_cap,
                           uint32_t* book_size, uint8_t* bits, uint64_t bits_cap,
                           uint64_t* bit_length, void* stream) {
    return guarded(ctx, [&]() -> int {
    if (!ctx || !book_size || !bit_length) return ACZ_ERR_INVALID;
    ctx->err.clear();
    Slot* sl = get_slot(ctx, 0);
    *book_size = 0;
    *bit_length = 0;
    if (n == 0) return ACZ_OK;  // ref src/huffman.cpp:108
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // alphabet = max symbol + 1 (dense GPU histogram; alphabets beyond 2^26 unsupported)
    uint32_t maxsym = 0;
    {
        std::vector<uint32_t> tmp;  // small reduction on device via the stats path is overkill
        const uint64_t chunk = 1 << 24;
        tmp.resize(std::min<uint64_t>(n, chunk));
        for (uint64_t o = 0; o < n; o += chunk) {
            const uint64_t m = std::min<uint64_t>(chunk, n - o);
            CK(cudaMemcpyAsync(tmp.data(), d_symbols + o, 4ull * m, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            for (uint64_t i = 0; i < m; ++i) maxsym = std::max(maxsym, tmp[i]);
        }
    }
    if (maxsym >= (1u << 26)) return fail(ctx, ACZ_ERR_PARAM, "symbol alphabet beyond 2^26 unsupported");
    const uint32_t alphabet = maxsym + 1;
    int rc = build_book(ctx, sl, d_symbols, 0, n, alphabet, 0, s);
    if (rc) return rc;
    if ((rc = book_wait(ctx, sl, s))) return rc;
    const BookInfo bi = sl->h_small->info;
    if (bi.flags & kFlagDepth64) return fail(ctx, ACZ_ERR_DECODE, "huffman code length exceeds 64 bits");
    if (bi.flags & kFlagLenTooLong) return fail(ctx, ACZ_ERR_FORMAT, "code length > 56 bits unsupported");
    if (bi.book_size > book_cap) return fail(ctx, ACZ_ERR_INVALID, "book capacity too small");
    if ((bi.total_bits + 7) / 8 > bits_cap) return fail(ctx, ACZ_ERR_INVALID, "bits capacity too small");
    acz_gpu_blob tmpb;
    rc = finish_encode(ctx, sl, &tmpb, d_symbols, 0, n, nullptr, 0, false, s);
    if (rc) {
        blob_arena_free(&tmpb, s);
        return rc;
    }
    CK(cudaMemcpyAsync(book_sym, tmpb.book_sym, 4ull * bi.book_size, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(book_len, tmpb.book_len, bi.book_size, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(bits, tmpb.words, (bi.total_bits + 7) / 8, cudaMemcpyDeviceToHost, s));
    blob_arena_free(&tmpb, s);
    CK(cudaStreamSynchronize(s));
    *book_size = bi.book_size;
    *bit_length = bi.total_bits;
    return ACZ_OK;
    });
}

int acz_gpu_huffman_decode(acz_gpu_ctx* ctx, const uint32_t* book_sym, const uint8_t* book_len,
                           uint32_t book_size, const uint8_t* bits, uint64_t bit_length,
                           uint64_t count, uint32_t* d_out, void* stream) {
    return guarded(ctx, [&]() -> int {
    if (!ctx) return ACZ_ERR_INVALID;
    ctx->err.clear();
    Slot* sl = get_slot(ctx, 0);
    if (count == 0) return ACZ_OK;  // ref src/huffman.cpp:140
    if (book_size == 0) return fail(ctx, ACZ_ERR_DECODE, "empty codebook");
    for (uint32_t i = 1; i < book_size; ++i)
        if (book_len[i - 1] > book_len[i] ||
            (book_len[i - 1] == book_len[i] && book_sym[i - 1] >= book_sym[i]))
            return fail(ctx, ACZ_ERR_DECODE, "codebook entries are not in canonical order");
    for (uint32_t i = 0; i < book_size; ++i)
        if (book_len[i] == 0 || book_len[i] > 64)
            return fail(ctx, ACZ_ERR_DECODE, "invalid code length in codebook");
    for (uint32_t i = 0; i < book_size; ++i)
        if (book_sym[i] >= (1u << 27))
            return fail(ctx, ACZ_ERR_PARAM, "symbol beyond 2^27 unsupported by the GPU decoder");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    acz_gpu_blob tmpb;
    const uint64_t nwords = (bit_length + 31) / 32;
    CK(blob_alloc(&tmpb, book_size, nwords, 0, 0, false, s));
    CK(cudaMemsetAsync(tmpb.words, 0, 4ull * (nwords + 32), s));
    CK(cudaMemcpyAsync(tmpb.words, bits, (bit_length + 7) / 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(tmpb.book_sym, book_sym, 4ull * book_size, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(tmpb.book_len, book_len, book_size, cudaMemcpyHostToDevice, s));
    CK(launch_build_tables(tmpb.book_sym, tmpb.book_len, book_size, tmpb.canon, tmpb.lut, nullptr,
                           s, &ctx->launches));
    CK(cudaMemsetAsync(&sl->d_small->flags, 0, sizeof(unsigned), s));
    ScanArgs sa{};
    sa.words = tmpb.words;
    sa.nwords = nwords;
    sa.bit_length = bit_length;
    sa.n = count;
    sa.lut = tmpb.lut;
    sa.canon = tmpb.canon;
    sa.book_sym = tmpb.book_sym;
    sa.out_index = nullptr;
    sa.n_outliers = 0;
    sa.interval = count;
    sa.side_bitoff = nullptr;
    sa.side_outl = nullptr;
    sa.sym_out = d_out;
    sa.plane_outl = nullptr;
    sa.plane_size = count;
    sa.flags = &sl->d_small->flags;
    CK(grow(&ctx->ws_scan, &ctx->ws_scan_cap, scan_decode_scratch_bytes(sa.bit_length)));
    CK(launch_scan_decode(sa, ctx->ws_scan, s, &ctx->launches));
    CK(cudaMemcpyAsync(&sl->h_small->flags, &sl->d_small->flags, sizeof(unsigned),
                       cudaMemcpyDeviceToHost, s));
    blob_arena_free(&tmpb, s);
    CK(cudaStreamSynchronize(s));
    const unsigned fl = sl->h_small->flags;
    if (fl & kDecTruncated) return fail(ctx, ACZ_ERR_DECODE, "truncated bitstream");
    if (fl & kDecNoMatch) return fail(ctx, ACZ_ERR_DECODE, "no codeword matches bitstream");
    return ACZ_OK;
    });
}

// ------------------------------------------------------------------ memory helpers --
int acz_gpu_malloc(acz_gpu_ctx* ctx, uint64_t bytes, void* stream, void** d_ptr) {
    if (!ctx || !d_ptr) return ACZ_ERR_INVALID;
    *d_ptr = nullptr;
    if (bytes == 0) return ACZ_OK;
    cudaError_t e = cudaMallocAsync(d_ptr, bytes, static_cast<cudaStream_t>(stream));
    if (e == cudaErrorMemoryAllocation) return fail(ctx, ACZ_ERR_NOMEM, "device allocation failed");
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMallocAsync");
    return ACZ_OK;
}

int acz_gpu_free(acz_gpu_ctx* ctx, void* d_ptr, void* stream) {
    if (!ctx) return ACZ_ERR_INVALID;
    if (d_ptr) CK(cudaFreeAsync(d_ptr, static_cast<cudaStream_t>(stream)));
    return ACZ_OK;
}

int acz_gpu_memcpy(acz_gpu_ctx* ctx, void* dst, const void* src, uint64_t bytes, int kind,
                   void* stream) {
    if (!ctx || (bytes && (!dst || !src))) return ACZ_ERR_INVALID;
    const cudaMemcpyKind k = kind == ACZ_COPY_H2D   ? cudaMemcpyHostToDevice
                             : kind == ACZ_COPY_D2H ? cudaMemcpyDeviceToHost
                             : kind == ACZ_COPY_D2D ? cudaMemcpyDeviceToDevice
                                                    : cudaMemcpyDefault;
    if (bytes) CK(cudaMemcpyAsync(dst, src, bytes, k, static_cast<cudaStream_t>(stream)));
    return ACZ_OK;
}

int acz_gpu_stream_sync(acz_gpu_ctx* ctx, void* stream) {
    if (!ctx) return ACZ_ERR_INVALID;
    CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    return ACZ_OK;
}

int acz_gpu_relu(acz_gpu_ctx* ctx, float* d_x, uint64_t n, void* stream) {
    if (!ctx || (n && !d_x)) return ACZ_ERR_INVALID;
    if (n) CK(launch_relu(d_x, n, ctx->sms, static_cast<cudaStream_t>(stream), &ctx->launches));
    return ACZ_OK;
}

// ----------------------------------------------------------------------- profiling --
int acz_gpu_profile_enable(acz_gpu_ctx* ctx, int on) {
    if (!ctx) return ACZ_ERR_INVALID;
    double ms[ACZ_K_COUNT];
    uint64_t n[ACZ_K_COUNT];
    acz_gpu_profile_read(ctx, ms, n);
    for (int i = 0; i < ACZ_K_COUNT; ++i) {
        ctx->prof_ms[i] = 0;
        ctx->prof_n[i] = 0;
    }
    ctx->prof = on != 0;
    return ACZ_OK;
}

int acz_gpu_profile_read(acz_gpu_ctx* ctx, double* ms, uint64_t* launches) {
    if (!ctx) return ACZ_ERR_INVALID;
    for (auto& p : ctx->pending) {
        cudaEventSynchronize(p.b);
        float t = 0;
        if (cudaEventElapsedTime(&t, p.a, p.b) == cudaSuccess) {
            ctx->prof_ms[p.cls] += t;
            ctx->prof_n[p.cls] += 1;
        }
        ctx->event_pool.push_back(p.a);
        ctx->event_pool.push_back(p.b);
    }
    ctx->pending.clear();
    for (int i = 0; i < ACZ_K_COUNT; ++i) {
        if (ms) ms[i] = ctx->prof_ms[i];
        if (launches) launches[i] = ctx->prof_n[i];
    }
    return ACZ_OK;
}

// --------------------------------------------------------------------------- debug --
int acz_gpu_debug_counters(acz_gpu_ctx* ctx, uint64_t* out, uint32_t n, int reset) {
    if (!ctx || !out || n < 8) return ACZ_ERR_INVALID;
    unsigned long long v[20];
    CK(quant_spec_stats(v, reset != 0));
    for (int i = 0; i < 8; ++i) out[i] = v[i];
    if (n >= 16) {
        unsigned long long c[8];
        CK(codebook_stats(c, reset != 0));
        for (int i = 0; i < 8; ++i) out[8 + i] = c[i];
    }
    if (n >= 20)
        for (int i = 0; i < 4; ++i) out[16 + i] = v[8 + i];
    if (n >= 24) {
        unsigned long long d[4];
        CK(decode_stats(d, reset != 0));
        for (int i = 0; i < 4; ++i) out[20 + i] = d[i];
    }
    if (n >= 28)
        for (int i = 0; i < 4; ++i) out[24 + i] = v[12 + i];
    else if (n >= 26)
        for (int i = 0; i < 2; ++i) out[24 + i] = v[12 + i];
    if (n >= 32)
        for (int i = 0; i < 4; ++i) out[28 + i] = v[16 + i];
    if (n >= 128) {  // per-segment phase durations of K2b, log2 buckets (stats builds)
        unsigned long long h[96];
        CK(quant_spec_hist(h, reset != 0));
        for (int i = 0; i < 96; ++i) out[32 + i] = h[i];
    }
    return ACZ_OK;
}

int acz_gpu_debug_last_symbols(acz_gpu_ctx* ctx, uint32_t* d_out, uint64_t n, void* stream) {
    if (!ctx || !d_out) return ACZ_ERR_INVALID;
    Slot* sl = get_slot(ctx, 0);
    if (n != sl->last_n || !sl->ws_sym) return fail(ctx, ACZ_ERR_SHAPE, "no symbols of that size");
    if (sl->last_sym16)
        CK(launch_widen_u16(static_cast<const uint16_t*>(sl->ws_sym), d_out, n, ctx->sms,
                            static_cast<cudaStream_t>(stream), &ctx->launches));
    else
        CK(cudaMemcpyAsync(d_out, sl->ws_sym, 4ull * n, cudaMemcpyDeviceToDevice,
                           static_cast<cudaStream_t>(stream)));
    return ACZ_OK;
}

}  // extern "C"
