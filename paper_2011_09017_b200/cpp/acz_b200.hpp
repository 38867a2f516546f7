// acz_b200.hpp -- C++ host layer of the B200 activation compressor.
//
// Keeps the reference's codec and adaptive error-bound API (namespace acz in
// /root/reference/proj/core) and calls the sm_100a kernels only through the C-ABI of
// include/acz_gpu.h (libacz_gpu.so). Header-only; needs no CUDA headers.
//
//   reference (proj/core)                         here
//   acz::Error hierarchy  include/acz/error.hpp   acz_b200::Error, ParamError, DomainError, ...
//   acz::CodecParams      include/acz/codec.hpp:17-23        CodecParams (validate)
//   acz::compress         include/acz/codec.hpp:54           compress(const Tensor&, params)
//   acz::decompress       include/acz/codec.hpp:59           decompress(blob, zero_filter)
//   acz::compression_ratio include/acz/codec.hpp:61          compression_ratio(blob)
//   acz::blob_to_bytes / blob_from_bytes  :69-70             CompressedTensor::bytes / blob_from_bytes
//   acz::nonzero_ratio / mean_abs  include/acz/tensor.hpp:82-99   nonzero_ratio / mean_abs (device)
//   acz::Controller       include/acz/controller.hpp:99-155  Controller (device activations)
//
// Device-resident activations (the training path) go through DeviceTensor / DeviceBlob;
// host tensors (the reference's own calling convention) through Tensor / CompressedTensor.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <iostream>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "acz_gpu.h"

namespace acz_b200 {

// ---------------------------------------------------------------- errors (error.hpp) --
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ShapeError : Error {
    using Error::Error;
};
struct DomainError : Error {
    using Error::Error;
};
struct ParamError : Error {
    using Error::Error;
};
struct FormatError : Error {
    using Error::Error;
};
struct DecodeError : Error {
    using Error::Error;
};
struct CudaError : Error {
    using Error::Error;
};

[[noreturn]] inline void raise_status(int rc, const std::string& msg) {
    switch (rc) {
        case ACZ_ERR_PARAM: throw ParamError(msg);
        case ACZ_ERR_DOMAIN: throw DomainError(msg);
        case ACZ_ERR_FORMAT: throw FormatError(msg);
        case ACZ_ERR_DECODE: throw DecodeError(msg);
        case ACZ_ERR_SHAPE: throw ShapeError(msg);
        case ACZ_ERR_CUDA: throw CudaError(msg);
        case ACZ_ERR_NOMEM: throw std::bad_alloc();
        default: throw Error(msg);
    }
}

// ------------------------------------------------------------------------- context --
// One context per (device, host thread) (ref SPEC.md:157-158: the pure API is reentrant
// across distinct inputs).
class Context {
public:
    explicit Context(int device = 0) {
        const int rc = acz_gpu_ctx_create(device, &c_);
        if (rc) raise_status(rc, "acz_gpu_ctx_create failed");
    }
    ~Context() {
        if (c_) acz_gpu_ctx_destroy(c_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    acz_gpu_ctx* get() const { return c_; }
    void check(int rc) const {
        if (rc) raise_status(rc, acz_gpu_last_error(c_));
    }
    void sync(void* stream = nullptr) const { check(acz_gpu_stream_sync(c_, stream)); }

    static Context& thread_default() {
        thread_local Context ctx(0);
        return ctx;
    }

private:
    acz_gpu_ctx* c_ = nullptr;
};

// --------------------------------------------------------------- params (codec.hpp) --
enum class Predictor : uint8_t { PrevValue = 0, Lorenzo2d = 1 };

struct CodecParams {
    double eb = 1e-4;                // absolute error bound
    uint32_t quant_radius = 32768;   // half-width of the code range, power of two
    Predictor predictor = Predictor::PrevValue;

    // ref src/codec.cpp:54-59
    void validate() const {
        if (!(eb > 0.0) || !std::isfinite(eb)) throw ParamError("error bound must be positive");
        if (quant_radius < 2 || quant_radius > (1u << 24) || (quant_radius & (quant_radius - 1)))
            throw ParamError("quant_radius must be a power of two in [2, 2^24]");
    }
};

// ------------------------------------------------------------------- host tensors --
struct Tensor {
    std::vector<size_t> shape;
    std::vector<float> data;
    Tensor() = default;
    Tensor(std::vector<size_t> s, std::vector<float> d) : shape(std::move(s)), data(std::move(d)) {
        size_t n = 1;
        for (size_t e : shape) n *= e;
        if (shape.empty()) n = 0;
        if (n != data.size()) throw ShapeError("tensor data size does not match shape");
    }
    size_t size() const { return data.size(); }
};

// Host blob: the ACZ1 byte image (bit-exact with ref blob_to_bytes) plus the optional
// decode sidecar that lets the GPU decode it chunk-parallel.
struct CompressedTensor {
    std::vector<size_t> shape;
    CodecParams params;
    std::vector<uint8_t> bytes;    // ACZ1
    std::vector<uint8_t> sidecar;  // ACZS (not part of ACZ1; may be empty)
    uint64_t uncompressed_bytes = 0;
    uint64_t compressed_bytes = 0;  // == bytes.size()
    size_t element_count() const {
        size_t n = 1;
        for (size_t e : shape) n *= e;
        return shape.empty() ? 0 : n;
    }
};

inline CompressedTensor compress(const Tensor& t, const CodecParams& p,
                                 Context& ctx = Context::thread_default()) {
    std::vector<uint64_t> shp(t.shape.begin(), t.shape.end());
    uint8_t *blob = nullptr, *side = nullptr;
    uint64_t bsz = 0, ssz = 0;
    ctx.check(acz_gpu_compress_host(ctx.get(), t.data.data(), shp.data(), (uint32_t)shp.size(),
                                    p.eb, p.quant_radius, (uint32_t)p.predictor, &blob, &bsz,
                                    &side, &ssz));
    CompressedTensor c;
    c.shape = t.shape;
    c.params = p;
    c.bytes.assign(blob, blob + bsz);
    c.sidecar.assign(side, side + ssz);
    acz_gpu_host_free(blob);
    acz_gpu_host_free(side);
    c.uncompressed_bytes = 4ull * t.size();
    c.compressed_bytes = bsz;
    return c;
}

inline Tensor decompress(const CompressedTensor& c, bool zero_filter = false,
                         Context& ctx = Context::thread_default()) {
    std::vector<float> out(c.element_count());
    ctx.check(acz_gpu_decompress_host(ctx.get(), c.bytes.data(), c.bytes.size(),
                                      c.sidecar.empty() ? nullptr : c.sidecar.data(),
                                      c.sidecar.size(), zero_filter ? 1 : 0, out.data(),
                                      out.size()));
    return Tensor(c.shape, std::move(out));
}

inline double compression_ratio(const CompressedTensor& c) {
    return (double)c.uncompressed_bytes / (double)c.compressed_bytes;  // ref src/codec.cpp:173-175
}

inline std::vector<uint8_t> blob_to_bytes(const CompressedTensor& c) { return c.bytes; }

// ref src/codec.cpp:201-262 (validation by the device parser: same checks and errors)
inline CompressedTensor blob_from_bytes(const uint8_t* data, size_t size,
                                        Context& ctx = Context::thread_default()) {
    acz_gpu_blob* b = nullptr;
    ctx.check(acz_gpu_blob_from_host(ctx.get(), data, size, nullptr, 0, nullptr, &b));
    acz_gpu_blob_info_t in{};
    acz_gpu_blob_info(b, &in);
    acz_gpu_blob_free(b);
    CompressedTensor c;
    c.shape.assign(in.shape, in.shape + in.rank);
    c.params.eb = in.eb;
    c.params.quant_radius = in.quant_radius;
    c.params.predictor = (Predictor)in.predictor;
    c.bytes.assign(data, data + size);
    c.uncompressed_bytes = in.uncompressed_bytes;
    c.compressed_bytes = size;
    return c;
}

// ----------------------------------------------------------------- device tensors --
// Owning device buffer of fp32 activations (stream-ordered allocation).
class DeviceTensor {
public:
    DeviceTensor() = default;
    DeviceTensor(std::vector<uint64_t> shape, Context& ctx, void* stream = nullptr)
        : shape_(std::move(shape)), ctx_(&ctx), stream_(stream) {
        void* p = nullptr;
        ctx.check(acz_gpu_malloc(ctx.get(), 4ull * size(), stream, &p));
        d_ = static_cast<float*>(p);
    }
    ~DeviceTensor() { reset(); }
    DeviceTensor(DeviceTensor&& o) noexcept { *this = std::move(o); }
    DeviceTensor& operator=(DeviceTensor&& o) noexcept {
        if (this != &o) {
            reset();
            shape_ = std::move(o.shape_);
            d_ = o.d_;
            ctx_ = o.ctx_;
            stream_ = o.stream_;
            o.d_ = nullptr;
        }
        return *this;
    }
    void reset() {
        if (d_ && ctx_) acz_gpu_free(ctx_->get(), d_, stream_);
        d_ = nullptr;
    }
    static DeviceTensor from_host(const Tensor& t, Context& ctx, void* stream = nullptr) {
        DeviceTensor d(std::vector<uint64_t>(t.shape.begin(), t.shape.end()), ctx, stream);
        ctx.check(acz_gpu_memcpy(ctx.get(), d.d_, t.data.data(), 4ull * t.size(), ACZ_COPY_H2D,
                                 stream));
        return d;
    }
    Tensor to_host() const {
        std::vector<float> h(size());
        ctx_->check(acz_gpu_memcpy(ctx_->get(), h.data(), d_, 4ull * size(), ACZ_COPY_D2H,
                                   stream_));
        ctx_->sync(stream_);
        return Tensor(std::vector<size_t>(shape_.begin(), shape_.end()), std::move(h));
    }
    float* data() const { return d_; }
    const std::vector<uint64_t>& shape() const { return shape_; }
    uint64_t size() const {
        uint64_t n = 1;
        for (uint64_t e : shape_) n *= e;
        return shape_.empty() ? 0 : n;
    }
    bool empty() const { return d_ == nullptr; }

private:
    std::vector<uint64_t> shape_;
    float* d_ = nullptr;
    Context* ctx_ = nullptr;
    void* stream_ = nullptr;
};

// Owning device blob (ACZ1 content + decode sidecar in HBM).
class DeviceBlob {
public:
    DeviceBlob() = default;
    explicit DeviceBlob(acz_gpu_blob* b) : b_(b) {
        if (b_) acz_gpu_blob_info(b_, &info_);
    }
    ~DeviceBlob() {
        if (b_) acz_gpu_blob_free(b_);
    }
    DeviceBlob(DeviceBlob&& o) noexcept : b_(o.b_), info_(o.info_) { o.b_ = nullptr; }
    DeviceBlob& operator=(DeviceBlob&& o) noexcept {
        if (this != &o) {
            if (b_) acz_gpu_blob_free(b_);
            b_ = o.b_;
            info_ = o.info_;
            o.b_ = nullptr;
        }
        return *this;
    }
    acz_gpu_blob* get() const { return b_; }
    const acz_gpu_blob_info_t& info() const { return info_; }
    uint64_t compressed_bytes() const { return info_.compressed_bytes; }
    double ratio() const { return (double)info_.uncompressed_bytes / (double)info_.compressed_bytes; }
    std::vector<uint8_t> to_bytes(Context& ctx, void* stream = nullptr) const {
        std::vector<uint8_t> out(info_.compressed_bytes);
        ctx.check(acz_gpu_blob_to_host(ctx.get(), b_, out.data(), out.size(), nullptr, stream));
        return out;
    }

private:
    acz_gpu_blob* b_ = nullptr;
    acz_gpu_blob_info_t info_{};
};

inline DeviceBlob compress(const DeviceTensor& t, const CodecParams& p, Context& ctx,
                           void* stream = nullptr) {
    acz_gpu_blob* b = nullptr;
    ctx.check(acz_gpu_compress(ctx.get(), t.data(), t.shape().data(), (uint32_t)t.shape().size(),
                               p.eb, p.quant_radius, (uint32_t)p.predictor, stream, &b));
    return DeviceBlob(b);
}

inline DeviceTensor decompress(const DeviceBlob& b, bool zero_filter, Context& ctx,
                               void* stream = nullptr) {
    const auto& in = b.info();
    DeviceTensor out(std::vector<uint64_t>(in.shape, in.shape + in.rank), ctx, stream);
    ctx.check(acz_gpu_decompress(ctx.get(), b.get(), zero_filter ? 1 : 0, out.data(), stream));
    return out;
}

// Controller statistics on device tensors (ref include/acz/tensor.hpp:82-99).
inline double nonzero_ratio(const DeviceTensor& t, Context& ctx, void* stream = nullptr) {
    double r = 0.0;
    ctx.check(acz_gpu_nonzero_ratio(ctx.get(), t.data(), t.size(), stream, &r));
    return r;
}
inline double mean_abs(const DeviceTensor& t, Context& ctx, void* stream = nullptr) {
    double m = 0.0;
    ctx.check(acz_gpu_mean_abs(ctx.get(), t.data(), t.size(), stream, &m));
    return m;
}
inline uint64_t nonzero_count(const DeviceTensor& t, Context& ctx, void* stream = nullptr) {
    uint64_t nz = 0;
    ctx.check(acz_gpu_zero_bitmap(ctx.get(), t.data(), t.size(), nullptr, &nz, stream));
    return nz;
}

// ------------------------------------------------------ controller (controller.hpp) --
enum class ZeroRestoration { CodecFilter, ReluRecompute };

struct ControllerConfig {
    int64_t collect_interval = 1000;  // W
    double sigma_fraction = 0.01;
    double coefficient_a = 0.32;
    double eb_min = 1e-8;
    double eb_max = 1e-1;
    ZeroRestoration zero_restoration = ZeroRestoration::CodecFilter;
    Predictor predictor = Predictor::PrevValue;
    uint32_t quant_radius = 32768;

    // ref src/controller.cpp:14-21
    void validate() const {
        if (collect_interval < 1) throw ParamError("collect_interval (W) must be >= 1");
        if (!(sigma_fraction > 0.0)) throw ParamError("sigma_fraction must be positive");
        if (!(coefficient_a > 0.0)) throw ParamError("coefficient_a must be positive");
        if (!(eb_min > 0.0) || !(eb_min <= eb_max))
            throw ParamError("error-bound clamps must satisfy 0 < eb_min <= eb_max");
        CodecParams{eb_min, quant_radius, predictor}.validate();
    }
};

struct LayerStats {
    int layer_id = -1;
    double l_bar = 0.0;
    double r = 0.0;
    double m_avg = 0.0;
    size_t batch = 0;
    int64_t collected_at = -1;
    bool degenerate = false;
};

struct LedgerRecord {
    int64_t iteration;
    int layer_id;
    double eb, predicted_sigma, l_bar, r, m_avg, ratio;
    bool fallback;
};

class CompressionLedger {
public:
    void append(const LedgerRecord& r) { records_.push_back(r); }
    const std::vector<LedgerRecord>& records() const { return records_; }
    // ref src/controller.cpp:67-76 (same header and %.17g formatting)
    std::string to_csv() const {
        std::string out = "iteration,layer,eb,predicted_sigma,L_bar,R,M_avg,ratio,fallback_flag\n";
        char line[256];
        for (const auto& r : records_) {
            std::snprintf(line, sizeof(line), "%lld,%d,%.17g,%.17g,%.17g,%.17g,%.17g,%.17g,%d\n",
                          (long long)r.iteration, r.layer_id, r.eb, r.predicted_sigma, r.l_bar,
                          r.r, r.m_avg, r.ratio, r.fallback ? 1 : 0);
            out += line;
        }
        return out;
    }

private:
    std::vector<LedgerRecord> records_;
};

// Stashed activation: exactly one of raw / blob engaged (ref include/acz/controller.hpp:65-78).
struct ActivationHandle {
    std::optional<DeviceTensor> raw;
    std::optional<DeviceBlob> blob;
    bool apply_relu = false;
    bool zero_filter = false;
    int layer_id = -1;
    size_t held_bytes = 0;
    double achieved_ratio = 1.0;
};

// Sums that make the controller statistics global across data-parallel ranks. The local
// sums are reduced by `reducer` (e.g. one ncclAllReduce of 7 doubles per layer every W
// iterations) before the ratios are formed; single process: identity.
using StatsReducer = std::function<void(double* sums, size_t count)>;

// Four-phase adaptive scheme (ref src/controller.cpp:94-253) over device activations.
class Controller {
public:
    Controller(const ControllerConfig& cfg, int num_layers, Context& ctx = Context::thread_default())
        : cfg_(cfg), ctx_(&ctx) {
        cfg_.validate();
        if (num_layers < 0) throw ParamError("controller needs a non-negative layer count");
        windows_.resize((size_t)num_layers);
    }
    void set_stats_reducer(StatsReducer r) { reducer_ = std::move(r); }

    void begin_iteration(int64_t iteration) {
        if (iteration < 0) throw ParamError("iteration must be >= 0");
        iteration_ = iteration;
    }
    int64_t iteration() const { return iteration_; }
    bool collecting() const { return iteration_ % cfg_.collect_interval == 0; }

    // Phase 1 (ref src/controller.cpp:124-152). L_bar and M_avg are means of |.|, R the
    // nonzero fraction; with a reducer they are global over ranks (sums then ratios).
    LayerStats collect_stats(int layer, const DeviceTensor& activation, const DeviceTensor& loss,
                             const DeviceTensor& momentum, size_t batch, void* stream = nullptr) {
        if (layer < 0 || (size_t)layer >= windows_.size())
            throw ParamError("collect_stats: unknown layer id");
        if (!collecting()) throw ParamError("collect_stats invoked outside a collection iteration");
        double sums[7] = {mean_abs(loss, *ctx_, stream) * (double)loss.size(), (double)loss.size(),
                          (double)nonzero_count(activation, *ctx_, stream),
                          (double)activation.size(),
                          mean_abs(momentum, *ctx_, stream) * (double)momentum.size(),
                          (double)momentum.size(), (double)batch};
        if (reducer_) reducer_(sums, 7);
        LayerStats st;
        st.layer_id = layer;
        st.l_bar = sums[1] > 0 ? sums[0] / sums[1] : 0.0;
        st.r = sums[3] > 0 ? sums[2] / sums[3] : 0.0;
        st.m_avg = sums[5] > 0 ? sums[4] / sums[5] : 0.0;
        st.batch = (size_t)sums[6];
        st.collected_at = iteration_;
        st.degenerate = st.l_bar == 0.0 || st.m_avg == 0.0 || st.r == 0.0;
        close_window(layer);
        Window& w = windows_[(size_t)layer];
        w = Window{};
        w.stats = st;
        w.open = true;
        if (!st.degenerate) {
            w.sigma = target_sigma(st, cfg_);
            w.eb = compute_error_bound(st, w.sigma, cfg_);
            w.fallback = false;
        }
        return st;
    }

    // Phase 2 (ref src/controller.cpp:154-157)
    static double target_sigma(const LayerStats& s, const ControllerConfig& cfg) {
        if (!(s.m_avg > 0.0)) throw ParamError("target_sigma: degenerate M_avg");
        return cfg.sigma_fraction * s.m_avg;
    }
    // Phase 3 (ref src/controller.cpp:159-168): eb = sigma / (a * L_bar * sqrt(N * R)), clamped
    static double compute_error_bound(const LayerStats& s, double sigma, const ControllerConfig& cfg) {
        if (!(sigma > 0.0)) throw ParamError("compute_error_bound: sigma must be positive");
        if (!(s.l_bar > 0.0) || !(s.r > 0.0)) throw ParamError("compute_error_bound: degenerate stats");
        const double eb = sigma / (cfg.coefficient_a * s.l_bar * std::sqrt((double)s.batch * s.r));
        return std::clamp(eb, cfg.eb_min, cfg.eb_max);
    }

    bool layer_active(int layer) const {
        if (layer < 0 || (size_t)layer >= windows_.size()) return false;
        const Window& w = windows_[(size_t)layer];
        return w.open && !w.fallback && iteration_ > w.stats.collected_at;
    }
    double layer_eb(int layer) const { return layer_active(layer) ? windows_[(size_t)layer].eb : 0.0; }
    const LayerStats* layer_stats(int layer) const {
        if (layer < 0 || (size_t)layer >= windows_.size()) return nullptr;
        const Window& w = windows_[(size_t)layer];
        return w.open ? &w.stats : nullptr;
    }

    // Phase 4, forward (ref src/controller.cpp:194-232): compress on the GPU or pass through;
    // a codec failure degrades to pass-through with a warning.
    ActivationHandle wrap_forward(int layer, DeviceTensor&& act, bool is_post_relu,
                                  void* stream = nullptr) {
        if (layer < 0 || (size_t)layer >= windows_.size())
            throw ParamError("wrap_forward: unknown layer id");
        const uint64_t in_bytes = 4ull * act.size();
        ActivationHandle h;
        h.layer_id = layer;
        auto pass = [&]() {
            h.held_bytes = in_bytes;
            h.raw = std::move(act);
            h.achieved_ratio = 1.0;
        };
        if (!layer_active(layer)) {
            pass();
        } else {
            const Window& w = windows_[(size_t)layer];
            try {
                CodecParams params{w.eb, cfg_.quant_radius, cfg_.predictor};
                DeviceBlob b = compress(act, params, *ctx_, stream);
                h.held_bytes = b.compressed_bytes();
                h.achieved_ratio = b.ratio();
                if (cfg_.zero_restoration == ZeroRestoration::ReluRecompute && is_post_relu)
                    h.apply_relu = true;
                else
                    h.zero_filter = true;
                h.blob = std::move(b);
                act.reset();  // release the original buffer
            } catch (const Error& e) {
                std::cerr << "warning: compression failed for layer " << layer << " (" << e.what()
                          << "); passing through\n";
                pass();
            }
        }
        Window& w = windows_[(size_t)layer];
        if (w.open) {
            w.bytes_in += in_bytes;
            w.bytes_stored += h.held_bytes;
        }
        total_in_ += in_bytes;
        total_stored_ += h.held_bytes;
        current_bytes_ += h.held_bytes;
        peak_bytes_ = std::max(peak_bytes_, current_bytes_);
        return h;
    }

    // Phase 4, backward (ref src/controller.cpp:234-249)
    DeviceTensor unwrap_backward(ActivationHandle& h, void* stream = nullptr) {
        if (h.raw) {
            DeviceTensor t = std::move(*h.raw);
            h.raw.reset();
            current_bytes_ -= h.held_bytes;
            h.held_bytes = 0;
            return t;
        }
        if (!h.blob) throw ParamError("unwrap_backward: handle already consumed");
        DeviceTensor t = decompress(*h.blob, h.zero_filter, *ctx_, stream);
        if (h.apply_relu) ctx_->check(acz_gpu_relu(ctx_->get(), t.data(), t.size(), stream));
        h.blob.reset();
        current_bytes_ -= h.held_bytes;
        h.held_bytes = 0;
        return t;
    }

    void finalize() {
        for (size_t i = 0; i < windows_.size(); ++i) close_window((int)i);
    }
    const CompressionLedger& ledger() const { return ledger_; }
    size_t current_stash_bytes() const { return current_bytes_; }
    size_t peak_stash_bytes() const { return peak_bytes_; }
    uint64_t total_bytes_in() const { return total_in_; }
    uint64_t total_bytes_stored() const { return total_stored_; }

private:
    struct Window {
        LayerStats stats;
        double eb = 0.0, sigma = 0.0;
        bool fallback = true, open = false;
        uint64_t bytes_in = 0, bytes_stored = 0;
    };
    // ref src/controller.cpp:98-122
    void close_window(int layer) {
        Window& w = windows_[(size_t)layer];
        if (!w.open) return;
        LedgerRecord r;
        r.iteration = w.stats.collected_at;
        r.layer_id = layer;
        r.eb = w.fallback ? 0.0 : w.eb;
        r.predicted_sigma = w.fallback ? 0.0 : w.sigma;
        r.l_bar = w.stats.l_bar;
        r.r = w.stats.r;
        r.m_avg = w.stats.m_avg;
        r.ratio = w.bytes_stored == 0 ? 1.0 : (double)w.bytes_in / (double)w.bytes_stored;
        r.fallback = w.fallback;
        ledger_.append(r);
        w.open = false;
    }

    ControllerConfig cfg_;
    Context* ctx_;
    StatsReducer reducer_;
    std::vector<Window> windows_;
    CompressionLedger ledger_;
    int64_t iteration_ = 0;
    size_t current_bytes_ = 0, peak_bytes_ = 0;
    uint64_t total_in_ = 0, total_stored_ = 0;
};

// Batch-size scheme (BASELINE config 5; the reference leaves it as a non-goal, SPEC.md:431,
// PAPER.md:531-533): the largest batch whose stashed bytes fit the activation budget, given
// the stash measured at the current batch (stash scales linearly with the batch).
inline size_t suggest_batch(size_t batch, size_t peak_stash_bytes, size_t budget_bytes,
                            size_t granularity = 8, size_t max_batch = 1u << 20) {
    if (batch == 0 || peak_stash_bytes == 0) return batch;
    const double per_sample = (double)peak_stash_bytes / (double)batch;
    size_t b = (size_t)((double)budget_bytes / per_sample);
    b = (b / granularity) * granularity;
    return std::max<size_t>(granularity, std::min(b, max_batch));
}

}  // namespace acz_b200
