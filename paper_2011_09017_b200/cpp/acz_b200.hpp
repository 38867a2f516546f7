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
//
// Device-resident activations (the training path) go through DeviceTensor / DeviceBlob;
// host tensors (the reference's own calling convention) through Tensor / CompressedTensor.
// The reference's Controller is not restated here: the proj/core drop-in
// (proj_core/gpu_codec.cpp replacing src/codec.cpp) runs the reference's own
// src/controller.cpp over the GPU codec (oracle/Makefile `dropin`, tests/test_gpu_dropin.py).
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
