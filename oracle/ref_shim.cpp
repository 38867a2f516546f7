// TEST INFRASTRUCTURE ONLY (oracle). Not part of the product path.
//
// extern "C" shim over the UNMODIFIED reference codec (/root/reference/proj/core),
// compiled from the reference's own sources by oracle/Makefile into
// oracle/_ref/libacz_ref.so. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it, and only as the checker or the
// timed CPU baseline.
//
// Wraps: acz::compress / acz::decompress (ref src/codec.cpp:61-171),
//        acz::blob_to_bytes / blob_from_bytes (src/codec.cpp:177-262),
//        acz::huffman_encode / huffman_decode (src/huffman.cpp:107-189),
//        acz::nonzero_ratio / mean_abs (include/acz/tensor.hpp:82-99).
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "acz/codec.hpp"
#include "acz/controller.hpp"
#include "acz/error.hpp"
#include "acz/huffman.hpp"
#include "acz/tensor.hpp"

namespace {

// Status codes shared with include/acz_gpu.h (ACZ_ERR_*).
int status_of(const std::exception& e) {
    if (dynamic_cast<const acz::ParamError*>(&e)) return 1;
    if (dynamic_cast<const acz::DomainError*>(&e)) return 2;
    if (dynamic_cast<const acz::FormatError*>(&e)) return 3;
    if (dynamic_cast<const acz::DecodeError*>(&e)) return 4;
    if (dynamic_cast<const acz::ShapeError*>(&e)) return 5;
    return 9;
}

void set_err(char* err, int cap, const char* msg) {
    if (err && cap > 0) {
        std::strncpy(err, msg, static_cast<std::size_t>(cap) - 1);
        err[cap - 1] = 0;
    }
}

template <class F>
int guarded(char* err, int cap, F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        set_err(err, cap, e.what());
        return status_of(e);
    }
}

std::vector<std::size_t> to_shape(const std::uint64_t* shape, int rank) {
    std::vector<std::size_t> s(static_cast<std::size_t>(rank));
    for (int i = 0; i < rank; ++i) s[static_cast<std::size_t>(i)] = shape[i];
    return s;
}

std::size_t volume(const std::uint64_t* shape, int rank) {
    std::size_t n = 1;
    for (int i = 0; i < rank; ++i) n *= shape[i];
    return rank == 0 ? 0 : n;
}

} // namespace

extern "C" {

void ref_free(void* p) { std::free(p); }

// compress -> ACZ1 bytes (malloc'd, caller frees with ref_free)
int ref_compress(const float* x, const std::uint64_t* shape, int rank, double eb,
                 std::uint32_t radius, int predictor, std::uint8_t** out,
                 std::uint64_t* out_size, char* err, int errcap) {
    return guarded(err, errcap, [&] {
        std::size_t n = volume(shape, rank);
        acz::Tensor t(to_shape(shape, rank), std::vector<float>(x, x + n));
        acz::CodecParams p{eb, radius, static_cast<acz::Predictor>(predictor)};
        acz::CompressedTensor c = acz::compress(t, p);
        auto bytes = acz::blob_to_bytes(c);
        if (bytes.size() != c.compressed_bytes) throw acz::Error("size mismatch");
        *out = static_cast<std::uint8_t*>(std::malloc(bytes.size() ? bytes.size() : 1));
        std::memcpy(*out, bytes.data(), bytes.size());
        *out_size = bytes.size();
    });
}

// ACZ1 bytes -> floats (out must hold n floats; n checked against the header)
int ref_decompress(const std::uint8_t* blob, std::uint64_t size, int zero_filter, float* out,
                   std::uint64_t n, char* err, int errcap) {
    return guarded(err, errcap, [&] {
        acz::CompressedTensor c = acz::blob_from_bytes(blob, size);
        acz::Tensor t = acz::decompress(c, zero_filter != 0);
        if (t.size() != n) throw acz::ShapeError("output size mismatch");
        std::memcpy(out, t.data(), n * sizeof(float));
    });
}

// Huffman encode of an arbitrary u32 stream: codebook (sym,len) arrays + packed bits.
int ref_huffman_encode(const std::uint32_t* syms, std::uint64_t n, std::uint32_t** book_sym,
                       std::uint8_t** book_len, std::uint64_t* book_size, std::uint8_t** bits,
                       std::uint64_t* bit_length, char* err, int errcap) {
    return guarded(err, errcap, [&] {
        std::vector<std::uint32_t> s(syms, syms + n);
        acz::HuffmanCode h = acz::huffman_encode(s);
        *book_size = h.codebook.size();
        *book_sym = static_cast<std::uint32_t*>(std::malloc(4 * (h.codebook.size() + 1)));
        *book_len = static_cast<std::uint8_t*>(std::malloc(h.codebook.size() + 1));
        for (std::size_t i = 0; i < h.codebook.size(); ++i) {
            (*book_sym)[i] = h.codebook[i].symbol;
            (*book_len)[i] = h.codebook[i].length;
        }
        *bits = static_cast<std::uint8_t*>(std::malloc(h.bits.size() + 1));
        std::memcpy(*bits, h.bits.data(), h.bits.size());
        *bit_length = h.bit_length;
    });
}

int ref_huffman_decode(const std::uint32_t* book_sym, const std::uint8_t* book_len,
                       std::uint64_t book_size, const std::uint8_t* bits,
                       std::uint64_t bit_length, std::uint64_t count, std::uint32_t* out,
                       char* err, int errcap) {
    return guarded(err, errcap, [&] {
        std::vector<acz::CodebookEntry> book(book_size);
        for (std::size_t i = 0; i < book_size; ++i) book[i] = {book_sym[i], book_len[i]};
        auto v = acz::huffman_decode(book, bits, bit_length, count);
        std::memcpy(out, v.data(), v.size() * 4);
    });
}

int ref_nonzero_ratio(const float* x, std::uint64_t n, double* r, char* err, int errcap) {
    return guarded(err, errcap, [&] {
        acz::Tensor t({static_cast<std::size_t>(n)}, std::vector<float>(x, x + n));
        *r = acz::nonzero_ratio(t);
    });
}

int ref_mean_abs(const float* x, std::uint64_t n, double* r, char* err, int errcap) {
    return guarded(err, errcap, [&] {
        acz::Tensor t({static_cast<std::size_t>(n)}, std::vector<float>(x, x + n));
        *r = acz::mean_abs(t);
    });
}

// CPU baseline: round trip (compress + decompress with zero filter) of a batch-sharded
// tensor. The leading dimension is split into `shards` contiguous pieces; `threads`
// std::threads each take shards round-robin and call the pure reference API
// (SPEC.md:157-158). Returns total ACZ1 bytes and wall seconds (steady_clock).
int ref_roundtrip_sharded(const float* x, const std::uint64_t* shape, int rank, double eb,
                          std::uint32_t radius, int predictor, int shards, int threads,
                          std::uint64_t* total_blob_bytes, double* seconds, char* err,
                          int errcap) {
    return guarded(err, errcap, [&] {
        if (rank < 1 || shards < 1 || threads < 1) throw acz::ParamError("bad shard args");
        std::size_t lead = shape[0];
        if (static_cast<std::size_t>(shards) > lead) shards = static_cast<int>(lead);
        std::size_t inner = volume(shape, rank) / lead;
        std::vector<std::uint64_t> bytes(static_cast<std::size_t>(shards), 0);
        std::vector<std::string> errs(static_cast<std::size_t>(threads));
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int w = 0; w < threads; ++w) {
            pool.emplace_back([&, w] {
                try {
                    for (int s = w; s < shards; s += threads) {
                        std::size_t b0 = lead * static_cast<std::size_t>(s) / shards;
                        std::size_t b1 = lead * static_cast<std::size_t>(s + 1) / shards;
                        std::vector<std::size_t> sh = to_shape(shape, rank);
                        sh[0] = b1 - b0;
                        acz::Tensor t(sh, std::vector<float>(x + b0 * inner, x + b1 * inner));
                        acz::CodecParams p{eb, radius, static_cast<acz::Predictor>(predictor)};
                        acz::CompressedTensor c = acz::compress(t, p);
                        bytes[static_cast<std::size_t>(s)] = c.compressed_bytes;
                        acz::Tensor d = acz::decompress(c, true);
                        if (d.size() != t.size()) throw acz::ShapeError("size");
                    }
                } catch (const std::exception& e) {
                    errs[static_cast<std::size_t>(w)] = e.what();
                }
            });
        }
        for (auto& th : pool) th.join();
        auto t1 = std::chrono::steady_clock::now();
        for (auto& e : errs)
            if (!e.empty()) throw acz::Error(e);
        std::uint64_t tot = 0;
        for (auto b : bytes) tot += b;
        *total_blob_bytes = tot;
        *seconds = std::chrono::duration<double>(t1 - t0).count();
    });
}

// The UNMODIFIED reference controller (src/controller.cpp) on one layer: config knobs,
// collection at iteration 0 with host activation/loss/momentum, then `wraps` forward
// passes at iteration 1 (compress-or-pass-through + unwrap); returns the layer stats, the
// window's bound and sigma, and the ledger CSV after finalize() (malloc'd).
int ref_controller_run_ex(std::int64_t W, double sigma_fraction, double coefficient_a,
                          double eb_min, double eb_max, const float* act,
                          const std::uint64_t* shape, int rank, const float* loss,
                          std::uint64_t nloss, const float* mom, std::uint64_t nmom,
                          std::uint64_t batch, int wraps, int relu_recompute, int is_post_relu,
                          float* back_out, double* stats_out, char** csv, char* err,
                          int errcap) {
    return guarded(err, errcap, [&] {
        acz::ControllerConfig cfg;
        cfg.collect_interval = W;
        cfg.sigma_fraction = sigma_fraction;
        cfg.coefficient_a = coefficient_a;
        cfg.eb_min = eb_min;
        cfg.eb_max = eb_max;
        if (relu_recompute) cfg.zero_restoration = acz::ZeroRestoration::ReluRecompute;
        acz::Controller c(cfg, 1);
        const std::size_t n = volume(shape, rank);
        acz::Tensor ta(to_shape(shape, rank), std::vector<float>(act, act + n));
        acz::Tensor tl({static_cast<std::size_t>(nloss)}, std::vector<float>(loss, loss + nloss));
        acz::Tensor tm({static_cast<std::size_t>(nmom)}, std::vector<float>(mom, mom + nmom));
        c.begin_iteration(0);
        acz::LayerStats st = c.collect_stats(0, ta, tl, tm, static_cast<std::size_t>(batch));
        stats_out[0] = st.l_bar;
        stats_out[1] = st.r;
        stats_out[2] = st.m_avg;
        stats_out[3] = st.degenerate ? 1.0 : 0.0;
        c.begin_iteration(1);
        stats_out[4] = c.layer_eb(0);
        stats_out[5] = c.layer_active(0) ? 1.0 : 0.0;
        for (int i = 0; i < wraps; ++i) {
            acz::Tensor copy = ta;
            acz::ActivationHandle h = c.wrap_forward(0, std::move(copy), is_post_relu != 0);
            stats_out[6] = static_cast<double>(h.held_bytes);
            acz::Tensor back = c.unwrap_backward(h);
            if (back_out) std::memcpy(back_out, back.data(), back.size() * sizeof(float));
        }
        c.finalize();
        const std::string s = c.ledger().to_csv();
        *csv = static_cast<char*>(std::malloc(s.size() + 1));
        std::memcpy(*csv, s.c_str(), s.size() + 1);
    });
}

int ref_controller_run(std::int64_t W, double sigma_fraction, double coefficient_a,
                       double eb_min, double eb_max, const float* act, const std::uint64_t* shape,
                       int rank, const float* loss, std::uint64_t nloss, const float* mom,
                       std::uint64_t nmom, std::uint64_t batch, int wraps, double* stats_out,
                       char** csv, char* err, int errcap) {
    return ref_controller_run_ex(W, sigma_fraction, coefficient_a, eb_min, eb_max, act, shape,
                                 rank, loss, nloss, mom, nmom, batch, wraps, 0, 1, nullptr,
                                 stats_out, csv, err, errcap);
}

} // extern "C"
