// Drives the reference's OWN acz::Controller (src/controller.cpp, compiled unmodified) through
// a synthetic training loop: every iteration wrap_forward() every layer's activation, then
// unwrap_backward() in reverse order, collect_stats() on collection iterations
// (ref src/controller.cpp:124-253). Linked twice by oracle/Makefile (`dropin` target):
//   dropin_cpu : with the reference's src/codec.cpp           (the CPU codec)
//   dropin_gpu : with paper_2011_09017_b200/proj_core/gpu_codec.cpp over libacz_gpu.so
// Everything observable is printed (FNV-1a of every ACZ1 blob and every unwrapped tensor,
// held bytes, ratios, the ledger CSV, stash accounting, blob-file round trips and the
// exception class of corrupted blobs): tests/test_gpu_dropin.py requires identical output.
//
// usage: dropin_controller {filter|relu} {prev|lorenzo2d} [iterations]
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "acz/codec.hpp"
#include "acz/controller.hpp"
#include "acz/error.hpp"
#include "acz/rng.hpp"
#include "acz/tensor.hpp"

namespace {

std::uint64_t fnv(const void* p, std::size_t n) {
    const auto* b = static_cast<const std::uint8_t*>(p);
    std::uint64_t h = 1469598103934665603ull;
    for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}

struct Layer {
    std::vector<std::size_t> shape;
    bool post_relu;
    double loss_scale, mom_scale;
};

acz::Tensor make(const std::vector<std::size_t>& shape, std::uint64_t seed, bool relu,
                 double scale) {
    acz::Rng rng(seed);
    std::size_t n = 1;
    for (auto e : shape) n *= e;
    std::vector<float> v(n);
    for (auto& x : v) {
        double g = acz::normal01(rng) * scale;
        x = static_cast<float>(relu && g < 0 ? 0.0 : g);
    }
    return acz::Tensor(shape, std::move(v));
}

const char* error_class(const std::exception& e) {
    if (dynamic_cast<const acz::FormatError*>(&e)) return "FormatError";
    if (dynamic_cast<const acz::DecodeError*>(&e)) return "DecodeError";
    if (dynamic_cast<const acz::ParamError*>(&e)) return "ParamError";
    if (dynamic_cast<const acz::DomainError*>(&e)) return "DomainError";
    if (dynamic_cast<const acz::ShapeError*>(&e)) return "ShapeError";
    if (dynamic_cast<const acz::Error*>(&e)) return "Error";
    return "std::exception";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s {filter|relu} {prev|lorenzo2d} [iterations]\n", argv[0]);
        return 2;
    }
    acz::ControllerConfig cfg;
    cfg.collect_interval = 3;
    cfg.eb_min = 1e-5;
    cfg.eb_max = 1e-2;
    cfg.zero_restoration = std::strcmp(argv[1], "relu") == 0
                               ? acz::ZeroRestoration::ReluRecompute
                               : acz::ZeroRestoration::CodecFilter;
    cfg.predictor = std::strcmp(argv[2], "lorenzo2d") == 0 ? acz::Predictor::Lorenzo2d
                                                            : acz::Predictor::PrevValue;
    const int iters = argc > 3 ? std::atoi(argv[3]) : 7;
    // an image-like dense conv1 input, post-ReLU feature maps, a long-plane tensor (the
    // speculative quantiser) and a rank-2 one
    const std::vector<Layer> layers = {
        {{2, 3, 67, 71}, false, 1e-2, 3e-4},
        {{4, 16, 28, 28}, true, 1e-2, 5e-4},
        {{4, 32, 14, 14}, true, 2e-2, 2e-4},
        {{1, 2, 300, 400}, true, 1e-2, 6e-4},
        {{3, 1000}, true, 5e-3, 1e-4},
    };
    acz::Controller ctl(cfg, static_cast<int>(layers.size()));
    std::vector<std::uint8_t> last_blob;
    std::vector<std::size_t> last_shape;
    for (int it = 0; it < iters; ++it) {
        ctl.begin_iteration(it);
        std::vector<acz::Tensor> acts;
        std::vector<acz::ActivationHandle> handles;
        for (std::size_t l = 0; l < layers.size(); ++l) {
            const Layer& L = layers[l];
            acz::Tensor a = make(L.shape, acz::mix_seed(20201118, it * 16 + l), L.post_relu, 1.0);
            acts.push_back(a);
            acz::ActivationHandle h = ctl.wrap_forward(static_cast<int>(l), std::move(a),
                                                       L.post_relu);
            std::printf("wrap it=%d layer=%zu eb=%.17g kind=%s held=%zu ratio=%.17g", it, l,
                        ctl.layer_active(static_cast<int>(l)) ? ctl.layer_eb(static_cast<int>(l))
                                                              : 0.0,
                        h.blob ? "blob" : "raw", h.held_bytes, h.achieved_ratio);
            if (h.blob) {
                const auto bytes = acz::blob_to_bytes(*h.blob);
                std::printf(" acz1=%zu fnv=%016llx book=%zu bits=%llu outliers=%zu relu=%d filter=%d",
                            bytes.size(), static_cast<unsigned long long>(fnv(bytes.data(), bytes.size())),
                            h.blob->codebook.size(),
                            static_cast<unsigned long long>(h.blob->bit_length),
                            h.blob->outliers.size(), h.apply_relu ? 1 : 0, h.zero_filter ? 1 : 0);
                last_blob = bytes;
                last_shape = L.shape;
            }
            std::printf(" stash=%zu\n", ctl.current_stash_bytes());
            handles.push_back(std::move(h));
        }
        for (std::size_t l = layers.size(); l-- > 0;) {
            acz::Tensor back = ctl.unwrap_backward(handles[l]);
            double maxerr = 0.0;
            for (std::size_t i = 0; i < back.size(); ++i) {
                double d = std::abs(static_cast<double>(back[i]) - static_cast<double>(acts[l][i]));
                if (d > maxerr) maxerr = d;
            }
            std::printf("unwrap it=%d layer=%zu fnv=%016llx maxerr=%.17g stash=%zu\n", it, l,
                        static_cast<unsigned long long>(
                            fnv(back.data(), back.size() * sizeof(float))),
                        maxerr, ctl.current_stash_bytes());
            try {
                ctl.unwrap_backward(handles[l]);
                std::printf("  second unwrap: no error\n");
            } catch (const std::exception& e) {
                std::printf("  second unwrap: %s\n", error_class(e));
            }
        }
        if (ctl.collecting()) {
            for (std::size_t l = 0; l < layers.size(); ++l) {
                const Layer& L = layers[l];
                acz::Tensor loss = make(L.shape, acz::mix_seed(7, it * 16 + l), false, L.loss_scale);
                acz::Tensor mom = make({64, 9}, acz::mix_seed(9, it * 16 + l), false, L.mom_scale);
                const std::size_t batch = L.shape[0];
                acz::LayerStats s = ctl.collect_stats(static_cast<int>(l), acts[l], loss, mom, batch);
                std::printf("stats it=%d layer=%zu l_bar=%.17g r=%.17g m_avg=%.17g degenerate=%d\n",
                            it, l, s.l_bar, s.r, s.m_avg, s.degenerate ? 1 : 0);
            }
        }
    }
    ctl.finalize();
    std::printf("ledger\n%s", ctl.ledger().to_csv().c_str());
    std::printf("peak_stash=%zu total_in=%llu total_stored=%llu\n", ctl.peak_stash_bytes(),
                static_cast<unsigned long long>(ctl.total_bytes_in()),
                static_cast<unsigned long long>(ctl.total_bytes_stored()));

    // the ACZ1 wire format: file round trip, then decompress a blob parsed from bytes
    // (no decode sidecar on the GPU side: rebuilt on the device)
    if (!last_blob.empty()) {
        acz::CompressedTensor c = acz::blob_from_bytes(last_blob.data(), last_blob.size());
        const std::string path = std::string("/tmp/acz_dropin_") + argv[1] + "_" + argv[2] + ".acz";
        acz::write_blob_file(path, c);
        acz::CompressedTensor c2 = acz::read_blob_file(path);
        std::remove(path.c_str());
        for (int zf = 0; zf < 2; ++zf) {
            acz::Tensor d = acz::decompress(c2, zf != 0);
            std::printf("file round trip zf=%d fnv=%016llx ratio=%.17g\n", zf,
                        static_cast<unsigned long long>(fnv(d.data(), d.size() * sizeof(float))),
                        acz::compression_ratio(c2));
        }
        // corruptions: truncation, trailing byte, bad magic, flipped codebook length
        std::vector<std::vector<std::uint8_t>> bad;
        bad.push_back(std::vector<std::uint8_t>(last_blob.begin(), last_blob.end() - 3));
        bad.push_back(last_blob);
        bad.back().push_back(0);
        bad.push_back(last_blob);
        bad.back()[0] = 'X';
        for (std::size_t i = 0; i < bad.size(); ++i) {
            try {
                acz::CompressedTensor cb = acz::blob_from_bytes(bad[i].data(), bad[i].size());
                acz::Tensor d = acz::decompress(cb, true);
                std::printf("corrupt %zu: accepted fnv=%016llx\n", i,
                            static_cast<unsigned long long>(fnv(d.data(), d.size() * 4)));
            } catch (const std::exception& e) {
                std::printf("corrupt %zu: %s\n", i, error_class(e));
            }
        }
    }
    // parameter / domain errors through the public API
    try {
        acz::compress(make({2, 2}, 1, false, 1.0), acz::CodecParams{-1.0, 32768, acz::Predictor::PrevValue});
    } catch (const std::exception& e) {
        std::printf("bad eb: %s\n", error_class(e));
    }
    try {
        acz::compress(acz::Tensor(), acz::CodecParams{});
    } catch (const std::exception& e) {
        std::printf("empty: %s\n", error_class(e));
    }
    return 0;
}
