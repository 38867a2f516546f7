// C++ host-layer test (paper_2011_09017_b200/cpp/acz_b200.hpp over libacz_gpu.so). Needs a
// GPU. Writes the ACZ1 bytes of a seeded input to <outdir>/host.acz1 (+ the input as
// host.f32) so tests/test_gpu_cpp_host.py can byte-compare them with the oracle.
#include <cassert>
#include <cmath>
#include <cstdio>
#include <random>
#include <string>

#include "acz_b200.hpp"

using namespace acz_b200;

static int fails = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        if (!(c)) {                                                           \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++fails;                                                          \
        }                                                                     \
    } while (0)

template <typename E, typename F>
static bool throws(F f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static Tensor relu_tensor(std::vector<size_t> shape, uint64_t seed) {
    std::mt19937_64 g(seed);
    std::normal_distribution<float> nd(0.0f, 1.0f);
    size_t n = 1;
    for (size_t e : shape) n *= e;
    std::vector<float> v(n);
    for (auto& x : v) x = std::max(0.0f, nd(g));
    return Tensor(std::move(shape), std::move(v));
}

int main(int argc, char** argv) {
    const std::string outdir = argc > 1 ? argv[1] : ".";
    Context& ctx = Context::thread_default();

    // ---- host codec: the reference's calling convention ----
    Tensor t = relu_tensor({4, 16, 56, 56}, 20201118);
    CodecParams p{1e-3, 32768, Predictor::PrevValue};
    CompressedTensor c = compress(t, p);
    CHECK(c.compressed_bytes == c.bytes.size());
    CHECK(compression_ratio(c) > 2.0);
    Tensor d0 = decompress(c, false);
    Tensor d1 = decompress(c, true);
    double maxerr = 0.0;
    for (size_t i = 0; i < t.size(); ++i) {
        maxerr = std::max(maxerr, std::fabs((double)t.data[i] - (double)d0.data[i]));
        if (t.data[i] == 0.0f) CHECK(d1.data[i] == 0.0f);  // zero preservation
        CHECK(std::fabs((double)t.data[i] - (double)d1.data[i]) <= 2 * p.eb);
    }
    CHECK(maxerr <= p.eb);
    {
        FILE* f = std::fopen((outdir + "/host.acz1").c_str(), "wb");
        std::fwrite(c.bytes.data(), 1, c.bytes.size(), f);
        std::fclose(f);
        f = std::fopen((outdir + "/host.f32").c_str(), "wb");
        std::fwrite(t.data.data(), 4, t.size(), f);
        std::fclose(f);
    }
    // blob_from_bytes round trip + validation errors (ref src/codec.cpp:201-262)
    CompressedTensor c2 = blob_from_bytes(c.bytes.data(), c.bytes.size());
    CHECK(c2.shape == c.shape && c2.params.eb == p.eb && c2.compressed_bytes == c.compressed_bytes);
    std::vector<uint8_t> bad = c.bytes;
    bad[0] = 'X';
    CHECK(throws<FormatError>([&] { blob_from_bytes(bad.data(), bad.size()); }));
    bad = c.bytes;
    bad.push_back(0);
    CHECK(throws<FormatError>([&] { blob_from_bytes(bad.data(), bad.size()); }));

    // ---- error mapping (ref include/acz/error.hpp) ----
    CHECK(throws<ParamError>([&] { compress(t, CodecParams{0.0, 32768, Predictor::PrevValue}); }));
    CHECK(throws<ParamError>([&] { compress(t, CodecParams{1e-3, 1000, Predictor::PrevValue}); }));
    Tensor tn = t;
    tn.data[77] = std::nanf("");
    CHECK(throws<DomainError>([&] { compress(tn, p); }));

    // ---- device path ----
    DeviceTensor dt = DeviceTensor::from_host(t, ctx);
    DeviceBlob db = compress(dt, p, ctx);
    CHECK(db.to_bytes(ctx) == c.bytes);
    Tensor dd = decompress(db, true, ctx).to_host();
    CHECK(dd.data == d1.data);
    CHECK(std::fabs(nonzero_ratio(dt, ctx) - 0.5) < 0.01);

    // ---- controller (ref src/controller.cpp) ----
    ControllerConfig cfg;
    cfg.collect_interval = 2;
    Controller ctl(cfg, 2, ctx);
    CHECK(throws<ParamError>([&] { Controller(ControllerConfig{0}, 1, ctx); }));
    Tensor loss = relu_tensor({4, 16, 56, 56}, 7), mom = relu_tensor({64, 16, 3, 3}, 8);
    for (auto& v : loss.data) v *= 1e-3f;
    for (auto& v : mom.data) v *= 1e-2f;
    DeviceTensor dl = DeviceTensor::from_host(loss, ctx), dm = DeviceTensor::from_host(mom, ctx);
    ctl.begin_iteration(0);
    CHECK(ctl.collecting());
    LayerStats st = ctl.collect_stats(0, dt, dl, dm, 4);
    CHECK(!st.degenerate);
    double la = 0, ma = 0;
    size_t nz = 0;
    for (float v : loss.data) la += std::fabs((double)v);
    for (float v : mom.data) ma += std::fabs((double)v);
    for (float v : t.data) nz += v != 0.0f;
    la /= loss.size();
    ma /= mom.size();
    CHECK(std::fabs(st.l_bar - la) <= 1e-12 * la);
    CHECK(std::fabs(st.m_avg - ma) <= 1e-12 * ma);
    CHECK(st.r == (double)nz / (double)t.size());
    const double sigma = cfg.sigma_fraction * st.m_avg;
    const double eb_expect =
        std::clamp(sigma / (cfg.coefficient_a * st.l_bar * std::sqrt(4.0 * st.r)), cfg.eb_min, cfg.eb_max);
    CHECK(!ctl.layer_active(0));  // the collection iteration itself runs uncompressed
    ctl.begin_iteration(1);
    CHECK(ctl.layer_active(0) && !ctl.layer_active(1));
    CHECK(std::fabs(ctl.layer_eb(0) - eb_expect) <= 1e-15 * eb_expect);
    {
        DeviceTensor a = DeviceTensor::from_host(t, ctx);
        ActivationHandle h = ctl.wrap_forward(0, std::move(a), true);
        CHECK(h.blob.has_value() && !h.raw.has_value() && a.empty());
        CHECK(ctl.current_stash_bytes() == h.held_bytes && h.achieved_ratio > 1.0);
        Tensor back = ctl.unwrap_backward(h).to_host();
        for (size_t i = 0; i < t.size(); ++i)
            CHECK(std::fabs((double)t.data[i] - (double)back.data[i]) <= 2 * ctl.layer_eb(0));
        CHECK(ctl.current_stash_bytes() == 0);
        CHECK(throws<ParamError>([&] { ctl.unwrap_backward(h); }));
        DeviceTensor a2 = DeviceTensor::from_host(t, ctx);
        ActivationHandle h2 = ctl.wrap_forward(1, std::move(a2), true);  // inactive: pass-through
        CHECK(h2.raw.has_value() && h2.held_bytes == 4 * t.size());
        ctl.unwrap_backward(h2);
    }
    ctl.finalize();
    CHECK(ctl.ledger().records().size() == 1);
    CHECK(ctl.ledger().to_csv().rfind("iteration,layer,eb,predicted_sigma,L_bar,R,M_avg,ratio,fallback_flag\n", 0) == 0);
    // distributed statistics: two identical ranks (sums doubled) -> same ratios, batch 2N
    Controller ctl2(cfg, 1, ctx);
    ctl2.set_stats_reducer([](double* s, size_t n) {
        for (size_t i = 0; i < n; ++i) s[i] *= 2.0;
    });
    ctl2.begin_iteration(0);
    LayerStats s2 = ctl2.collect_stats(0, dt, dl, dm, 4);
    CHECK(s2.batch == 8 && std::fabs(s2.l_bar - st.l_bar) <= 1e-15 * st.l_bar && s2.r == st.r);
    ctl2.begin_iteration(1);
    CHECK(std::fabs(ctl2.layer_eb(0) * std::sqrt(2.0) - ctl.layer_eb(0)) <= 1e-12 * ctl.layer_eb(0) ||
          ctl.layer_eb(0) == 0.0);
    // batch-size scheme
    CHECK(suggest_batch(256, 1000u << 20, 4000u << 20) == 1024);

    if (fails) {
        std::fprintf(stderr, "%d check(s) failed\n", fails);
        return 1;
    }
    std::printf("cpp host layer OK: ratio %.3f, max err %.3g, eb %.3g\n", compression_ratio(c), maxerr,
                eb_expect);
    return 0;
}
