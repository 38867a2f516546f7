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

    // batch-size scheme
    CHECK(suggest_batch(256, 1000u << 20, 4000u << 20) == 1024);

    if (fails) {
        std::fprintf(stderr, "%d check(s) failed\n", fails);
        return 1;
    }
    std::printf("cpp host layer OK: ratio %.3f, max err %.3g\n", compression_ratio(c), maxerr);
    return 0;
}
