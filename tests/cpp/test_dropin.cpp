// C++ tests of the sfconv:: drop-in (libsfc_b200.so) written against the reference's
// own API -- the same calls and expectations as proj/tests/test_quant.cpp,
// test_catalog.cpp and test_conv.cpp, on int8-valued tensors (the device path).
//
//   test_dropin            run all checks, print PASS/FAIL per case, exit 1 on failure
//   test_dropin run SPEC PAD BITS B C H W OC x.bin w.bin out.bin
//                          quantized_fast_conv2d on raw int8 inputs; writes the fp64
//                          output followed by {mse, signal_energy, snr_db, saturations,
//                          values_quantized} for tests/test_cpp_dropin.py
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iterator>
#include <limits>
#include <fstream>
#include <functional>
#include <random>
#include <stdexcept>
#include <thread>
#include <string>
#include <vector>

#include "sfconv/conv.hpp"
#include "sfconv/manifest.hpp"
#include "sfconv/quant.hpp"
#include "sfconv/spec.hpp"
#include "sfconv/tensor.hpp"

using namespace sfconv;

namespace {
int g_fail = 0, g_checks = 0;
bool g_host_only = false;  // --host-only: skip the cases that need a GPU
std::string g_case;

#define CHECK(cond)                                                                          \
    do {                                                                                     \
        ++g_checks;                                                                          \
        if (!(cond)) {                                                                       \
            ++g_fail;                                                                        \
            std::printf("  FAIL %s:%d [%s] %s\n", __FILE__, __LINE__, g_case.c_str(), #cond); \
        }                                                                                    \
    } while (0)

template <class E, class F>
bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

void run_case(const char* name, const std::function<void()>& fn, bool device = true) {
    if (device && g_host_only) {
        std::printf("[SKIP] %s\n", name);
        return;
    }
    g_case = name;
    const int before = g_fail;
    try {
        fn();
    } catch (const std::exception& e) {
        ++g_fail;
        std::printf("  FAIL [%s] unexpected exception: %s\n", name, e.what());
    }
    std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name);
}

DenseTensor int8_tensor(std::vector<int> shape, std::uint64_t seed, int lo = -128, int hi = 127) {
    DenseTensor t(std::move(shape));
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<int> d(lo, hi);
    for (auto& v : t.data) v = double(d(rng));
    return t;
}

DenseTensor naive_conv(const DenseTensor& x, const DenseTensor& f, int pad) {
    const int B = x.dim(0), C = x.dim(1), H = x.dim(2), W = x.dim(3), OC = f.dim(0), R = f.dim(2);
    const int HO = H + 2 * pad - R + 1, WO = W + 2 * pad - R + 1;
    DenseTensor y({B, OC, HO, WO});
    for (int b = 0; b < B; ++b)
        for (int o = 0; o < OC; ++o)
            for (int i = 0; i < HO; ++i)
                for (int j = 0; j < WO; ++j) {
                    double acc = 0;
                    for (int c = 0; c < C; ++c)
                        for (int u = 0; u < R; ++u)
                            for (int v = 0; v < R; ++v) {
                                const int ih = i - pad + u, iw = j - pad + v;
                                if (ih >= 0 && ih < H && iw >= 0 && iw < W) acc += x.at4(b, c, ih, iw) * f.at4(o, c, u, v);
                            }
                    y.at4(b, o, i, j) = acc;
                }
    return y;
}

double max_rel(const DenseTensor& got, const DenseTensor& want) {
    double m = 0, e = 0;
    for (std::size_t i = 0; i < want.data.size(); ++i) {
        m = std::max(m, std::abs(want.data[i]));
        e = std::max(e, std::abs(got.data[i] - want.data[i]));
    }
    return m > 0 ? e / m : e;
}

int run_mode(int argc, char** argv) {
    if (argc != 13 && argc != 16) {
        std::fprintf(stderr, "usage: test_dropin run SPEC PAD BITS B C H W OC [ACT FIL SEARCH] x.bin w.bin out.bin\n");
        return 2;
    }
    const int fa = argc == 16 ? 3 : 0;  // optional QuantConfig scopes before the file arguments
    const std::string spec = argv[2];
    const int pad = std::atoi(argv[3]), bits = std::atoi(argv[4]);
    const int B = std::atoi(argv[5]), C = std::atoi(argv[6]), H = std::atoi(argv[7]), W = std::atoi(argv[8]);
    const int OC = std::atoi(argv[9]);
    const bool f64 = std::getenv("SFC_TEST_F64") != nullptr;  // inputs are raw doubles, not int8
    auto load = [f64](const char* path, DenseTensor& t) {
        std::ifstream f(path, std::ios::binary);
        if (f64) {
            f.read(reinterpret_cast<char*>(t.data.data()), std::streamsize(t.data.size() * sizeof(double)));
            if (!f) throw std::runtime_error(std::string("short read: ") + path);
            return;
        }
        std::vector<int8_t> raw(t.data.size());
        f.read(reinterpret_cast<char*>(raw.data()), std::streamsize(raw.size()));
        if (!f) throw std::runtime_error(std::string("short read: ") + path);
        for (std::size_t i = 0; i < raw.size(); ++i) t.data[i] = double(raw[i]);
    };
    const AlgorithmSpec& s = catalog_algorithm(spec);
    DenseTensor x({B, C, H, W}), w({OC, C, s.R, s.R});
    load(argv[10 + fa], x);
    load(argv[11 + fa], w);
    QuantConfig cfg;
    cfg.bits = bits;
    if (fa) {
        cfg.act_scope = ActScaleScope(std::atoi(argv[10]));
        cfg.filter_scope = FilterScaleScope(std::atoi(argv[11]));
        cfg.search = ScaleSearch(std::atoi(argv[12]));
    }
    const QuantReport rep = quantized_fast_conv2d(x, w, s, pad, cfg);
    std::ofstream o(argv[12 + fa], std::ios::binary);
    o.write(reinterpret_cast<const char*>(rep.output.data.data()), std::streamsize(rep.output.data.size() * 8));
    const double tail[5] = {rep.mse, rep.signal_energy, rep.snr_db, double(rep.saturations),
                            double(rep.values_quantized)};
    o.write(reinterpret_cast<const char*>(tail), sizeof tail);
    return o ? 0 : 1;
}
}  // namespace

// test_dropin sfct-copy IN OUT: load_sfct then save_sfct (cross-checked against the Python writer)
int sfct_copy(int argc, char** argv) {
    if (argc != 4) return 2;
    try {
        save_sfct(argv[3], load_sfct(argv[2]));
    } catch (const std::runtime_error& e) {
        std::printf("%s\n", e.what());
        return 1;
    }
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 1 && std::string(argv[1]) == "run") return run_mode(argc, argv);
    if (argc > 1 && std::string(argv[1]) == "sfct-copy") return sfct_copy(argc, argv);
    g_host_only = argc > 1 && std::string(argv[1]) == "--host-only";

    run_case("catalog holds the SFC algorithms (test_catalog.cpp:31-39, catalog.cpp:246-250)", [] {
        const auto& n = catalog_names();
        CHECK((n == std::vector<std::string>{"sfc4-4x4-3x3", "sfc6-6x6-3x3", "sfc6-7x7-3x3", "sfc6-6x6-5x5",
                                             "sfc6-4x4-7x7"}));
        CHECK(catalog_algorithm("sfc6-6x6-5x5").R == 5 && catalog_algorithm("sfc6-4x4-7x7").R == 7);
        CHECK(throws<std::invalid_argument>([] { catalog_algorithm("wino-9x9-3x3"); }));
    }, false);

    run_case("SFCT round trip and error messages (test_tensor.cpp:38-83)", [] {
        const std::string path = "/tmp/sfc_dropin_test.sfct";
        DenseTensor t({2, 3, 4, 5});
        for (std::size_t i = 0; i < t.data.size(); ++i) t.data[i] = std::ldexp(double(i) - 60.5, int(i % 7) - 3);
        t.data[7] = -0.0;
        t.data[8] = 1e-308;
        t.data[9] = std::numeric_limits<double>::denorm_min();
        save_sfct(path, t);
        const DenseTensor u = load_sfct(path);
        CHECK(u.shape == t.shape);
        CHECK(std::memcmp(u.data.data(), t.data.data(), t.data.size() * 8) == 0);
        std::ifstream raw(path, std::ios::binary);
        std::string bytes((std::istreambuf_iterator<char>(raw)), std::istreambuf_iterator<char>());
        const std::string header = "{\"dtype\":\"f64\",\"layout\":\"row-major-nchw\",\"shape\":[2,3,4,5]}";
        CHECK(bytes.compare(0, 8, "SFCT0001") == 0);
        CHECK(std::uint8_t(bytes[8]) == header.size() && bytes[9] == 0 && bytes[10] == 0 && bytes[11] == 0);
        CHECK(bytes.compare(12, header.size(), header) == 0);
        CHECK(bytes.size() == 12 + header.size() + t.data.size() * 8);
        auto message = [](const std::string& p) {
            try {
                load_sfct(p);
            } catch (const std::runtime_error& e) {
                return std::string(e.what());
            }
            return std::string("no error");
        };
        { std::ofstream(path, std::ios::binary) << "NOTSFCT!xxxx"; }
        CHECK(message(path) == "not an SFCT file: " + path);
        { std::ofstream(path, std::ios::binary) << bytes.substr(0, 10); }
        CHECK(message(path) == "truncated SFCT header: " + path);
        { std::ofstream(path, std::ios::binary) << bytes.substr(0, bytes.size() - 1); }
        CHECK(message(path) == "truncated SFCT payload: " + path);
        std::string f32 = bytes;
        f32.replace(12 + 10, 3, "f32");
        { std::ofstream(path, std::ios::binary) << f32; }
        CHECK(message(path) == "unsupported SFCT dtype: f32");
        CHECK(message("/tmp/definitely_not_here.sfct") == "cannot open: /tmp/definitely_not_here.sfct");
        std::remove(path.c_str());
    }, false);

    run_case("layer lists and run manifests (test_tensor.cpp:85-131, manifest.cpp:7-16)", [] {
        const std::string path = "/tmp/sfc_dropin_layers.json";
        {
            std::ofstream o(path);
            o << "[{\"name\": \"a\", \"in_channels\": 3, \"out_channels\": 8, \"height\": 32, \"width\": 30,"
                 " \"kernel\": 3, \"padding\": 1}, {\"in_channels\": 2, \"out_channels\": 2, \"height\": 9,"
                 " \"width\": 9, \"kernel\": 5, \"stride\": 2}]";
        }
        const std::vector<LayerConfig> ls = load_layer_configs(path);
        CHECK(ls.size() == 2 && ls[0].name == "a" && ls[0].width == 30 && ls[0].padding == 1 && ls[0].stride == 1);
        CHECK(ls[1].name == "layer1" && ls[1].kernel == 5 && ls[1].stride == 2 && ls[1].padding == 0);
        const std::string js = layer_configs_to_json(ls);
        CHECK(js.rfind("[\n  {\n    \"height\": 32,\n    \"in_channels\": 3,\n    \"kernel\": 3,\n    \"name\": \"a\",", 0) == 0);
        { std::ofstream(path) << js; }
        const std::vector<LayerConfig> again = load_layer_configs(path);
        CHECK(again.size() == 2 && again[1].name == "layer1" && again[1].stride == 2);
        { std::ofstream(path) << "[{\"in_channels\": 0, \"out_channels\": 1, \"height\": 1, \"width\": 1, \"kernel\": 3}]"; }
        CHECK(throws<std::runtime_error>([&] { load_layer_configs(path); }));
        { std::ofstream(path) << "{\"in_channels\": 1}"; }
        CHECK(throws<std::runtime_error>([&] { load_layer_configs(path); }));
        CHECK(throws<std::runtime_error>([] { load_layer_configs("/nonexistent/layers.json"); }));
        std::remove(path.c_str());
        RunManifest m;
        m.command = "quantsim";
        m.seed = 0x5fc07751u;
        m.output_dir = "out";
        m.catalog_hash = 18446744073709551615ull;
        CHECK(m.to_json() == "{\n  \"catalog_hash\": 18446744073709551615,\n  \"command\": \"quantsim\",\n"
                             "  \"config_path\": \"\",\n  \"output_dir\": \"out\",\n  \"seed\": 1606448977\n}");
    }, false);

    run_case("channel and product counts (test_catalog.cpp:101-126)", [] {
        struct Row { const char* name; int K; long full, reduced; double pct; };
        for (const Row& r : {Row{"sfc4-4x4-3x3", 7, 49, 46, 31.94}, Row{"sfc6-6x6-3x3", 10, 100, 88, 27.16},
                             Row{"sfc6-7x7-3x3", 12, 144, 132, 29.93}}) {
            const AlgorithmSpec& s = catalog_algorithm(r.name);
            CHECK(s.K() == r.K && s.mults_full() == r.full && s.mults_reduced() == r.reduced);
            CHECK(std::abs(s.complexity_pct() - r.pct) < 0.01);
        }
    }, false);

    run_case("correction schedules (test_catalog.cpp:128-144)", [] {
        auto eq = [](const AlgorithmSpec& s, std::vector<CorrectionTerm> want) { return s.corrections == want; };
        CHECK(eq(catalog_algorithm("sfc6-6x6-3x3"), {{0, 0, 6, 0}, {5, 7, 1, 2}}));
        CHECK(eq(catalog_algorithm("sfc4-4x4-3x3"), {{0, 0, 4, 0}, {3, 5, 1, 2}}));
        CHECK(eq(catalog_algorithm("sfc6-7x7-3x3"), {{0, 0, 6, 0}, {6, 7, 1, 1}, {5, 7, 1, 2}, {6, 8, 2, 2}}));
        CHECK(derive_correction_spec(6, 6, 5).corrections.size() == 6);
        CHECK(derive_correction_spec(6, 4, 7).corrections.size() == 6);
    }, false);

    run_case("sfc6-6x6-3x3 window rows (test_catalog.cpp:165-187)", [] {
        const AlgorithmSpec& s = catalog_algorithm("sfc6-6x6-3x3");
        const std::int64_t bt[8][6] = {{1, 1, 1, 1, 1, 1},   {1, 1, 0, -1, -1, 0}, {0, -1, -1, 0, 1, 1},
                                       {1, 0, -1, -1, 0, 1}, {1, 0, -1, 1, 0, -1}, {0, -1, 1, 0, -1, 1},
                                       {1, -1, 0, 1, -1, 0}, {1, -1, 1, -1, 1, -1}};
        const std::int64_t g[8][3] = {{1, 1, 1}, {0, 1, 1}, {-1, -1, 0}, {-1, 0, 1},
                                      {-1, 0, 1}, {1, -1, 0}, {0, -1, 1}, {1, -1, 1}};
        CHECK(s.offset == 1 && s.a_denom == 6);
        for (int k = 0; k < 8; ++k) {
            CHECK(s.BT.at(k, 0) == Rat(0) && s.BT.at(k, 7) == Rat(0));
            for (int t = 0; t < 6; ++t) CHECK(s.BT.at(k, 1 + t) == Rat(bt[k][t]));
            for (int j = 0; j < 3; ++j) CHECK(s.G.at(k, j) == Rat(g[k][j]));
        }
    }, false);

    run_case("exactness gate, 1000 tiles each (acceptance.cpp:127-135)", [] {
        for (const auto& n : catalog_names()) {
            const ValidationReport r = validate_algorithm(catalog_algorithm(n), 1000, 0x5fc0de);
            CHECK(r.ok && r.mismatches == 0);
        }
        // derived larger kernels through the same construction (catalog.cpp:249-250)
        CHECK(validate_algorithm(derive_correction_spec(6, 6, 5), 200, 7).ok);
        CHECK(validate_algorithm(derive_correction_spec(6, 4, 7), 200, 7).ok);
    }, false);

    run_case("exact tile execution with large values (test_catalog.cpp:189-206)", [] {
        std::mt19937_64 rng(77);
        std::uniform_int_distribution<std::int64_t> big(-2000, 2000);
        const AlgorithmSpec& s = catalog_algorithm("sfc6-6x6-3x3");
        for (int trial = 0; trial < 10; ++trial) {
            std::vector<std::int64_t> x(64), f(9);
            for (auto& v : x) v = big(rng);
            for (auto& v : f) v = big(rng);
            const auto y = execute_tile_exact(s, x, f);
            for (int i = 0; i < 6; ++i)
                for (int j = 0; j < 6; ++j) {
                    std::int64_t want = 0;
                    for (int a = 0; a < 3; ++a)
                        for (int b = 0; b < 3; ++b) want += x[(i + a) * 8 + j + b] * f[a * 3 + b];
                    CHECK(y[i * 6 + j] == want);
                }
        }
    }, false);

    run_case("rounding is nearest-even (test_quant.cpp:34-42)", [] {
        std::int64_t sat = 0;
        CHECK(quantize_value(2.5, 1.0, 8, &sat) == 2);
        CHECK(quantize_value(3.5, 1.0, 8, &sat) == 4);
        CHECK(quantize_value(-2.5, 1.0, 8, &sat) == -2);
        CHECK(quantize_value(2.4999, 1.0, 8, &sat) == 2);
        CHECK(quantize_value(0.26, 0.1, 8, &sat) == 3);
        CHECK(sat == 0);
    }, false);

    run_case("clamping counts saturations (test_quant.cpp:44-58)", [] {
        std::int64_t sat = 0;
        CHECK(quantize_value(127.6, 1.0, 8, &sat) == 127 && sat == 1);
        CHECK(quantize_value(-130.0, 1.0, 8, &sat) == -128 && sat == 2);
        CHECK(quantize_value(9.0, 1.0, 4, &sat) == 7 && quantize_value(-9.0, 1.0, 4, &sat) == -8 && sat == 4);
    }, false);

    run_case("minmax scale (test_quant.cpp:60-72)", [] {
        std::vector<double> v{-3.0, 1.0, 2.0};
        CHECK(std::abs(scale_minmax(v, 8) - 3.0 / 127.0) < 1e-15);
        CHECK(scale_minmax(std::vector<double>(10, 0.0), 8) == 1e-8);
    }, false);

    run_case("direct_conv2d and transform_filters on the device (test_conv.cpp:194-209)", [] {
        const DenseTensor x = int8_tensor({2, 3, 9, 11}, 1), f = int8_tensor({4, 3, 3, 3}, 2, -127, 127);
        CHECK(max_rel(direct_conv2d(x, f, 1, 1), naive_conv(x, f, 1)) == 0.0);
        const AlgorithmSpec& s = catalog_algorithm("sfc6-7x7-3x3");
        const DenseTensor u = transform_filters(f, s);
        for (int o = 0; o < 4; ++o)
            for (int c = 0; c < 3; ++c)
                for (int k = 0; k < s.K(); ++k)
                    for (int l = 0; l < s.K(); ++l) {
                        double acc = 0;
                        for (int a = 0; a < 3; ++a)
                            for (int b = 0; b < 3; ++b)
                                acc += s.G.at(k, a).to_double() * f.at4(o, c, a, b) * s.G.at(l, b).to_double();
                        CHECK(u.at4(o, c, k, l) == acc);
                    }
        CHECK(throws<std::invalid_argument>([&] { transform_filters(DenseTensor({1, 1, 5, 5}), s); }));
    });

    run_case("constant input concentrates energy at DC (test_quant.cpp:97-107)", [] {
        DenseTensor x({1, 1, 14, 14});
        for (auto& v : x.data) v = 1.0;
        const auto e = frequency_energy(x, catalog_algorithm("sfc6-6x6-3x3"), 0);
        CHECK(e[0] == 1296.0);
        for (std::size_t i = 1; i < e.size(); ++i) CHECK(e[i] == 0.0);
    });

    run_case("quantized path tracks the exact conv at 8 bits (test_quant.cpp:109-125)", [] {
        const DenseTensor x = int8_tensor({1, 3, 14, 14}, 60), f = int8_tensor({4, 3, 3, 3}, 61, -127, 127);
        const AlgorithmSpec& s = catalog_algorithm("sfc6-6x6-3x3");
        const QuantReport rep = quantized_fast_conv2d(x, f, s, 1, QuantConfig{});
        CHECK(rep.snr_db > 25.0);
        CHECK(rep.saturations == 0);
        const DenseTensor ref = naive_conv(x, f, 1);
        double err = 0, sig = 0;
        for (std::size_t i = 0; i < ref.data.size(); ++i) {
            err += (rep.output.data[i] - ref.data[i]) * (rep.output.data[i] - ref.data[i]);
            sig += ref.data[i] * ref.data[i];
        }
        CHECK(std::abs(rep.mse - err / double(ref.data.size())) <= 1e-9 * rep.mse);
        CHECK(std::abs(rep.snr_db - 10.0 * std::log10(rep.signal_energy / rep.mse)) < 1e-6);
        const int th = (14 + s.M - 1) / s.M, freqs = s.K() * s.K();
        CHECK(rep.values_quantized == 4 * 3 * freqs + th * th * 3 * freqs);
    });

    run_case("more bits, less error (test_quant.cpp:127-140)", [] {
        const DenseTensor x = int8_tensor({1, 2, 12, 12}, 62), f = int8_tensor({2, 2, 3, 3}, 63, -127, 127);
        double prev = 1e300;
        for (int bits : {4, 6, 8}) {
            QuantConfig cfg;
            cfg.bits = bits;
            const double mse = quantized_fast_conv2d(x, f, catalog_algorithm("sfc4-4x4-3x3"), 1, cfg).mse;
            CHECK(mse < prev);
            prev = mse;
        }
    });

    run_case("width limits and shape errors (test_quant.cpp:190-199)", [] {
        const DenseTensor x = int8_tensor({1, 1, 8, 8}, 68), f = int8_tensor({1, 1, 3, 3}, 69);
        const AlgorithmSpec& s = catalog_algorithm("sfc4-4x4-3x3");
        for (int bits : {1, 17}) {
            QuantConfig cfg;
            cfg.bits = bits;
            CHECK(throws<std::invalid_argument>([&] { quantized_fast_conv2d(x, f, s, 1, cfg); }));
        }
        CHECK(throws<std::invalid_argument>([&] { quantized_fast_conv2d(int8_tensor({1, 2, 8, 8}, 1), f, s, 1, {}); }));
        DenseTensor frac = x;  // real values take the fp64 path (not refused)
        frac.data[0] = 0.5;
        CHECK(!throws<std::invalid_argument>([&] { quantized_fast_conv2d(frac, f, s, 1, {}); }));
        CHECK(throws<std::invalid_argument>([&] { fast_conv2d(x, int8_tensor({1, 1, 5, 5}, 2), s, 1); }));
    });

    run_case("fast_conv2d matches the direct method (test_conv.cpp:78-90)", [] {
        std::mt19937_64 rng(73);
        std::normal_distribution<double> nd(0.0, 1.0);
        for (const std::string& name : catalog_names()) {
            const AlgorithmSpec& s = catalog_algorithm(name);
            DenseTensor x({2, 3, 17, 15}), f({4, 3, s.R, s.R});
            for (auto& v : x.data) v = nd(rng);
            for (auto& v : f.data) v = nd(rng);
            const int pad = s.R / 2;
            ConvCounters cnt;
            FastConvOptions opts;
            opts.counters = &cnt;
            const DenseTensor a = fast_conv2d(x, f, s, pad, opts), b = direct_conv2d(x, f, 1, pad);
            double md = 0.0, mr = 0.0;
            for (std::size_t i = 0; i < b.data.size(); ++i) {
                md = std::max(md, std::abs(a.data[i] - b.data[i]));
                mr = std::max(mr, std::abs(b.data[i]));
            }
            CHECK(md / mr <= 1e-10);
            const int th = (17 + 2 * pad - s.R + 1 + s.M - 1) / s.M, tw = (15 + 2 * pad - s.R + 1 + s.M - 1) / s.M;
            CHECK(cnt.tiles == 2 * th * tw && cnt.multiplications == cnt.tiles * 4 * 3 * s.K() * s.K());
        }
    });

    run_case("reduced schedule skips the paired products and changes nothing else (test_conv.cpp:140-162)", [] {
        std::mt19937_64 rng(91);
        std::normal_distribution<double> nd(0.0, 1.0);
        DenseTensor x({1, 2, 20, 20});
        for (auto& v : x.data) v = nd(rng);
        for (const std::string& name : catalog_names()) {
            const AlgorithmSpec& s = catalog_algorithm(name);
            DenseTensor f({3, 2, s.R, s.R});
            for (auto& v : f.data) v = nd(rng);
            ConvCounters full_ctr, red_ctr;
            FastConvOptions full_opts, red_opts;
            full_opts.counters = &full_ctr;
            red_opts.counters = &red_ctr;
            red_opts.reduced_products = true;
            const DenseTensor yf = fast_conv2d(x, f, s, 1, full_opts), yr = fast_conv2d(x, f, s, 1, red_opts);
            double md = 0.0, mr = 0.0;
            for (std::size_t i = 0; i < yf.data.size(); ++i) {
                md = std::max(md, std::abs(yr.data[i] - yf.data[i]));
                mr = std::max(mr, std::abs(yf.data[i]));
            }
            CHECK(md / mr < 1e-12);
            CHECK(full_ctr.multiplications == s.mults_full() * full_ctr.tiles * 2 * 3);
            CHECK(red_ctr.multiplications == s.mults_reduced() * red_ctr.tiles * 2 * 3);
            CHECK(red_ctr.multiplications < full_ctr.multiplications);
        }
    });

    run_case("bitwise determinism across calls and threads (test_conv.cpp:177-192)", [] {
        const DenseTensor x = int8_tensor({2, 16, 20, 20}, 70), f = int8_tensor({8, 16, 3, 3}, 71, -127, 127);
        const AlgorithmSpec& s = catalog_algorithm("sfc6-7x7-3x3");
        const QuantReport a = quantized_fast_conv2d(x, f, s, 1, {});
        QuantReport b;
        std::thread t([&] { b = quantized_fast_conv2d(x, f, s, 1, {}); });
        t.join();
        CHECK(a.output.data == b.output.data);
    });

    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
