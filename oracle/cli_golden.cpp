// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// Golden-vector driver for the command-line drop-in (tests/test_cli.py): the
// reference's sfconv_cli cannot be built here (its argument-parser and JSON headers
// are not vendored), so this driver restates the two things its
// quantsim / bench subcommands do before calling the library -- seed the
// mt19937_64 stream and draw inputs with the 'gaussian' / 'onef' generators
// (proj/tools/sfconv_cli.cpp:43-85, 299-305, 370-374) -- and then calls the
// UNMODIFIED reference library (quantized_fast_conv2d quant.cpp:152-293,
// fast_conv2d conv.cpp:384-553, direct_conv2d conv.cpp:320-350), built from
// /root/reference/proj/src by oracle/Makefile.
//
//   cli_golden quantsim SEED ALGO BITS ACT FIL SEARCH GEN LAYERS
//       LAYERS = name:C:OC:H:W:K:PAD[,name:...]; one line per layer:
//       name mse snr_db saturations values_quantized   (%.17g)
//   cli_golden bench SEED ALGO GEN C OC SIZE PAD REDUCED
//       prints: rel multiplications tiles
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "sfconv/conv.hpp"
#include "sfconv/quant.hpp"
#include "sfconv/spec.hpp"

using sfconv::DenseTensor;

static void gaussian(DenseTensor& t, std::mt19937_64& rng) {
    std::normal_distribution<double> dist(0.0, 1.0);
    for (std::size_t i = 0; i < t.data.size(); ++i) t.data[i] = dist(rng);
}

static void onef(DenseTensor& t, std::mt19937_64& rng) {
    gaussian(t, rng);
    const int B = t.shape[0], C = t.shape[1], H = t.shape[2], W = t.shape[3];
    std::vector<double> tmp(std::size_t(H > W ? H : W));
    for (int it = 0; it < 3; ++it)
        for (int b = 0; b < B; ++b)
            for (int c = 0; c < C; ++c) {
                for (int h = 0; h < H; ++h) {
                    for (int w = 0; w < W; ++w) {
                        const int wl = w - 1 < 0 ? 0 : w - 1, wr = w + 1 > W - 1 ? W - 1 : w + 1;
                        tmp[w] = (t.at4(b, c, h, wl) + t.at4(b, c, h, w) + t.at4(b, c, h, wr)) / 3.0;
                    }
                    for (int w = 0; w < W; ++w) t.at4(b, c, h, w) = tmp[w];
                }
                for (int w = 0; w < W; ++w) {
                    for (int h = 0; h < H; ++h) {
                        const int hu = h - 1 < 0 ? 0 : h - 1, hd = h + 1 > H - 1 ? H - 1 : h + 1;
                        tmp[h] = (t.at4(b, c, hu, w) + t.at4(b, c, h, w) + t.at4(b, c, hd, w)) / 3.0;
                    }
                    for (int h = 0; h < H; ++h) t.at4(b, c, h, w) = tmp[h];
                }
            }
    double e = 0.0;
    for (double v : t.data) e += v * v;
    const double s = e > 0.0 ? std::sqrt(double(t.data.size()) / e) : 1.0;
    for (double& v : t.data) v *= s;
}

static void fill(DenseTensor& t, const std::string& gen, std::mt19937_64& rng) {
    if (gen == "onef") onef(t, rng);
    else gaussian(t, rng);
}

int main(int argc, char** argv) {
    try {
        const std::string mode = argc > 1 ? argv[1] : "";
        if (mode == "quantsim" && argc == 10) {
            std::mt19937_64 rng(std::strtoull(argv[2], nullptr, 0));
            const sfconv::AlgorithmSpec& spec = sfconv::catalog_algorithm(argv[3]);
            sfconv::QuantConfig cfg;
            cfg.bits = std::atoi(argv[4]);
            cfg.act_scope = std::string(argv[5]) == "frequency" ? sfconv::ActScaleScope::PerFrequency
                                                                 : sfconv::ActScaleScope::PerTensor;
            const std::string fil = argv[6];
            cfg.filter_scope = fil == "frequency"           ? sfconv::FilterScaleScope::PerFrequency
                               : fil == "channel-frequency" ? sfconv::FilterScaleScope::PerChannelFrequency
                                                            : sfconv::FilterScaleScope::PerChannel;
            cfg.search = std::string(argv[7]) == "mse" ? sfconv::ScaleSearch::MseGrid : sfconv::ScaleSearch::MinMax;
            const std::string gen = argv[8];
            std::stringstream layers(argv[9]);
            std::string item;
            while (std::getline(layers, item, ',')) {
                char name[128];
                int C, OC, H, W, K, pad;
                if (std::sscanf(item.c_str(), "%127[^:]:%d:%d:%d:%d:%d:%d", name, &C, &OC, &H, &W, &K, &pad) != 7)
                    return 2;
                DenseTensor x({1, C, H, W}), f({OC, C, K, K});
                fill(x, gen, rng);
                gaussian(f, rng);
                const sfconv::QuantReport r = sfconv::quantized_fast_conv2d(x, f, spec, pad, cfg);
                std::printf("%s %.17g %.17g %lld %lld\n", name, r.mse, r.snr_db, (long long)r.saturations,
                            (long long)r.values_quantized);
            }
            return 0;
        }
        if (mode == "bench" && argc == 10) {
            std::mt19937_64 rng(std::strtoull(argv[2], nullptr, 0));
            const sfconv::AlgorithmSpec& spec = sfconv::catalog_algorithm(argv[3]);
            const int C = std::atoi(argv[5]), OC = std::atoi(argv[6]), S = std::atoi(argv[7]), pad = std::atoi(argv[8]);
            DenseTensor x({1, C, S, S}), f({OC, C, spec.R, spec.R});
            fill(x, argv[4], rng);
            gaussian(f, rng);
            sfconv::ConvCounters ctr;
            sfconv::FastConvOptions o;
            o.reduced_products = std::atoi(argv[9]) != 0;
            o.counters = &ctr;
            const DenseTensor ref = sfconv::direct_conv2d(x, f, 1, pad);
            const DenseTensor fast = sfconv::fast_conv2d(x, f, spec, pad, o);
            double md = 0.0, mr = 0.0;
            for (std::size_t i = 0; i < ref.data.size(); ++i) {
                md = std::max(md, std::abs(ref.data[i] - fast.data[i]));
                mr = std::max(mr, std::abs(ref.data[i]));
            }
            std::printf("%.17g %lld %lld\n", md / std::max(mr, 1e-300), (long long)ctr.multiplications,
                        (long long)ctr.tiles);
            return 0;
        }
        std::fprintf(stderr, "usage: see the header of oracle/cli_golden.cpp\n");
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
