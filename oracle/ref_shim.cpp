// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// extern "C" shim over the *unmodified* reference library (sfconv, built from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets the
// Python test-suite, the golden-vector generator and bench.py's reference arm
// call the reference's own entry points through ctypes:
//
//   quantized_fast_conv2d   proj/src/quant.cpp:152-293
//   quantize_value          proj/src/quant.cpp:102-115
//   scale_minmax/mse_grid   proj/src/quant.cpp:117-134
//   frequency_energy        proj/src/quant.cpp:136-150
//   direct_conv2d           proj/src/conv.cpp:320-350
//   transform_filters       proj/src/conv.cpp:352-382
//   fast_conv2d             proj/src/conv.cpp:384-553
//   catalog_algorithm       proj/src/catalog.cpp:275-287
//   catalog_export_json     proj/src/catalog.cpp:562-591
//   execute_tile_exact      proj/src/catalog.cpp:403-414
//
// Every function returns 0 on success and a negative code when the reference
// threw; the exception text is kept in a thread-local buffer (ref_last_error).
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "sfconv/conv.hpp"
#include "sfconv/quant.hpp"
#include "sfconv/spec.hpp"

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, -1);
    } catch (const std::domain_error& e) {
        return fail(e, -2);
    } catch (const std::overflow_error& e) {
        return fail(e, -3);
    } catch (const std::exception& e) {
        return fail(e, -4);
    }
}

sfconv::DenseTensor make4(const double* p, int a, int b, int c, int d) {
    sfconv::DenseTensor t({a, b, c, d});
    std::memcpy(t.data.data(), p, t.data.size() * sizeof(double));
    return t;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_catalog_json(char* buf, int cap, uint64_t* hash) {
    return guarded([&] {
        std::string s = sfconv::catalog_export_json();
        if (hash) *hash = sfconv::catalog_hash();
        if (buf && cap > 0) {
            std::size_t n = std::min<std::size_t>(s.size(), std::size_t(cap - 1));
            std::memcpy(buf, s.data(), n);
            buf[n] = 0;
        }
        if (int(s.size()) >= cap) throw std::length_error("buffer too small");
    });
}

// dims: K, n_in, M, R, N, offset, a_denom, n_corrections, mults_full, mults_reduced
int ref_spec(const char* name, int64_t* dims, int64_t* bt, int64_t* g, int64_t* a) {
    return guarded([&] {
        const sfconv::AlgorithmSpec& s = sfconv::catalog_algorithm(name);
        dims[0] = s.K();
        dims[1] = s.n_in();
        dims[2] = s.M;
        dims[3] = s.R;
        dims[4] = s.N;
        dims[5] = s.offset;
        dims[6] = s.a_denom;
        dims[7] = int64_t(s.corrections.size());
        dims[8] = s.mults_full();
        dims[9] = s.mults_reduced();
        auto dump = [](const sfconv::RatMatrix& m, int64_t* out) {
            if (!out) return;
            for (std::size_t i = 0; i < m.a.size(); ++i) {
                if (m.a[i].den != 1) throw std::domain_error("non-integral spec entry");
                out[i] = m.a[i].num;
            }
        };
        dump(s.BT, bt);
        dump(s.G, g);
        dump(s.A, a);
    });
}

int ref_quantize_value(double v, double scale, int bits, int64_t* sat, int64_t* q) {
    return guarded([&] { *q = sfconv::quantize_value(v, scale, bits, sat); });
}

int ref_scale(const double* v, int64_t n, int bits, int mse_grid, double* out) {
    return guarded([&] {
        std::vector<double> vals(v, v + n);
        *out = mse_grid ? sfconv::scale_mse_grid(vals, bits) : sfconv::scale_minmax(vals, bits);
    });
}

int ref_frequency_energy(const double* x, int B, int C, int H, int W, const char* spec, int pad,
                         double* energy) {
    return guarded([&] {
        auto e = sfconv::frequency_energy(make4(x, B, C, H, W), sfconv::catalog_algorithm(spec), pad);
        std::memcpy(energy, e.data(), e.size() * sizeof(double));
    });
}

// report: mse, signal_energy, snr_db, saturations, values_quantized
int ref_quantized_fast_conv2d(const double* x, int B, int C, int H, int W, const double* w, int OC,
                              int IC, int R, const char* spec, int pad, int bits, int act_scope,
                              int filter_scope, int search, double* out, double* report) {
    return guarded([&] {
        sfconv::QuantConfig cfg;
        cfg.bits = bits;
        cfg.act_scope = sfconv::ActScaleScope(act_scope);
        cfg.filter_scope = sfconv::FilterScaleScope(filter_scope);
        cfg.search = sfconv::ScaleSearch(search);
        sfconv::QuantReport rep = sfconv::quantized_fast_conv2d(
            make4(x, B, C, H, W), make4(w, OC, IC, R, R), sfconv::catalog_algorithm(spec), pad, cfg);
        if (out) std::memcpy(out, rep.output.data.data(), rep.output.data.size() * sizeof(double));
        if (report) {
            report[0] = rep.mse;
            report[1] = rep.signal_energy;
            report[2] = rep.snr_db;
            report[3] = double(rep.saturations);
            report[4] = double(rep.values_quantized);
        }
    });
}

int ref_direct_conv2d(const double* x, int B, int C, int H, int W, const double* w, int OC, int IC,
                      int R, int stride, int pad, double* out) {
    return guarded([&] {
        auto y = sfconv::direct_conv2d(make4(x, B, C, H, W), make4(w, OC, IC, R, R), stride, pad);
        std::memcpy(out, y.data.data(), y.data.size() * sizeof(double));
    });
}

int ref_transform_filters(const double* w, int OC, int IC, int R, const char* spec, double* out) {
    return guarded([&] {
        auto u = sfconv::transform_filters(make4(w, OC, IC, R, R), sfconv::catalog_algorithm(spec));
        std::memcpy(out, u.data.data(), u.data.size() * sizeof(double));
    });
}

int ref_fast_conv2d(const double* x, int B, int C, int H, int W, const double* w, int OC, int IC,
                    int R, const char* spec, int pad, int threads, int reduced, double* out,
                    int64_t* mults) {
    return guarded([&] {
        sfconv::ConvCounters cnt;
        sfconv::FastConvOptions opt;
        opt.threads = threads;
        opt.reduced_products = reduced != 0;
        opt.counters = &cnt;
        auto y = sfconv::fast_conv2d(make4(x, B, C, H, W), make4(w, OC, IC, R, R),
                                     sfconv::catalog_algorithm(spec), pad, opt);
        std::memcpy(out, y.data.data(), y.data.size() * sizeof(double));
        if (mults) {
            mults[0] = cnt.multiplications;
            mults[1] = cnt.tiles;
        }
    });
}

int ref_execute_tile_exact(const char* spec, const int64_t* x, const int64_t* f, int64_t* y) {
    return guarded([&] {
        const sfconv::AlgorithmSpec& s = sfconv::catalog_algorithm(spec);
        std::vector<int64_t> xv(x, x + std::size_t(s.n_in()) * s.n_in());
        std::vector<int64_t> fv(f, f + std::size_t(s.R) * s.R);
        auto r = sfconv::execute_tile_exact(s, xv, fv);
        std::memcpy(y, r.data(), r.size() * sizeof(int64_t));
    });
}

int ref_validate(const char* spec, int trials, uint64_t seed, int64_t* mismatches) {
    return guarded([&] {
        auto rep = sfconv::validate_algorithm(sfconv::catalog_algorithm(spec), trials, seed);
        *mismatches = rep.mismatches;
        if (!rep.ok && rep.mismatches == 0) throw std::domain_error(rep.detail);
    });
}

}  // extern "C"
