// sfconv:: drop-in over the B200 C-ABI (include/sfc_b200.h).
//
// Same signatures, argument meaning and exception types as the reference's
// proj/include/sfconv/{spec,conv,quant}.hpp.  The numerical stages run on the
// device (libsfc_b200.so kernels); this file only converts DenseTensor <-> int8
// device buffers and maps C-ABI error codes onto the reference's exceptions.
// Calls are synchronous and use the per-thread default stream, so concurrent
// host threads do not serialise on one stream.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

#include "../../include/sfc_b200.h"
#include "../../include/sfconv/quant.hpp"
#include "plan.hpp"

namespace sfconv {

// ============================================================================ rationals
RatMatrix::RatMatrix(std::initializer_list<std::initializer_list<std::int64_t>> init) {
    rows = int(init.size());
    cols = rows ? int(init.begin()->size()) : 0;
    for (const auto& r : init) {
        if (int(r.size()) != cols) throw std::invalid_argument("ragged matrix initializer");
        for (std::int64_t v : r) a.emplace_back(v);
    }
}

RatMatrix RatMatrix::identity(int n) {
    RatMatrix m(n, n);
    for (int i = 0; i < n; ++i) m.at(i, i) = Rat(1);
    return m;
}

RatMatrix RatMatrix::transposed() const {
    RatMatrix t(cols, rows);
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) t.at(j, i) = at(i, j);
    return t;
}

RatMatrix operator*(const RatMatrix& x, const RatMatrix& y) {
    if (x.cols != y.rows) throw std::invalid_argument("matrix dimension mismatch");
    RatMatrix r(x.rows, y.cols);
    for (int i = 0; i < x.rows; ++i)
        for (int k = 0; k < x.cols; ++k)
            if (!x.at(i, k).is_zero())
                for (int j = 0; j < y.cols; ++j) r.at(i, j) += x.at(i, k) * y.at(k, j);
    return r;
}

std::vector<double> RatMatrix::to_double() const {
    std::vector<double> d(a.size());
    for (std::size_t i = 0; i < a.size(); ++i) d[i] = a[i].to_double();
    return d;
}

namespace {
// Gauss-Jordan on an augmented system; returns the rank and leaves the reduced form.
int reduce(RatMatrix& m, int ncols, std::vector<int>& pivots) {
    int row = 0;
    pivots.clear();
    for (int col = 0; col < ncols && row < m.rows; ++col) {
        int p = row;
        while (p < m.rows && m.at(p, col).is_zero()) ++p;
        if (p == m.rows) continue;
        for (int j = 0; j < m.cols; ++j) std::swap(m.at(p, j), m.at(row, j));
        const Rat inv = Rat(1) / m.at(row, col);
        for (int j = 0; j < m.cols; ++j) m.at(row, j) = m.at(row, j) * inv;
        for (int r = 0; r < m.rows; ++r) {
            if (r == row || m.at(r, col).is_zero()) continue;
            const Rat f = m.at(r, col);
            for (int j = 0; j < m.cols; ++j) m.at(r, j) -= f * m.at(row, j);
        }
        pivots.push_back(col);
        ++row;
    }
    return row;
}
}  // namespace

RatMatrix RatMatrix::inverse() const {
    if (rows != cols) throw std::invalid_argument("inverse of non-square matrix");
    RatMatrix aug(rows, 2 * rows);
    for (int i = 0; i < rows; ++i) {
        for (int j = 0; j < rows; ++j) aug.at(i, j) = at(i, j);
        aug.at(i, rows + i) = Rat(1);
    }
    std::vector<int> piv;
    if (reduce(aug, rows, piv) != rows) throw std::domain_error("singular matrix");
    RatMatrix inv(rows, rows);
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < rows; ++j) inv.at(i, j) = aug.at(i, rows + j);
    return inv;
}

std::vector<Rat> solve_exact(const RatMatrix& M, const std::vector<Rat>& b) {
    if (int(b.size()) != M.rows) throw std::invalid_argument("solve_exact: rhs size mismatch");
    RatMatrix aug(M.rows, M.cols + 1);
    for (int i = 0; i < M.rows; ++i) {
        for (int j = 0; j < M.cols; ++j) aug.at(i, j) = M.at(i, j);
        aug.at(i, M.cols) = b[i];
    }
    std::vector<int> piv;
    const int rank = reduce(aug, M.cols, piv);
    for (int r = rank; r < M.rows; ++r)
        if (!aug.at(r, M.cols).is_zero()) throw std::domain_error("solve_exact: inconsistent system");
    std::vector<Rat> x(M.cols, Rat(0));
    for (int r = 0; r < rank; ++r) x[piv[r]] = aug.at(r, M.cols);
    return x;
}

// ============================================================================ helpers
namespace {

void check(int rc) {
    if (rc == SFC_OK) return;
    const std::string msg = sfc_last_error();
    if (rc == SFC_ERR_INVALID || rc == SFC_ERR_UNSUPPORTED) throw std::invalid_argument(msg);
    if (rc == SFC_ERR_DOMAIN) throw std::domain_error(msg);
    throw std::runtime_error(msg);
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    explicit DevBuf(std::size_t n) { ck(cudaMalloc(&p, (n ? n : 1) * sizeof(T)), "cudaMalloc"); }
    ~DevBuf() { cudaFree(p); }
    DevBuf(DevBuf&& o) noexcept : p(o.p) { o.p = nullptr; }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

cudaStream_t stream() { return cudaStreamPerThread; }

// DenseTensor (fp64) -> int8 device copy; the device path takes int8-valued tensors.
DevBuf<int8_t> to_device_int8(const DenseTensor& t, const char* what) {
    std::vector<int8_t> h(t.data.size());
    for (std::size_t i = 0; i < h.size(); ++i) {
        const double v = t.data[i];
        if (!(v == std::nearbyint(v)) || v < -128.0 || v > 127.0)
            throw std::invalid_argument(std::string(what) + ": the B200 path needs int8-valued tensors");
        h[i] = int8_t(v);
    }
    DevBuf<int8_t> d(h.size());
    ck(cudaMemcpyAsync(d.p, h.data(), h.size(), cudaMemcpyHostToDevice, stream()), "copy to device");
    return d;
}

bool int8_valued(const DenseTensor& t) {
    for (double v : t.data)
        if (!(v == std::nearbyint(v)) || v < -128.0 || v > 127.0) return false;
    return true;
}

DevBuf<double> to_device_f64(const DenseTensor& t) {
    DevBuf<double> d(t.data.size());
    ck(cudaMemcpyAsync(d.p, t.data.data(), t.data.size() * sizeof(double), cudaMemcpyHostToDevice, stream()),
       "copy to device");
    return d;
}

template <class T>
std::vector<T> to_host(const T* d, std::size_t n) {
    std::vector<T> h(n);
    ck(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, stream()), "copy to host");
    ck(cudaStreamSynchronize(stream()), "sync");
    return h;
}

void check_conv_shapes(const DenseTensor& input, const DenseTensor& filters) {  // conv.cpp:17-24
    if (input.shape.size() != 4 || filters.shape.size() != 4)
        throw std::invalid_argument("conv2d expects 4-d NCHW tensors");
    if (filters.shape[2] != filters.shape[3]) throw std::invalid_argument("conv2d expects square filters");
    if (input.shape[1] != filters.shape[1]) throw std::invalid_argument("input channel count does not match filters");
}

sfc_plan_t plan_handle(const AlgorithmSpec& spec) {
    sfc_plan_t p = nullptr;
    check(sfc_plan_create(spec.name.c_str(), &p));
    return p;
}

struct PlanGuard {
    sfc_plan_t p;
    ~PlanGuard() { sfc_plan_destroy(p); }
};

AlgorithmSpec spec_from_plan(const sfcb200::SfcPlan& p) {
    AlgorithmSpec s;
    s.name = p.name;
    s.family = AlgoFamily::Sfc;
    s.N = p.N;
    s.M = p.M;
    s.R = p.R;
    s.offset = p.offset;
    s.a_denom = p.a_denom;
    auto mat = [](const std::vector<int64_t>& v, int r, int c) {
        RatMatrix m(r, c);
        for (int i = 0; i < r * c; ++i) m.a[std::size_t(i)] = Rat(v[std::size_t(i)]);
        return m;
    };
    s.BT = mat(p.BT, p.K, p.n_in);
    s.G = mat(p.G, p.K, p.R);
    s.A = mat(p.A, p.K, p.M);
    s.overlap_form = mat(p.overlap, p.n_overlap, p.n_overlap);
    for (const auto& c : p.corrections) s.corrections.push_back({c.out, c.desired, c.wrapped, c.tap});
    for (std::size_t i = 0; i + 2 < p.triples.size(); i += 3)
        s.triples.push_back({p.triples[i], p.triples[i + 1], p.triples[i + 2]});
    return s;
}

std::uint64_t splitmix64(std::uint64_t& s) {
    std::uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

}  // namespace

// ============================================================================ catalog
AlgorithmSpec derive_correction_spec(int N, int M, int R) {
    if (N != 4 && N != 6) throw std::invalid_argument("derive_correction_spec: N must be 4 or 6");
    if (M + R - 1 < N) throw std::invalid_argument("derive_correction_spec: tile smaller than transform");
    return spec_from_plan(sfcb200::derive_sfc_plan(N, M, R));
}

const std::vector<std::string>& catalog_names() { return sfcb200::plan_names(); }

const AlgorithmSpec& catalog_algorithm(const std::string& name) {
    static std::mutex mu;
    static std::map<std::string, AlgorithmSpec> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(name);
    if (it != cache.end()) return it->second;
    return cache.emplace(name, spec_from_plan(sfcb200::plan_for(name))).first->second;
}

std::string catalog_export_json() { return sfcb200::plan_export_json(sfcb200::plan_names()); }
std::uint64_t catalog_hash() { return sfcb200::fnv1a64(catalog_export_json()); }

std::vector<std::int64_t> execute_tile_exact(const AlgorithmSpec& spec, const std::vector<std::int64_t>& x,
                                             const std::vector<std::int64_t>& f) {
    const int K = spec.K(), n = spec.n_in(), R = spec.R, M = spec.M;
    if (int(x.size()) != n * n) throw std::invalid_argument("bad input tile size");
    if (int(f.size()) != R * R) throw std::invalid_argument("bad filter tile size");
    for (const Rat& v : spec.BT.a)
        if (v.den != 1) throw std::invalid_argument("execute_tile_exact: non-integral transform");
    for (const Rat& v : spec.A.a)
        if (v.den != 1) throw std::invalid_argument("execute_tile_exact: non-integral transform");
    for (const Rat& v : spec.G.a)
        if (v.den != 1) throw std::invalid_argument("execute_tile_exact: non-integral transform");
    using I = __int128;
    std::vector<I> V(std::size_t(K) * K), U(std::size_t(K) * K), tmp(std::size_t(K) * n), tf(std::size_t(K) * R);
    for (int i = 0; i < K; ++i)
        for (int j = 0; j < n; ++j) {
            I acc = 0;
            for (int t = 0; t < n; ++t) acc += I(spec.BT.at(i, t).num) * x[std::size_t(t) * n + j];
            tmp[std::size_t(i) * n + j] = acc;
        }
    for (int i = 0; i < K; ++i)
        for (int j = 0; j < K; ++j) {
            I acc = 0;
            for (int t = 0; t < n; ++t) acc += tmp[std::size_t(i) * n + t] * spec.BT.at(j, t).num;
            V[std::size_t(i) * K + j] = acc;
        }
    for (int i = 0; i < K; ++i)
        for (int j = 0; j < R; ++j) {
            I acc = 0;
            for (int t = 0; t < R; ++t) acc += I(spec.G.at(i, t).num) * f[std::size_t(t) * R + j];
            tf[std::size_t(i) * R + j] = acc;
        }
    for (int i = 0; i < K; ++i)
        for (int j = 0; j < K; ++j) {
            I acc = 0;
            for (int t = 0; t < R; ++t) acc += tf[std::size_t(i) * R + t] * spec.G.at(j, t).num;
            U[std::size_t(i) * K + j] = acc;
        }
    std::vector<std::int64_t> y(std::size_t(M) * M);
    const I d2 = I(spec.a_denom) * spec.a_denom;
    for (int t1 = 0; t1 < M; ++t1)
        for (int t2 = 0; t2 < M; ++t2) {
            I acc = 0;
            for (int k = 0; k < K; ++k)
                for (int l = 0; l < K; ++l)
                    acc += I(spec.A.at(k, t1).num) * spec.A.at(l, t2).num * V[std::size_t(k) * K + l] *
                           U[std::size_t(k) * K + l];
            if (acc % d2 != 0) throw std::domain_error(spec.name + ": output not divisible by denominator fold");
            y[std::size_t(t1) * M + t2] = std::int64_t(acc / d2);
        }
    return y;
}

ValidationReport validate_algorithm(const AlgorithmSpec& spec, int trials, std::uint64_t seed) {
    ValidationReport rep;
    rep.trials = trials;
    const int n = spec.n_in(), R = spec.R, M = spec.M;
    std::uint64_t state = seed ^ 0x8f3c9a1d526bce07ULL;
    for (int tr = 0; tr < trials; ++tr) {
        std::vector<std::int64_t> x(std::size_t(n) * n), f(std::size_t(R) * R);
        for (auto& v : x) v = std::int64_t(splitmix64(state) % 17) - 8;
        for (auto& v : f) v = std::int64_t(splitmix64(state) % 17) - 8;
        std::vector<std::int64_t> got;
        try {
            got = execute_tile_exact(spec, x, f);
        } catch (const std::exception& e) {
            rep.detail = e.what();
            return rep;
        }
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < M; ++j) {
                std::int64_t want = 0;
                for (int a = 0; a < R; ++a)
                    for (int b = 0; b < R; ++b) want += x[std::size_t(i + a) * n + j + b] * f[std::size_t(a) * R + b];
                if (got[std::size_t(i) * M + j] != want) ++rep.mismatches;
            }
        if (rep.mismatches && rep.detail.empty()) rep.detail = "first mismatch at trial " + std::to_string(tr);
    }
    rep.ok = rep.mismatches == 0;
    return rep;
}

// ============================================================================ scalars
std::int64_t quantize_value(double v, double scale, int bits, std::int64_t* saturated) {
    const std::int64_t qmax = (std::int64_t(1) << (bits - 1)) - 1, qmin = -(std::int64_t(1) << (bits - 1));
    std::int64_t q = std::int64_t(std::nearbyint(v / scale));
    if (q > qmax || q < qmin) {
        q = q > qmax ? qmax : qmin;
        if (saturated) ++*saturated;
    }
    return q;
}

double scale_minmax(const std::vector<double>& values, int bits) {
    double m = 0.0;
    for (double v : values) m = std::max(m, std::abs(v));
    return std::max(m / double((std::int64_t(1) << (bits - 1)) - 1), 1e-8);
}

double scale_mse_grid(const std::vector<double>& values, int bits) {
    const double qmax = double((std::int64_t(1) << (bits - 1)) - 1), qmin = -double(std::int64_t(1) << (bits - 1));
    auto mse = [&](double s) {
        double err = 0.0;
        for (double v : values) {
            const double q = std::min(qmax, std::max(qmin, std::nearbyint(v / s)));
            const double d = v - q * s;
            err += d * d;
        }
        return err;
    };
    const double base = scale_minmax(values, bits);
    double best = base, best_err = mse(base);
    for (int i = 0; i < 100; ++i) {
        const double s = std::max(base * (0.3 + 0.7 * double(i) / 99.0), 1e-8);
        const double e = mse(s);
        if (e < best_err) best = s, best_err = e;
    }
    return best;
}

// ============================================================================ device entry points
DenseTensor direct_conv2d(const DenseTensor& input, const DenseTensor& filters, int stride, int padding) {
    check_conv_shapes(input, filters);
    if (stride < 1) throw std::invalid_argument("stride must be positive");
    const int B = input.dim(0), C = input.dim(1), H = input.dim(2), W = input.dim(3);
    const int OC = filters.dim(0), R = filters.dim(2);
    const int HO = (H + 2 * padding - R) / stride + 1, WO = (W + 2 * padding - R) / stride + 1;
    if (HO <= 0 || WO <= 0 || H + 2 * padding < R || W + 2 * padding < R)
        throw std::invalid_argument("filter larger than padded input");
    DenseTensor out({B, OC, HO, WO});
    if (!int8_valued(input) || !int8_valued(filters)) {
        // Real-valued tensors: fp64 direct convolution in conv.cpp:62-89's accumulation order.
        DevBuf<double> xd = to_device_f64(input), wd = to_device_f64(filters), yd(out.data.size());
        check(sfc_direct_conv_f64(xd.p, B, C, H, W, wd.p, OC, R, stride, padding, yd.p, stream()));
        out.data = to_host(yd.p, out.data.size());
        return out;
    }
    DevBuf<int8_t> x = to_device_int8(input, "input"), w = to_device_int8(filters, "filters");
    DevBuf<int32_t> y(out.data.size());
    check(sfc_direct_conv_int8(x.p, B, C, H, W, w.p, OC, R, stride, padding, y.p, stream()));
    const auto h = to_host(y.p, out.data.size());
    for (std::size_t i = 0; i < h.size(); ++i) out.data[i] = double(h[i]);
    return out;
}

DenseTensor transform_filters(const DenseTensor& filters, const AlgorithmSpec& spec) {
    if (filters.shape.size() != 4 || filters.dim(2) != spec.R || filters.dim(3) != spec.R)
        throw std::invalid_argument("filter shape does not match algorithm");
    PlanGuard plan{plan_handle(spec)};
    const int OC = filters.dim(0), IC = filters.dim(1), K = spec.K();
    DenseTensor u({OC, IC, K, K});
    if (!int8_valued(filters)) {
        DevBuf<double> wd = to_device_f64(filters), ud(u.data.size());
        check(sfc_transform_filters_f64(plan.p, wd.p, OC, IC, ud.p, stream()));
        u.data = to_host(ud.p, u.data.size());
        return u;
    }
    DevBuf<int8_t> w = to_device_int8(filters, "filters");
    DevBuf<int32_t> d(u.data.size());
    check(sfc_transform_filters_int8(plan.p, w.p, OC, IC, d.p, stream()));
    const auto h = to_host(d.p, u.data.size());
    for (std::size_t i = 0; i < h.size(); ++i) u.data[i] = double(h[i]);
    return u;
}

DenseTensor fast_conv2d(const DenseTensor& input, const DenseTensor& filters, const AlgorithmSpec& spec, int padding,
                        const FastConvOptions& opts) {
    check_conv_shapes(input, filters);
    if (filters.dim(2) != spec.R) throw std::invalid_argument("filter size does not match algorithm");
    const int B = input.dim(0), C = input.dim(1), H = input.dim(2), W = input.dim(3), OC = filters.dim(0);
    const int HO = H + 2 * padding - spec.R + 1, WO = W + 2 * padding - spec.R + 1;
    if (HO <= 0 || WO <= 0) throw std::invalid_argument("filter larger than padded input");
    PlanGuard plan{plan_handle(spec)};
    DevBuf<double> x = to_device_f64(input), w = to_device_f64(filters);
    DenseTensor out({B, OC, HO, WO});
    DevBuf<double> d_out(out.data.size());
    std::int64_t counters[2] = {0, 0};
    check(sfc_fast_conv_f64(plan.p, x.p, B, C, H, W, w.p, OC, padding, opts.reduced_products ? 1 : 0, d_out.p,
                            counters, stream()));
    ck(cudaMemcpyAsync(out.data.data(), d_out.p, out.data.size() * sizeof(double), cudaMemcpyDeviceToHost,
                       stream()),
       "copy output");
    ck(cudaStreamSynchronize(stream()), "sync");
    if (opts.counters) {  // opts.threads is a host-CPU knob: the device result does not depend on it
        opts.counters->multiplications += counters[0];
        opts.counters->tiles += counters[1];
    }
    return out;
}

std::vector<double> frequency_energy(const DenseTensor& input, const AlgorithmSpec& spec, int padding) {
    if (input.shape.size() != 4) throw std::invalid_argument("conv2d expects 4-d NCHW tensors");
    const int B = input.dim(0), C = input.dim(1), H = input.dim(2), W = input.dim(3);
    const int HO = H + 2 * padding - spec.R + 1, WO = W + 2 * padding - spec.R + 1;
    if (HO <= 0 || WO <= 0) throw std::invalid_argument("filter larger than padded input");
    PlanGuard plan{plan_handle(spec)};
    DevBuf<int8_t> x = to_device_int8(input, "input");
    const int F = spec.K() * spec.K();
    DevBuf<unsigned long long> s{std::size_t(F)};
    ck(cudaMemsetAsync(s.p, 0, sizeof(unsigned long long) * F, stream()), "memset");
    check(sfc_frequency_energy_int8(plan.p, x.p, B, C, H, W, padding, s.p, stream()));
    const auto h = to_host(s.p, std::size_t(F));
    const double groups = double(B) * ((HO + spec.M - 1) / spec.M) * ((WO + spec.M - 1) / spec.M) * C;
    std::vector<double> e(static_cast<std::size_t>(F));
    for (int i = 0; i < F; ++i) e[std::size_t(i)] = double(h[std::size_t(i)]) / groups;
    return e;
}

// Real-valued tensors: V, U and the scales in the reference's own fp64 order on the device,
// the int8 contraction and the fp64 epilogue (sfc_layer_create_f64 / sfc_conv_forward_f64).
static QuantReport quantized_fast_conv2d_real(const DenseTensor& input, const DenseTensor& filters, const AlgorithmSpec& spec,
                                       int padding, const QuantConfig& config, sfc_plan_t plan) {
    const int B = input.dim(0), C = input.dim(1), H = input.dim(2), W = input.dim(3), OC = filters.dim(0);
    const int HO = H + 2 * padding - spec.R + 1, WO = W + 2 * padding - spec.R + 1;
    DevBuf<double> x = to_device_f64(input), w = to_device_f64(filters);
    sfc_layer_t layer = nullptr;
    check(sfc_layer_create_f64(plan, w.p, OC, C, config.bits, int(config.act_scope), int(config.filter_scope),
                               int(config.search), stream(), &layer));
    struct LayerGuard {
        sfc_layer_t l;
        ~LayerGuard() { sfc_layer_destroy(l); }
    } lg{layer};
    std::size_t ws_bytes = 0;
    check(sfc_conv_workspace_size(layer, B, H, W, padding, &ws_bytes));
    DevBuf<uint8_t> ws(ws_bytes);
    QuantReport rep;
    rep.output = DenseTensor({B, OC, HO, WO});
    const std::size_t n = rep.output.data.size();
    DevBuf<double> out(n), ref(n);
    sfc_outputs o{};
    o.out_f64 = out.p;
    check(sfc_conv_forward_f64(layer, x.p, B, H, W, padding, ws.p, ws_bytes, &o, stream()));
    check(sfc_direct_conv_f64(x.p, B, C, H, W, w.p, OC, spec.R, 1, padding, ref.p, stream()));
    double sums[2] = {0.0, 0.0};
    check(sfc_report_sq_err_f64(out.p, ref.p, int64_t(n), sums, stream()));
    std::int64_t stats[6] = {};
    check(sfc_conv_stats(layer, B, H, W, padding, ws.p, ws_bytes, stats, stream()));
    std::int64_t fsat = 0;
    check(sfc_layer_saturations(layer, &fsat));
    ck(cudaMemcpyAsync(rep.output.data.data(), out.p, n * sizeof(double), cudaMemcpyDeviceToHost, stream()),
       "copy output");
    ck(cudaStreamSynchronize(stream()), "sync");
    rep.mse = sums[0] / double(n);
    rep.signal_energy = sums[1] / double(n);
    rep.snr_db = 10.0 * std::log10(sums[1] / std::max(sums[0], 1e-300));
    rep.saturations = stats[2] + fsat;
    rep.values_quantized = stats[4];
    return rep;
}

QuantReport quantized_fast_conv2d(const DenseTensor& input, const DenseTensor& filters, const AlgorithmSpec& spec,
                                  int padding, const QuantConfig& config) {
    if (config.bits < 2 || config.bits > 16)  // quant.cpp:155-156
        throw std::invalid_argument("quantization width must be between 2 and 16 bits");
    check_conv_shapes(input, filters);
    if (filters.dim(2) != spec.R) throw std::invalid_argument("filter shape does not match algorithm");
    const int B = input.dim(0), C = input.dim(1), H = input.dim(2), W = input.dim(3), OC = filters.dim(0);
    const int HO = H + 2 * padding - spec.R + 1, WO = W + 2 * padding - spec.R + 1;
    if (HO <= 0 || WO <= 0) throw std::invalid_argument("filter larger than padded input");

    PlanGuard plan{plan_handle(spec)};
    if (!int8_valued(input) || !int8_valued(filters))
        return quantized_fast_conv2d_real(input, filters, spec, padding, config, plan.p);
    DevBuf<int8_t> x = to_device_int8(input, "input"), w = to_device_int8(filters, "filters");
    sfc_layer_t layer = nullptr;
    check(sfc_layer_create_ex(plan.p, w.p, OC, C, config.bits, int(config.act_scope), int(config.filter_scope),
                              int(config.search), stream(), &layer));
    struct LayerGuard {
        sfc_layer_t l;
        ~LayerGuard() { sfc_layer_destroy(l); }
    } lg{layer};
    std::size_t ws_bytes = 0;
    check(sfc_conv_workspace_size(layer, B, H, W, padding, &ws_bytes));
    DevBuf<uint8_t> ws(ws_bytes);
    QuantReport rep;
    rep.output = DenseTensor({B, OC, HO, WO});
    const std::size_t n = rep.output.data.size();
    DevBuf<double> out(n);
    DevBuf<int32_t> ref(n);
    sfc_outputs o{};
    o.out_f64 = out.p;
    check(sfc_conv_forward(layer, x.p, B, H, W, padding, ws.p, ws_bytes, &o, stream()));
    // report: exact int8 direct conv and the squared-error sums on the device (quant.cpp:282-291)
    check(sfc_direct_conv_int8(x.p, B, C, H, W, w.p, OC, spec.R, 1, padding, ref.p, stream()));
    double sums[2] = {0.0, 0.0};
    check(sfc_report_sq_err(out.p, ref.p, int64_t(n), sums, stream()));
    std::int64_t stats[6] = {};
    check(sfc_conv_stats(layer, B, H, W, padding, ws.p, ws_bytes, stats, stream()));
    std::int64_t fsat = 0;
    check(sfc_layer_saturations(layer, &fsat));
    ck(cudaMemcpyAsync(rep.output.data.data(), out.p, n * sizeof(double), cudaMemcpyDeviceToHost, stream()),
       "copy output");
    ck(cudaStreamSynchronize(stream()), "sync");
    rep.mse = sums[0] / double(n);
    rep.signal_energy = sums[1] / double(n);
    rep.snr_db = 10.0 * std::log10(sums[1] / std::max(sums[0], 1e-300));
    rep.saturations = stats[2] + fsat;
    rep.values_quantized = stats[4];
    return rep;
}

}  // namespace sfconv
