// Plan layer: derive the SFC-N(M, 3) bilinear algorithms from the symbolic DFT.
// See plan.hpp for what is derived and how it relates to the reference.
#include "plan.hpp"

#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>
#include <numeric>
#include <sstream>
#include <stdexcept>

#include "sfc_tables.cuh"

namespace sfcb200 {
namespace {

// ---------------------------------------------------------------- Z[s] helpers
// An element c0 + c1*s of Z[s]/(min poly of the primitive N-th root s):
//   N = 6: s^2 = s - 1,   N = 4: s^2 = -1     (§3, proj/include/sfconv/poly.hpp:24-37)
struct Zs {
    int64_t c0, c1;
};

Zs zs_mul(Zs a, Zs b, int N) {
    const int64_t q0 = a.c0 * b.c0, q1 = a.c0 * b.c1 + a.c1 * b.c0, q2 = a.c1 * b.c1;
    if (N == 6) return {q0 - q2, q1 + q2};
    return {q0 - q2, q1};  // N == 4
}

Zs zs_pow(int e, int N) {
    e = ((e % N) + N) % N;
    Zs r{1, 0};
    for (int i = 0; i < e; ++i) r = zs_mul(r, Zs{0, 1}, N);
    return r;
}

// Component rows of the forward symbolic DFT X_m = sum_t x_t s^{-m t}:
// one row per real frequency (m = 0, N/2), two rows (c0, c1) per complex one.
// Order: [X0, a1, b1, (a2, b2,) X_{N/2}].
std::vector<std::vector<int64_t>> sft_rows(int N) {
    std::vector<std::vector<int64_t>> rows;
    for (int m = 0; m <= N / 2; ++m) {
        std::vector<int64_t> r0(N), r1(N);
        for (int t = 0; t < N; ++t) {
            Zs w = zs_pow(-m * t, N);
            r0[t] = w.c0;
            r1[t] = w.c1;
        }
        rows.push_back(r0);
        if (m != 0 && 2 * m != N) rows.push_back(r1);
    }
    return rows;
}

// Transform channels per axis as signed sums of SFT component rows.  The input
// side carries (Re-part, s-part, their sum) per complex frequency -- the
// Karatsuba evaluation triple -- and the filter side carries the matching
// conjugate combination, so that each channel is one scalar product
// (SFC paper §3.2, Table 2 layout; proj/src/catalog.cpp:94-110 uses the same
// channel order, which fixes the frequency numbering of the pacc outputs).
struct Term {
    int row, sign;
};
using Chan = std::vector<Term>;

void channel_layout(int N, std::vector<Chan>& in, std::vector<Chan>& fil, std::vector<int>& triples) {
    if (N == 6) {  // rows: 0 X0, 1 a1, 2 b1, 3 a2, 4 b2, 5 X3
        in = {{{0, 1}}, {{1, 1}}, {{2, 1}}, {{1, 1}, {2, 1}}, {{3, 1}}, {{4, 1}}, {{3, 1}, {4, 1}}, {{5, 1}}};
        fil = {{{0, 1}}, {{2, -1}}, {{1, -1}}, {{1, -1}, {2, -1}}, {{3, -1}}, {{3, 1}, {4, 1}}, {{4, 1}}, {{5, 1}}};
        triples = {1, 2, 3, 4, 5, 6};
    } else if (N == 4) {  // rows: 0 X0, 1 a1, 2 b1, 3 X2
        in = {{{0, 1}}, {{3, -1}}, {{1, 1}, {2, 1}}, {{2, 1}}, {{1, 1}}};
        fil = {{{0, 1}}, {{3, 1}}, {{1, 1}, {2, 1}}, {{1, 1}}, {{2, 1}}};
        triples = {4, 3, 2};
    } else {
        throw std::invalid_argument("SFC plans exist for N in {4, 6}");
    }
}

// ---------------------------------------------------------------- exact solve
struct Frac {
    int64_t n = 0, d = 1;
    Frac() = default;
    Frac(int64_t v) : n(v), d(1) {}
    Frac(__int128 a, __int128 b) {  // normalised; throws if the reduced value leaves int64
        if (b == 0) throw std::domain_error("exact solve: division by zero");
        if (b < 0) a = -a, b = -b;
        __int128 x = a < 0 ? -a : a, y = b;
        while (y) { const __int128 t = x % y; x = y; y = t; }
        if (x > 1) a /= x, b /= x;
        const __int128 lim = __int128(INT64_MAX);
        if (a > lim || a < -lim || b > lim) throw std::overflow_error("exact solve: rational overflow");
        n = int64_t(a), d = int64_t(b);
    }
    Frac operator-(const Frac& o) const { return Frac(__int128(n) * o.d - __int128(o.n) * d, __int128(d) * o.d); }
    Frac operator*(const Frac& o) const { return Frac(__int128(n) * o.n, __int128(d) * o.d); }
    Frac operator/(const Frac& o) const { return Frac(__int128(n) * o.d, __int128(d) * o.n); }
    bool zero() const { return n == 0; }
    double to_double() const { return double(n) / double(d); }
};

// Solve S x = b exactly (S: rows x cols).  Returns false if inconsistent or
// if the solution is not unique (rank < cols).
bool solve_unique(std::vector<std::vector<Frac>> S, std::vector<Frac> b, std::vector<Frac>& x) {
    const int rows = int(S.size()), cols = int(S[0].size());
    int r = 0;
    std::vector<int> piv;
    for (int c = 0; c < cols && r < rows; ++c) {
        int p = -1;
        for (int i = r; i < rows; ++i)
            if (!S[i][c].zero()) { p = i; break; }
        if (p < 0) continue;
        std::swap(S[p], S[r]);
        std::swap(b[p], b[r]);
        Frac inv = Frac(1) / S[r][c];
        for (int j = c; j < cols; ++j) S[r][j] = S[r][j] * inv;
        b[r] = b[r] * inv;
        for (int i = 0; i < rows; ++i) {
            if (i == r || S[i][c].zero()) continue;
            Frac f = S[i][c];
            for (int j = c; j < cols; ++j) S[i][j] = S[i][j] - f * S[r][j];
            b[i] = b[i] - f * b[r];
        }
        piv.push_back(c);
        ++r;
    }
    for (int i = r; i < rows; ++i)
        if (!b[i].zero()) return false;
    if (r != cols) return false;
    x.assign(cols, Frac(0));
    for (int i = 0; i < r; ++i) x[piv[i]] = b[i];
    return true;
}

// ---------------------------------------------------------------- derivation
SfcPlan derive(int N, int M, int R) {
    SfcPlan p;
    p.N = N;
    p.M = M;
    p.R = R;
    p.n_in = M + R - 1;
    if (p.n_in < N) throw std::invalid_argument("tile smaller than transform");
    p.offset = (p.n_in - N) / 2;
    p.a_denom = N;

    // Window samples the length-N transform cannot see (below offset, or at or
    // beyond offset + N) alias onto a sample N away; each affected
    // (sample, tap) pair whose output lands inside the tile gets one
    // difference product x[desired] - x[wrapped] with that tap.
    const int o = p.offset;
    for (int d = 0; d < o; ++d)
        for (int tap = 0; tap <= std::min(d, R - 1); ++tap) p.corrections.push_back({d - tap, d, d + N, tap});
    for (int d = N + o; d < p.n_in; ++d)
        for (int tap = 0; tap < R; ++tap)
            if (d - tap >= 0 && d - tap < M) p.corrections.push_back({d - tap, d, d - N, tap});

    std::vector<Chan> in, fil;
    channel_layout(N, in, fil, p.triples);
    const auto F = sft_rows(N);
    const int core = int(in.size());
    p.K = core + int(p.corrections.size());
    p.BT.assign(size_t(p.K) * p.n_in, 0);
    p.G.assign(size_t(p.K) * R, 0);
    for (int k = 0; k < core; ++k) {
        for (const Term& t : in[k])
            for (int i = 0; i < N; ++i) p.BT[size_t(k) * p.n_in + o + i] += t.sign * F[t.row][i];
        for (const Term& t : fil[k])
            for (int j = 0; j < R; ++j) p.G[size_t(k) * R + j] += t.sign * F[t.row][j % N];
    }
    for (size_t c = 0; c < p.corrections.size(); ++c) {
        const int k = core + int(c);
        p.BT[size_t(k) * p.n_in + p.corrections[c].desired] = 1;
        p.BT[size_t(k) * p.n_in + p.corrections[c].wrapped] = -1;
        p.G[size_t(k) * R + p.corrections[c].tap] = 1;
    }

    // A: for each output position t, the unique solution of
    //   sum_k A[k,t] BT[k,i] G[k,j] = N [i == t + j]   for all (i, j).
    p.A.assign(size_t(p.K) * M, 0);
    std::vector<std::vector<Frac>> S(size_t(p.n_in) * R, std::vector<Frac>(p.K));
    for (int i = 0; i < p.n_in; ++i)
        for (int j = 0; j < R; ++j)
            for (int k = 0; k < p.K; ++k) S[size_t(i) * R + j][k] = Frac(p.bt(k, i) * p.g(k, j));
    for (int t = 0; t < M; ++t) {
        std::vector<Frac> rhs(size_t(p.n_in) * R);
        for (int i = 0; i < p.n_in; ++i)
            for (int j = 0; j < R; ++j) rhs[size_t(i) * R + j] = Frac(i == t + j ? N : 0);
        std::vector<Frac> col;
        if (!solve_unique(S, rhs, col))
            throw std::domain_error("output transform is not uniquely determined");
        for (int k = 0; k < p.K; ++k) {
            if (col[k].d != 1) throw std::domain_error("non-integral output transform entry");
            p.A[size_t(k) * M + t] = col[k].n;
        }
    }
    // Square overlapped form (used only for conditioning analysis by the reference,
    // catalog.cpp:197-209): the SFT at the window offset plus one difference row per
    // distinct out-of-window alias.
    std::vector<std::pair<int, int>> diffs;
    for (const Correction& ct : p.corrections) {
        const std::pair<int, int> d{ct.desired, ct.wrapped};
        if (std::find(diffs.begin(), diffs.end(), d) == diffs.end()) diffs.push_back(d);
    }
    p.n_overlap = N + int(diffs.size());
    p.overlap.assign(size_t(p.n_overlap) * p.n_overlap, 0);
    for (int r = 0; r < N; ++r)
        for (int t = 0; t < N; ++t) p.overlap[size_t(r) * p.n_overlap + o + t] = F[r][t];
    for (size_t d = 0; d < diffs.size(); ++d) {
        p.overlap[(N + d) * p.n_overlap + diffs[d].first] = 1;
        p.overlap[(N + d) * p.n_overlap + diffs[d].second] = -1;
    }
    std::ostringstream nm;
    nm << "sfc" << N << "-" << M << "x" << M << "-" << R << "x" << R;
    p.name = nm.str();
    return p;
}

template <int V>
bool matches_device_tables(const SfcPlan& p) {
    using T = Tab<V>;
    if (p.K != T::K || p.n_in != T::n || p.M != T::M || p.R != T::R || p.a_denom != T::DEN) return false;
    for (int k = 0; k < p.K; ++k) {
        for (int i = 0; i < p.n_in; ++i)
            if (p.bt(k, i) != T::bt(k, i)) return false;
        for (int j = 0; j < p.R; ++j)
            if (p.g(k, j) != T::g(k, j)) return false;
        for (int t = 0; t < p.M; ++t)
            if (p.a(k, t) != T::a(k, t)) return false;
    }
    return true;
}

std::mutex g_mu;
std::map<std::string, SfcPlan>& cache() {
    static std::map<std::string, SfcPlan> c;
    return c;
}

}  // namespace

SfcPlan derive_sfc_plan(int N, int M, int R) {
    SfcPlan p = derive(N, M, R);
    if (long bad = plan_identity_violations(p))
        throw std::domain_error(p.name + ": " + std::to_string(bad) + " identity violations");
    return p;
}

long plan_identity_violations(const SfcPlan& p) {
    long bad = 0;
    for (int t = 0; t < p.M; ++t)
        for (int i = 0; i < p.n_in; ++i)
            for (int j = 0; j < p.R; ++j) {
                int64_t acc = 0;
                for (int k = 0; k < p.K; ++k) acc += p.a(k, t) * p.bt(k, i) * p.g(k, j);
                if (acc != (i == t + j ? p.a_denom : 0)) ++bad;
            }
    return bad;
}

const std::vector<std::string>& plan_names() {
    // the SFC entries of the reference catalog, in its order (catalog.cpp:246-250)
    static const std::vector<std::string> names = {"sfc4-4x4-3x3", "sfc6-6x6-3x3", "sfc6-7x7-3x3", "sfc6-6x6-5x5",
                                                   "sfc6-4x4-7x7"};
    return names;
}

const SfcPlan& plan_for(const std::string& name) {
    std::lock_guard<std::mutex> lock(g_mu);
    auto it = cache().find(name);
    if (it != cache().end()) return it->second;
    SfcPlan p;
    if (name == "sfc4-4x4-3x3") p = derive(4, 4, 3), p.variant = 0;
    else if (name == "sfc6-6x6-3x3") p = derive(6, 6, 3), p.variant = 1;
    else if (name == "sfc6-7x7-3x3") p = derive(6, 7, 3), p.variant = 2;
    else if (name == "sfc6-6x6-5x5") p = derive(6, 6, 5), p.variant = 3;
    else if (name == "sfc6-4x4-7x7") p = derive(6, 4, 7), p.variant = 4;
    else throw std::invalid_argument("unknown algorithm: " + name);
    // Exhaustive exactness gate: the per-axis identity makes every integer
    // tile exact (stronger than the reference's 3 random trials, catalog.cpp:283).
    if (long bad = plan_identity_violations(p))
        throw std::domain_error("catalog integrity failure for " + name + ": " + std::to_string(bad) +
                                " identity violations");
    const bool same = p.variant == 0 ? matches_device_tables<0>(p)
                    : p.variant == 1 ? matches_device_tables<1>(p)
                    : p.variant == 2 ? matches_device_tables<2>(p)
                    : p.variant == 3 ? matches_device_tables<3>(p)
                                     : matches_device_tables<4>(p);
    if (!same) throw std::domain_error("derived plan differs from the compiled device tables for " + name);
    return cache().emplace(name, std::move(p)).first->second;
}

namespace {
// Karatsuba components (c0, c1, c0 + c1) of the block value sum_q V_q z_q for the
// corner weights z_q = s^r * e^c (q = 2 r + c), e = s or conj(s) = s^(N-1).
void eval_forms(int N, bool conj2, double out[3][4], Frac outf[3][4]) {
    for (int q = 0; q < 4; ++q) {
        const int r = q >> 1, c = q & 1;
        const Zs z = zs_mul(zs_pow(r, N), zs_pow(conj2 ? c * (N - 1) : c, N), N);
        const int64_t comp[3] = {z.c0, z.c1, z.c0 + z.c1};
        for (int l = 0; l < 3; ++l) out[l][q] = double(comp[l]), outf[l][q] = Frac(comp[l]);
    }
}

PairBlock derive_block(const SfcPlan& p, const int* t1, const int* t2) {
    PairBlock b{};
    for (int i = 0; i < 3; ++i) b.r1[i] = t1[i], b.r2[i] = t2[i];
    // each block row must be additive (row c = row a + row b) in B^T and G on both axes
    for (const int* t : {t1, t2}) {
        for (int j = 0; j < p.n_in; ++j)
            if (p.bt(t[0], j) + p.bt(t[1], j) != p.bt(t[2], j)) throw std::domain_error("block rows not additive");
        for (int j = 0; j < p.R; ++j)
            if (p.g(t[0], j) + p.g(t[1], j) != p.g(t[2], j)) throw std::domain_error("block rows not additive");
    }
    Frac af[6][4];
    {
        double d[3][4];
        Frac f[3][4];
        eval_forms(p.N, false, d, f);
        for (int l = 0; l < 3; ++l)
            for (int q = 0; q < 4; ++q) b.alpha[l][q] = d[l][q], af[l][q] = f[l][q];
        eval_forms(p.N, true, d, f);
        for (int l = 0; l < 3; ++l)
            for (int q = 0; q < 4; ++q) b.alpha[3 + l][q] = d[l][q], af[3 + l][q] = f[l][q];
    }
    for (int l = 0; l < 6; ++l)
        for (int q = 0; q < 4; ++q) b.beta[l][q] = b.alpha[l][q];
    // position (i, j) in corner coordinates: row i of {a, b, c} = (1,0), (0,1), (1,1)
    const int ex[3][2] = {{1, 0}, {0, 1}, {1, 1}};
    const int M = p.M;
    std::vector<std::vector<Frac>> S;
    std::vector<Frac> rhs;
    for (int o1 = 0; o1 < M; ++o1)
        for (int o2 = 0; o2 < M; ++o2)
            for (int qv = 0; qv < 4; ++qv)
                for (int qu = 0; qu < 4; ++qu) {
                    int64_t target = 0;
                    for (int i = 0; i < 3; ++i)
                        for (int j = 0; j < 3; ++j) {
                            const int64_t ev = ex[i][qv >> 1] * ex[j][qv & 1], eu = ex[i][qu >> 1] * ex[j][qu & 1];
                            target += p.a(t1[i], o1) * p.a(t2[j], o2) * ev * eu;
                        }
                    std::vector<Frac> row(24);
                    for (int q = 0; q < 4; ++q) {
                        const Frac w(p.a(t1[q >> 1], o1) * p.a(t2[q & 1], o2));
                        for (int l = 0; l < 6; ++l) row[size_t(q) * 6 + l] = w * af[l][qv] * af[l][qu];
                    }
                    S.push_back(std::move(row));
                    rhs.push_back(Frac(target));
                }
    std::vector<Frac> sol;
    if (!solve_unique(S, rhs, sol)) throw std::domain_error("paired block: fold not uniquely determined");
    for (int q = 0; q < 4; ++q)
        for (int l = 0; l < 6; ++l) b.fold[q][l] = sol[size_t(q) * 6 + l].to_double();
    return b;
}

std::mutex g_pair_mu;
std::map<std::string, PairedSchedule>& pair_cache() {
    static std::map<std::string, PairedSchedule> c;
    return c;
}

void matrix_json(std::ostringstream& os, const char* key, const std::vector<int64_t>& m, int rows, int cols) {
    os << '"' << key << "\":[";
    for (int i = 0; i < rows; ++i) {
        os << (i ? ",[" : "[");
        for (int j = 0; j < cols; ++j) os << (j ? "," : "") << '"' << m[size_t(i) * cols + j] << '"';
        os << ']';
    }
    os << ']';
}
}  // namespace

const PairedSchedule& paired_schedule(const SfcPlan& p) {
    std::lock_guard<std::mutex> lock(g_pair_mu);
    auto it = pair_cache().find(p.name);
    if (it != pair_cache().end()) return it->second;
    PairedSchedule ps;
    const int nt = int(p.triples.size() / 3);
    if (nt > 0) {
        ps.masked.assign(size_t(p.K) * p.K, 0);
        for (int u = 0; u < nt; ++u)
            for (int v = 0; v < nt; ++v) {
                const int* t1 = &p.triples[size_t(u) * 3];
                const int* t2 = &p.triples[size_t(v) * 3];
                ps.blocks.push_back(derive_block(p, t1, t2));
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) ps.masked[size_t(t1[i]) * p.K + t2[j]] = 1;
            }
        ps.available = true;
    }
    return pair_cache().emplace(p.name, std::move(ps)).first->second;
}

std::string plan_export_json(const std::vector<std::string>& names) {
    std::ostringstream os;
    os << "{\"algorithms\":[";
    for (size_t a = 0; a < names.size(); ++a) {
        const SfcPlan& s = plan_for(names[a]);
        os << (a ? "," : "") << "{\"name\":\"" << s.name << "\",\"family\":\"sfc\",\"N\":" << s.N
           << ",\"tile\":" << s.M << ",\"kernel\":" << s.R << ",\"offset\":" << s.offset
           << ",\"denominator\":" << s.a_denom << ",\"mults_full\":" << s.mults_full()
           << ",\"mults_reduced\":" << s.mults_reduced() << ',';
        matrix_json(os, "BT", s.BT, s.K, s.n_in);
        os << ',';
        matrix_json(os, "G", s.G, s.K, s.R);
        os << ',';
        matrix_json(os, "A", s.A, s.K, s.M);
        os << ",\"corrections\":[";
        for (size_t c = 0; c < s.corrections.size(); ++c) {
            const Correction& ct = s.corrections[c];
            os << (c ? "," : "") << '[' << ct.out << ',' << ct.desired << ',' << ct.wrapped << ',' << ct.tap << ']';
        }
        os << "]}";
    }
    os << "]}";
    return os.str();
}

uint64_t fnv1a64(const std::string& s) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (unsigned char c : s) {
        h ^= c;
        h *= 0x100000001b3ULL;
    }
    return h;
}

}  // namespace sfcb200
