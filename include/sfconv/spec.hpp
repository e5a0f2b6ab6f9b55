// sfconv:: drop-in (B200 build) -- algorithm specs and the catalog.
// Declarations match the reference's include/sfconv/spec.hpp (AlgorithmSpec
// spec.hpp:36-62, catalog spec.hpp:76-79, validation spec.hpp:85-99).  The
// catalog of this build serves the device path: the five SFC algorithms
// ("sfc4-4x4-3x3", "sfc6-6x6-3x3", "sfc6-7x7-3x3", "sfc6-6x6-5x5", "sfc6-4x4-7x7"), derived by the plan layer
// (paper_2407_02913_b200/csrc/plan.cpp), exactness-gated, and identical to the
// reference's entries.  Other names throw std::invalid_argument("unknown
// algorithm: ...") exactly like an unknown name in the reference.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "sfconv/rational.hpp"

namespace sfconv {

enum class AlgoFamily { Direct, Winograd, Sfc };

struct CorrectionTerm {
    int out = 0;      // output sample the product patches
    int desired = 0;  // window sample the transform cannot reach
    int wrapped = 0;  // its alias modulo N, double-counted by the transform
    int tap = 0;      // filter tap of the patch product
    friend bool operator==(const CorrectionTerm& x, const CorrectionTerm& y) {
        return x.out == y.out && x.desired == y.desired && x.wrapped == y.wrapped && x.tap == y.tap;
    }
};

struct TripleChannels {
    int a = 0, b = 0, c = 0;  // row c = row a + row b in B^T and G
};

// y = A^T [(G f G^T) .* (B^T x B)] A / a_denom^2 per tile.
struct AlgorithmSpec {
    std::string name;
    AlgoFamily family = AlgoFamily::Direct;
    int N = 0;
    int M = 0;
    int R = 0;
    int offset = 0;
    RatMatrix BT;  // K x n_in
    RatMatrix G;   // K x R
    RatMatrix A;   // K x M
    std::int64_t a_denom = 1;
    RatMatrix overlap_form;
    std::vector<CorrectionTerm> corrections;
    std::vector<TripleChannels> triples;

    int K() const { return BT.rows; }
    int n_in() const { return BT.cols; }
    long mults_full() const { return long(K()) * K(); }
    long mults_reduced() const {
        const long t = long(triples.size());
        return mults_full() - 3 * t * t;
    }
    double complexity_pct() const { return 100.0 * double(mults_reduced()) / (double(M) * M * R * R); }
};

AlgorithmSpec derive_correction_spec(int N, int M, int R);

const AlgorithmSpec& catalog_algorithm(const std::string& name);
const std::vector<std::string>& catalog_names();
std::string catalog_export_json();
std::uint64_t catalog_hash();

struct ValidationReport {
    bool ok = false;
    int trials = 0;
    long mismatches = 0;
    std::string detail;
};

ValidationReport validate_algorithm(const AlgorithmSpec& spec, int trials, std::uint64_t seed);

std::vector<std::int64_t> execute_tile_exact(const AlgorithmSpec& spec, const std::vector<std::int64_t>& x,
                                             const std::vector<std::int64_t>& f);

}  // namespace sfconv
