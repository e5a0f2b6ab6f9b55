// Host-side plan layer: the SFC bilinear algorithms for 3x3 kernels.
//
// Mirrors the reference's catalog for the three 3x3 SFC variants
// (proj/src/catalog.cpp:246-248, derive_correction_spec at catalog.cpp:132-215)
// but derives them differently: B^T and G are assembled from the symbolic DFT
// component rows, and the output transform A is *solved* exactly from the
// correlation identity  sum_k A[k,t] BT[k,i] G[k,j] = N * [i == t + j]
// (the same constraint the reference's repair tool uses, catalog.cpp:477-542),
// so it is not a transcription of the reference's A tables.  Every plan passes
// an exhaustive exactness gate before use and is checked against the tables
// compiled into the CUDA kernels.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace sfcb200 {

struct Correction {
    int out, desired, wrapped, tap;
};

struct SfcPlan {
    std::string name;
    int N = 0, M = 0, R = 0, offset = 0;
    int K = 0, n_in = 0;
    int64_t a_denom = 1;
    std::vector<int64_t> BT;  // K x n_in
    std::vector<int64_t> G;   // K x R
    std::vector<int64_t> A;   // K x M
    std::vector<Correction> corrections;
    std::vector<int> triples;  // flattened (a, b, c) per axis triple
    int n_overlap = 0;
    std::vector<int64_t> overlap;  // n_overlap x n_overlap: SFT rows + one difference row per alias
    int variant = -1;          // index into the compiled device tables

    long mults_full() const { return long(K) * K; }
    long mults_reduced() const {
        long t = long(triples.size() / 3);
        return mults_full() - 3 * t * t;
    }
    double complexity_pct() const { return 100.0 * double(mults_reduced()) / (double(M) * M * R * R); }
    int64_t bt(int k, int i) const { return BT[size_t(k) * n_in + i]; }
    int64_t g(int k, int j) const { return G[size_t(k) * R + j]; }
    int64_t a(int k, int t) const { return A[size_t(k) * M + t]; }
};

// Paired-product schedule of fast_conv2d's reduced_products option (conv.cpp:39-295,
// 466-509): on each (axis-1 triple) x (axis-2 triple) block the nine positionwise
// products collapse to six -- the block's 2-D value evaluated at (s, s) and (s, conj s),
// each multiplied Karatsuba-style -- folded back onto the four corner positions.
struct PairBlock {
    int r1[3], r2[3];    // (a, b, c) transform rows per axis; corners are a/b x a/b
    double alpha[6][4];  // product l = (alpha[l] . V corners) * (beta[l] . U corners)
    double beta[6][4];
    double fold[4][6];   // corner q = 2 r + c gets sum_l fold[q][l] * product l
};
struct PairedSchedule {
    bool available = false;
    std::vector<uint8_t> masked;  // K*K: position inside some block (no direct product)
    std::vector<PairBlock> blocks;
};
// Derived here (not transcribed): alpha/beta are the Karatsuba components of the two
// evaluations, and fold is the unique exact solution of the block's output identity
//   sum_{ij in block} A_i(o1) A_j(o2) V_ij U_ij = sum_{corners} A_r(o1) A_c(o2) fold . products
// for every output pair (o1, o2) and every V, U.  Throws std::domain_error if the
// identity has no unique solution.
const PairedSchedule& paired_schedule(const SfcPlan& p);

// Throws std::invalid_argument for unknown names and std::domain_error when the
// exactness gate fails.  Returned references live for the process lifetime.
const SfcPlan& plan_for(const std::string& name);

// Host-only derivation of SFC-N(M, R) for N in {4, 6} (any M, R with M + R - 1 >= N);
// not bound to device tables (variant = -1).  derive_correction_spec, catalog.cpp:132-215.
SfcPlan derive_sfc_plan(int N, int M, int R);
const std::vector<std::string>& plan_names();

// Number of (t, i, j) triples violating sum_k A BT G = a_denom [i == t + j].
long plan_identity_violations(const SfcPlan& p);

// JSON in the reference's catalog_export_json layout (catalog.cpp:562-591)
// restricted to `names`; FNV-1a 64 over that text.
std::string plan_export_json(const std::vector<std::string>& names);
uint64_t fnv1a64(const std::string& s);

}  // namespace sfcb200
