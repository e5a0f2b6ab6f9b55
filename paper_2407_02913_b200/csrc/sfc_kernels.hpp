// Internal launch API for the SFC CUDA kernels (not part of the C-ABI).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace sfcb200 {

// Geometry of one quantized SFC convolution call (stride 1, symmetric pad).
struct ConvGeom {
    int B, C, H, W, pad;
    int HO, WO, th, tw;
    int T;      // tiles = B * th * tw
    int Tpad;   // T rounded up to the GEMM row block (128)
    int Cpad;   // input channels rounded up to the GEMM K chunk (BK)
    int BK;     // 64 or 128 bytes of K per pipeline stage
    int OC, OCpad, BN;
    // output-transform launches over a chunk of image tile rows (P chunked, see PChunk):
    // rows [row0, row0 + nrows) of the B * th rows; geom_init sets the whole range
    int row0, nrows;
    // P storage: 0 = int32 [F][Tpad][OCpad]; 1 = 24-bit [F][Tpad] rows of 3*OCpad bytes: byte
    // planes b0 | b1 | b2 of OCpad bytes, P = b0 + 2^8 b1 + 2^16 b2 (exact when |P| < 2^23, i.e.
    // qmax^2 * Cin < 2^23).  2 = the same 24-bit values unit-major for the tensor-core output
    // transform (pu_offset below).  geom_init sets 0; run_conv decides (p24_wanted).
    int p24;
    // unit-major P with a sparse plane 2 (p2_flags_offset below); run_conv decides (p2_sparse_wanted)
    int p2s;
};

// 24-bit P, unit-major (ConvGeom::p24 == 2): the A operands of the tensor-core output
// transform (out_mma.cu), written pre-swizzled by the GEMM epilogue.  A unit is kUnitOc output
// channels x kUnitTiles consecutive tiles = 128 MMA rows (row = tt * 32 + oc).  Storage
// [OCpad / 32][3 byte planes][F][Tpad / 4][128 B]: byte plane b0, b1 (unsigned), b2 (signed)
// (P = b0 + 2^8 b1 + 2^16 b2); the 128-byte row (f, unit) holds [tt][32 oc] with 16-byte chunk
// c at c ^ (f & 7), the 128B-swizzle pattern of an MN-major tcgen05 operand.  The F rows of a
// unit land in shared memory as that operand with one TMA box; the GEMM writes the rows of 8
// consecutive units (1 KB contiguous) per box.  (Measured: with each unit's rows contiguous
// instead -- [oc block][tile group][plane][F] -- the output transform is no faster and the
// GEMM's 128-byte writes 38 KB apart cost 0.1-0.7 ms per VGG-16 step.)
//
// Sparse plane 2 (ConvGeom::p2s): the GEMM stores P' = P + 2^15, so every value within 16 bits
// has a zero third byte; row (f, unit) of plane 2 is written only when one of its 128 values
// leaves that range, and a flag byte per (unit, f) says so: flags [OCpad / 32][Tpad / 32][F][8]
// (8 consecutive tile groups per entry) after the three planes.  The output transform loads
// the flagged rows, zero-fills the others, skips the all-zero K steps and subtracts the bias
// 2^15 * sum_f W[o][f] per output.  Post-ReLU activations leave only the DC frequency outside
// 16 bits, so about a third of the P traffic disappears; with every row flagged the layout
// degenerates to the dense one plus the flags.
constexpr int kUnitTiles = 4, kUnitOc = 32;
__host__ __device__ inline size_t p2_flags_offset(int F, int Tpad, int OCpad) { return size_t(3) * F * Tpad * OCpad; }
__host__ __device__ inline size_t p2_flag_index(int ob, int tg, int f, int Tpad, int F) {
    return ((size_t(ob) * (Tpad / (8 * kUnitTiles)) + tg / 8) * F + f) * 8 + (tg & 7);
}
__host__ __device__ inline size_t pu_offset(int ob, int tg, int plane, int f, int n_tg, int F) {
    return (((size_t(ob) * 3 + plane) * F + f) * n_tg + tg) * 128;
}

// P chunking (opt-in: SFC_PCHUNK_MB = budget in MB; unset or 0 = never chunk).  P (4 B per
// (frequency, tile, oc)) is the largest intermediate; when the whole of it exceeds the
// budget, GEMM and output transform alternate over chunks of `rows` image tile rows so
// each chunk's P is consumed from L2 and discarded there (never written back to HBM), and
// the workspace holds one chunk (config 5: 52 MB instead of 472 MB).  Measured on config
// 5 it is slower (0.49 ms at 64 MB vs 0.41 ms whole): the serialised per-chunk ramp-up /
// drain of two bandwidth kernels costs more than the HBM traffic it saves, so it is a
// workspace-memory cap, not the default; overlapping chunk i's output transform with
// chunk i+1's GEMM is the open follow-up.
struct PChunk {
    int rows;   // image tile rows per chunk (last chunk may be shorter)
    int tcpad;  // P rows per chunk buffer: rows * tw rounded up to the GEMM row block
    int n;      // chunks
};
PChunk p_chunk(const ConvGeom& g, int F);

// Activation quantizer derived on device from the global absmax (so multi-GPU
// callers can all-reduce the absmax first).
struct QuantParams {
    double sa;        // activation scale  max(vmax / qmax, 1e-8)     (quant.cpp:117-120)
    long long mul;    // exact fast path: q = (v * mul + 2^(shift-1)) >> shift
    int shift;
    int exact;        // 1 when the fast path was proven equal to rint(v / sa) on [-vmax, vmax]
    int vmax;
    int qmax;
};

void geom_init(ConvGeom& g, int variant, int B, int C, int H, int W, int pad, int OC);
// Workspace header: vmax @0, saturations @8, QuantParams @64; general QuantConfig:
// maxima @512 (fp64 bit patterns x F), activation scales @2304 (fp64 x F); F <= 196.
constexpr size_t kWsHeader = 4096, kWsMaxima = 512, kWsActScales = 2304;
size_t workspace_bytes(const ConvGeom& g, int F);

// `pdl`: launch with programmatic stream serialization (overlap the predecessor's tail).
cudaError_t launch_filter_prepare(int variant, const int8_t* w, int OC, int IC, int Cpad, int OCpad, int bits,
                                  double* sf, int* umax, int8_t* uqB, unsigned long long* sat, cudaStream_t st);
// pdl: launched under programmatic stream serialization; the CTAs stage and transform
// their tiles before waiting on the predecessor (which zeroes *vmax).
// vkeep != nullptr: also keep V as int16 [F][Tpad][Cpad] for launch_quant_kept.
// Whether the 3x3 activation kernels take the two-channel SWAR form for this layer (large
// layers; SFC_ACT_PAIR=0/1 forces either).
bool act_pair_wanted(const ConvGeom& g);
// Register-resident SWAR transform (3x3 variants, act_reg.cu): mode 1 quantizes into vqA,
// otherwise max|V| (+ the kept V when vkeep).  act_reg_wanted: variant supported and not
// disabled (SFC_ACT_REG=0).
bool act_reg_wanted(int variant, const ConvGeom& g);
cudaError_t launch_act_reg(int variant, int mode, const int8_t* x, const ConvGeom& g, int* vmax, int16_t* vkeep,
                           const int* vmax_in, int bits, QuantParams* qp, int8_t* vqA, unsigned long long* sat,
                           cudaStream_t st, bool pdl);
cudaError_t launch_act_absmax(int variant, const int8_t* x, const ConvGeom& g, int* vmax, int16_t* vkeep,
                              cudaStream_t st, bool pdl = false);
// vq = q(kept V) for t < T, channels >= C zeroed (streaming; replaces launch_act_quant's
// recomputation of the transform).
cudaError_t launch_quant_kept(const int16_t* vkeep, const ConvGeom& g, int F, const int* vmax, int bits,
                              QuantParams* qp, int8_t* vqA, unsigned long long* sat, cudaStream_t st, bool pdl);
// Zero `words` 32-bit words (<= 32) at p once the predecessor kernel has finished --
// a PDL kernel instead of a memset node, which costs ~3 us in a graph / stream chain.
cudaError_t launch_zero_words(uint32_t* p, int words, cudaStream_t st);
enum TlKernel { kTlZero = 0, kTlAbsmax = 1, kTlQuant = 2, kTlGemm = 3, kTlOutput = 4, kTlCount = 8 };
// Activation quantization fused into the GEMM (k_gemm<..., QF = true>): converter warps
// read the int16 V kept by the absmax pass and write the quantized A tiles in shared
// memory; the vq round trip through HBM and the quantize launch disappear.
struct QFuse {
    const int16_t* v;           // kept V [F][Tpad][Cpad]
    const int* vmax;            // global max|V| (after any multi-GPU all-reduce)
    const QuantParams* qtab;    // qparams_table(false) or nullptr
    QuantParams* qp_out;        // written by CTA 0 for the output transform / stats
    unsigned long long* sat;    // saturation counter of the non-verified quantizer path
    int bits;
};
cudaError_t launch_gemm_qfused(const QFuse& q, const int8_t* uqB, int32_t* P, const ConvGeom& g, int F, cudaStream_t st,
                               bool pdl);
// The same with the V tiles TMA-staged in shared memory (SFC_QFUSE=2).
cudaError_t launch_gemm_qtma(const QFuse& q, const int8_t* uqB, int32_t* P, const ConvGeom& g, int F, cudaStream_t st,
                             bool pdl);

// Timeline stamps of the debug build ([8][3] per unit; cudaErrorNotSupported otherwise).
cudaError_t tl_read_act(unsigned long long* out, bool reset);
cudaError_t tl_read_reg(unsigned long long* out, bool reset);
cudaError_t tl_read_gemm(unsigned long long* out, bool reset);
cudaError_t tl_read_out(unsigned long long* out, bool reset);
cudaError_t tl_read_aux(unsigned long long* out, bool reset);
cudaError_t launch_act_quant(int variant, const int8_t* x, const ConvGeom& g, const int* vmax, int bits,
                             QuantParams* qp, int8_t* vqA, unsigned long long* sat, cudaStream_t st, bool pdl);
// P rows [t0, t0 + tcpad) of the full problem into a P buffer of tcpad rows (a P chunk).
cudaError_t launch_gemm_rows(const int8_t* vqA, const int8_t* uqB, int32_t* P, const ConvGeom& g, int F, int t0,
                             int tcpad, cudaStream_t st, bool pdl);
cudaError_t launch_gemm(const int8_t* vqA, const int8_t* uqB, int32_t* P, const ConvGeom& g, int F, cudaStream_t st,
                        bool pdl);
// Output pointers of the output-transform kernel (any may be null).
struct OutPtrs {
    int32_t* y32;
    int64_t* y64;
    float* f32;
    double* f64;
    int8_t* i8;
    double requant;
    // general QuantConfig (mode 2): per-frequency activation scales and the (oc, f) filter
    // scale table; the epilogue dequantises P before the inverse transform in fp64
    const double* gen_act = nullptr;
    int gen_per_freq = 0;
    const double* gen_fil = nullptr;  // [OC][F]
    int pairs = 1;  // the persistent output kernel may store column pairs (8-byte stores)
    // when set (the P chunk buffer): every block discards the P lines it consumed from L2
    // (discard.global.L2), so chunked P is never written back to HBM
    const void* p_discard = nullptr;
};
// mode 0: exact int32 y, 1: exact int64 y, 2: general QuantConfig (fp64, no y_int),
// 3: fp64 P [F][Tpad][OCpad] of the float path (no dequantisation)
// Cin <= 4, exact int32 y: dp4a contraction fused with the output transform (no P);
// vq4 = compact [F][T][4] int8 from the quantizing transform.
cudaError_t launch_output_smallc(int variant, const int8_t* vq4, const int8_t* uq, const ConvGeom& g,
                                 const QuantParams* qp, const double* sf, const OutPtrs& o, cudaStream_t st, bool pdl);
// Tensor-core output transform over unit-major 24-bit P (g.p24 == 2; 3x3 variants, int32-exact
// y, every output kind): cudaErrorNotSupported when not applicable.
cudaError_t launch_output_mma(int variant, const void* P, const ConvGeom& g, const QuantParams* qp, const double* sf,
                              const OutPtrs& o, cudaStream_t st, bool pdl);
// The 5-D map over unit-major P: (128-byte row, tile group, f, plane, oc block), box rows x
// tile groups x frequencies as given; swizzle as given (the data itself is pre-swizzled).
bool make_pu_map(CUtensorMap* m, void* P, const ConvGeom& g, int F, int box_tg, int box_f, bool swizzle128,
                 int box_planes = 1);
bool output_mma_supported(int variant, const ConvGeom& g, const OutPtrs& o);
// Batched fp64 NT contraction P_f = V_f U_f^T (f64_gemm.cu): the 9-16 bit exact-integer path
// and the float fast_conv2d path.
cudaError_t launch_dgemm_freq(const double* U, const double* V, double* P, int Tpad, int OCpad, int Cpad, int batch,
                              cudaStream_t st);
cudaError_t launch_output(int variant, int mode, const void* P, const ConvGeom& g, const QuantParams* qp,
                          const double* sf, const OutPtrs& o, cudaStream_t st, bool pdl);
// report sums: `sums` holds 2 + 2 * kSqErrBlocks doubles (result in [0..1], block partials after)
constexpr int kSqErrBlocks = 148 * 8;
cudaError_t launch_sq_err(const double* out, const int32_t* ref, long long n, double* sums, cudaStream_t st);
cudaError_t launch_sq_err_f64(const double* out, const double* ref, long long n, double* sums, cudaStream_t st);
// Device table of verified quantizer parameters (common.cuh, kQpTableMax).  build=true
// derives it synchronously on a private stream the first time (layer creation -- never
// inside a graph capture); build=false returns it or nullptr (kernels then derive per CTA).
const QuantParams* qparams_table(bool build);
cudaError_t launch_quant_params(const int* vmax, int bits, QuantParams* qp, unsigned long long* sat,
                                cudaStream_t st);
cudaError_t launch_debug_quant(const QuantParams* qp, int vmax, int32_t* q, unsigned long long* sat, cudaStream_t st);
cudaError_t launch_direct_conv(const int8_t* x, int B, int C, int H, int W, const int8_t* w, int OC, int R,
                               int stride, int pad, int32_t* out, cudaStream_t st);
cudaError_t launch_freq_energy(int variant, const int8_t* x, const ConvGeom& g, unsigned long long* sum,
                               cudaStream_t st);
cudaError_t launch_transform_filters(int variant, const int8_t* w, int OC, int IC, int32_t* u, cudaStream_t st);

// General QuantConfig (general_kernels.cu).  Filters: per-group scales of U [OC][IC][F]
// (scope 0 PerChannel, 1 PerFrequency, 2 PerChannelFrequency; MinMax or MseGrid), uq and the
// expanded [OC][F] scale table.  err_tmp: groups * 101 doubles.
// bits > 8: uqB / vqA hold integer-valued doubles (the exact fp64 GEMM of the wide path),
// else int8 tensor-core operands.
cudaError_t launch_fil_general(const int32_t* U, int OC, int IC, int F, int scope, int mse, int bits, int Cpad,
                               int OCpad, double* scale_native, double* err_tmp, void* uqB, double* fil_full,
                               unsigned long long* sat, cudaStream_t st);
// Activations from the kept V: maxima (1 or F slots, zeroed on entry; fp64 bit patterns),
// MinMax / MseGrid scales act_scale[1 or F] and vq (exact fp64 quantizer, saturations counted).
cudaError_t launch_act_general(const int16_t* V, const ConvGeom& g, int F, int per_freq, int mse, int bits,
                               unsigned long long* vmax, double* act_scale, void* vqA, unsigned long long* sat,
                               double* err_tmp, cudaStream_t st);
// The same in steps, for the batch-sharded general path: local maxima (fp64 bit patterns,
// 1 or F slots zeroed beforehand), the MseGrid partial sums continuing from err_in ([groups]
// [101]; nullptr = batch start), the pick (err nullptr = MinMax), the quantize.
cudaError_t launch_act_maxima(const int16_t* V, const ConvGeom& g, int F, int per_freq, unsigned long long* vmax,
                              cudaStream_t st);
cudaError_t launch_act_mse(const int16_t* V, const ConvGeom& g, int F, int per_freq, const unsigned long long* vmax,
                           int bits, const double* err_in, double* err_out, cudaStream_t st);
cudaError_t launch_act_pick(int F, int per_freq, const unsigned long long* vmax, int bits, const double* err,
                            double* act_scale, cudaStream_t st);
cudaError_t launch_act_quantize(const int16_t* V, const ConvGeom& g, int F, int per_freq, const double* act_scale,
                                int bits, void* vqA, unsigned long long* sat, cudaStream_t st);
// Real-valued (fp64) inputs and filters, the reference's own arithmetic order:
// V [F][Tpad][Cpad] (gather_tiles), U [OC][IC][F] (transform_filters), direct conv.
cudaError_t launch_act_general_f64(const double* V, const ConvGeom& g, int F, int per_freq, int mse, int bits,
                                   unsigned long long* vmax, double* act_scale, void* vqA, unsigned long long* sat,
                                   double* err_tmp, cudaStream_t st);
cudaError_t launch_fil_general_f64(const double* U, int OC, int IC, int F, int scope, int mse, int bits, int Cpad,
                                   int OCpad, double* scale_native, double* err_tmp, void* uqB, double* fil_full,
                                   unsigned long long* sat, cudaStream_t st);
cudaError_t launch_act_f64(int variant, const double* x, const ConvGeom& g, double* Vd, cudaStream_t st);
cudaError_t launch_filters_f64(int variant, const double* w, int OC, int IC, double* U, cudaStream_t st);
cudaError_t launch_direct_f64(const double* x, int B, int C, int H, int W, const double* w, int OC, int R, int stride,
                              int pad, double* out, cudaStream_t st);
cudaError_t launch_pack_u_f64(const double* U, int OC, int IC, int F, int Cpad, int OCpad, double* Ub,
                              cudaStream_t st);
// Paired-product schedule of fast_conv2d (plan.hpp PairedSchedule): slice s of the
// reduced batch is sum_k a[k] * src[f[k]] (V side) / sum_k b[k] * src[f[k]] (U side);
// n == 1 is a direct (unpaired) position.
struct PairSlice {
    int n, f[4];
    double a[4], b[4];
};
// Position f of P after the reduced batch: kind 0 zero (inside a block, not a corner),
// 1 copy of slice src, 2 corner: sum_l w[l] * slice (src + l).
struct PairFold {
    int kind, src;
    double w[6];
};
cudaError_t launch_pair_gather(const double* src, long long elems, const PairSlice* tab, int nslices, bool filter_side,
                               double* dst, cudaStream_t st);
cudaError_t launch_pair_fold(const double* Pr, long long elems, const PairFold* tab, int F, double* P,
                             cudaStream_t st);

}  // namespace sfcb200
