// C-ABI implementation (include/sfc_b200.h).  Host orchestration only: every
// numerical stage runs in the CUDA kernels of kernels.cu; there is no CPU
// fallback -- a missing / failing device path returns SFC_ERR_CUDA.
#include "../../include/sfc_b200.h"
#include "devcache.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <new>
#include <stdexcept>
#include <string>

#include "plan.hpp"
#include "sfc_kernels.hpp"

using namespace sfcb200;

struct sfc_plan {
    const SfcPlan* p;
};

struct sfc_layer {
    const SfcPlan* plan;
    int variant, OC, IC, bits, BK, Cpad, BN, OCpad, F;
    int8_t* d_uq = nullptr;        // [F][OCpad][Cpad]
    double* d_sf = nullptr;        // [OC]
    int* d_umax = nullptr;         // [OC]
    unsigned long long* d_sat = nullptr;
    int64_t max_a_col_l1 = 0;      // for the int32 output bound
    // QuantConfig beyond PerTensor / PerChannel / MinMax (general_kernels.cu)
    int act_scope = 0, filter_scope = 0, search = 0;
    bool general = false;
    double* d_fil = nullptr;       // [OC][F] filter scale per (oc, f)
    double* d_fil_native = nullptr;  // scales as the scope defines them (OC, F or OC*F)
    int n_fil_native = 0;
    // bits 9-16 (the reference's full width range): uq as integer-valued doubles
    // [F][OCpad][Cpad], contracted by an exact fp64 GEMM (|P| <= IC * 2^30 < 2^53)
    double* d_uqw = nullptr;
};

namespace {
thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

struct CudaFail : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaFail(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return SFC_OK;
    } catch (const CudaFail& e) {
        return set_err(SFC_ERR_CUDA, e.what());
    } catch (const std::invalid_argument& e) {
        return set_err(SFC_ERR_INVALID, e.what());
    } catch (const std::domain_error& e) {
        return set_err(SFC_ERR_DOMAIN, e.what());
    } catch (const std::length_error& e) {
        return set_err(SFC_ERR_UNSUPPORTED, e.what());
    } catch (const std::bad_alloc&) {
        return set_err(SFC_ERR_CUDA, "out of host memory");
    } catch (const std::exception& e) {
        return set_err(SFC_ERR_CUDA, e.what());
    }
}

struct Unsupported : std::length_error {
    using std::length_error::length_error;
};

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

// P_f[t][o] = sum_c V_f[t][c] U_f[o][c] for `batch` frequency slices (row-major): the fp64
// contractions tcgen05 has no kind for (f64_gemm.cu).
void dgemm_freq(const double* U, const double* V, double* P, const ConvGeom& g, int batch, cudaStream_t st) {
    ck(launch_dgemm_freq(U, V, P, g.Tpad, g.OCpad, g.Cpad, batch, st), "fp64 contraction launch");
}

// The wide (9-16 bit) tail of a general forward: vq as integer-valued doubles from the
// activation quantizer, the exact fp64 contraction, then the mode-4 epilogue (fp64 P
// dequantised per (oc, f) in the reference's order, quant.cpp:251-278).  `quantize`
// fills vq (already zeroed, [F][Tpad][Cpad]).
template <class Q>
void wide_tail(const sfc_layer* L, const ConvGeom& g, const OutPtrs& op, const QuantParams* qp, Q&& quantize,
               cudaStream_t st) {
    const size_t nv = size_t(L->F) * g.Tpad * g.Cpad, np = size_t(L->F) * g.Tpad * g.OCpad;
    double *vq = nullptr, *P = nullptr;
    ck(cudaMallocAsync(&vq, nv * sizeof(double), st), "alloc wide vq");
    ck(cudaMallocAsync(&P, np * sizeof(double), st), "alloc wide P");
    ck(cudaMemsetAsync(vq, 0, nv * sizeof(double), st), "memset wide vq");
    quantize(vq);
    dgemm_freq(L->d_uqw, vq, P, g, L->F, st);
    ck(launch_output(L->variant, 4, P, g, qp, L->d_sf, op, st, false), "output launch");
    ck(cudaFreeAsync(vq, st), "free wide vq");
    ck(cudaFreeAsync(P, st), "free wide P");
}

// Workspace carve-up (kept in sync with workspace_bytes()).
struct WsView {
    int* vmax;
    unsigned long long* sat;
    QuantParams* qp;
    int8_t* vq;
    int32_t* P;
    int16_t* vkeep;  // V kept by sfc_act_transform for the streaming quantizer
    unsigned long long* vmaxf;  // general QuantConfig: maxima (fp64 bit patterns)
    double* act_scale;  // general QuantConfig: activation scales (1 or F)
};
WsView carve(void* ws, const ConvGeom& g, int F) {
    auto up = [](size_t v) { return (v + 255) / 256 * 256; };
    uint8_t* base = static_cast<uint8_t*>(ws);
    WsView v;
    v.vmax = reinterpret_cast<int*>(base);
    v.sat = reinterpret_cast<unsigned long long*>(base + 8);
    v.qp = reinterpret_cast<QuantParams*>(base + 64);
    v.vmaxf = reinterpret_cast<unsigned long long*>(base + kWsMaxima);
    v.act_scale = reinterpret_cast<double*>(base + kWsActScales);
    v.vq = reinterpret_cast<int8_t*>(base + up(kWsHeader));
    v.P = reinterpret_cast<int32_t*>(base + up(kWsHeader) + up(size_t(F) * g.Tpad * g.Cpad));
    v.vkeep = reinterpret_cast<int16_t*>(reinterpret_cast<uint8_t*>(v.P) +
                                         up(size_t(F) * p_chunk(g, F).tcpad * g.OCpad * 4));
    return v;
}

// GEMM and output transform over P chunks (PChunk): one pair of launches when P fits the
// chunk budget, else for each chunk of image tile rows the GEMM writes that chunk's P
// rows into the chunk buffer and the output kernel consumes and discards them from L2.
// `pdl` is the PDL flag of the next launch and is left as the caller's chain expects.
void gemm_output(const sfc_layer* L, const ConvGeom& g, const WsView& v, int mode, const OutPtrs& op, bool do_gemm,
                 bool do_out, cudaStream_t st, bool& pdl, bool full_pdl) {
    const PChunk pc = p_chunk(g, L->F);
    for (int c = 0; c < pc.n; ++c) {
        const int r0 = c * pc.rows, nr = std::min(pc.rows, g.nrows - r0);
        if (do_gemm) {
            if (pc.n == 1) ck(launch_gemm(v.vq, L->d_uq, v.P, g, L->F, st, pdl), "gemm launch");
            else ck(launch_gemm_rows(v.vq, L->d_uq, v.P, g, L->F, r0 * g.tw, pc.tcpad, st, pdl), "gemm launch");
            pdl = full_pdl;
        }
        if (do_out) {
            ConvGeom gc = g;
            OutPtrs oc = op;
            if (pc.n > 1) gc.row0 = r0, gc.nrows = nr, gc.Tpad = pc.tcpad, oc.p_discard = v.P;
            ck(launch_output(L->variant, mode, v.P, gc, v.qp, L->d_sf, oc, st, pdl), "output launch");
            pdl = full_pdl;
        }
    }
}

// 24-bit planar P (ConvGeom::p24): exact while qmax^2 * Cin < 2^23 (|vq|, |uq| <= qmax under
// MinMax), for the exact int32 / int64 outputs of the 3x3 variants with P whole; the P
// round trip (GEMM epilogue writes, output transform reads) shrinks by a quarter.
// SFC_P24=0 keeps int32 P (A/B knob).
bool p24_wanted(const sfc_layer* L, const ConvGeom& g);

// |y| bound of the layer needs 64-bit accumulation (see needs_y64)
bool y_bound_needs64(const sfc_layer* L) {
    const double qmax = double((1 << (L->bits - 1)) - 1);
    return double(L->max_a_col_l1) * double(L->max_a_col_l1) * L->IC * qmax * qmax >= 2147483647.0;
}

// P storage of a GEMM + output-transform call (ConvGeom::p24): 2 = unit-major 24-bit P for the
// tensor-core output transform (out_mma.cu; 3x3 variants, int32-exact y, OC <= 1024), else
// 1 = 24-bit rows for the CUDA-core output kernels, 0 = int32.  SFC_OUT_MMA=0 keeps layout 1
// (A/B knob, read per call).
int p_layout_of(const sfc_layer* L, const ConvGeom& g) {
    if (!p24_wanted(L, g)) return 0;
    const char* e = std::getenv("SFC_OUT_MMA");
    if (e && e[0] == '0') return 1;
    if (L->variant > 2 || y_bound_needs64(L) || g.OC > 1024) return 1;
    // small grids (config 2: 200 units of 128 pairs) are latency-bound in the persistent
    // tensor-core kernel; the one-block CUDA-core kernels cover them in one short wave
    const long units = long((g.OC + kUnitOc - 1) / kUnitOc) * ((g.T + kUnitTiles - 1) / kUnitTiles);
    return units < 2L * device_sm_count() ? 1 : 2;
}

// Unit-major P stores plane 2 sparsely (sfc_kernels.hpp p2_flags_offset).  SFC_P2_DENSE=1
// keeps every row of plane 2 (A/B knob, read per call; the Python views() reads it too).
bool p2_sparse_wanted(const ConvGeom& g) {
    if (g.p24 != 2) return false;
    const char* e = std::getenv("SFC_P2_DENSE");
    return !(e && e[0] == '1');
}

bool p24_wanted(const sfc_layer* L, const ConvGeom& g) {
    const char* e = std::getenv("SFC_P24");
    if (e && e[0] == '0') return false;
    if (L->general || L->variant > 2 || p_chunk(g, L->F).n > 1) return false;
    const double qmax = double((1 << (L->bits - 1)) - 1);
    return qmax * qmax * double(L->IC) < 8388608.0;
}

// Layers with Cin <= 4 (3x3 variants, exact int32 y, whole P): the dp4a contraction fused
// with the output transform replaces the GEMM and P (launch_output_smallc); vq is written
// compact [F][T][4].  SFC_SMALLC=0 keeps the tensor-core GEMM (A/B knob, read per call).
bool small_c(const sfc_layer* L, const ConvGeom& g) {
    if (L->general || L->variant > 2 || g.C > 4 || p_chunk(g, L->F).n > 1) return false;
    if (L->max_a_col_l1 * double(L->max_a_col_l1) * L->IC * 127.0 * 127.0 >= 2147483647.0) return false;
    const char* e = std::getenv("SFC_SMALLC");
    return !(e && e[0] == '0');
}

// sfc_conv_forward's schedule (see there): recompute V when the GEMM has several output-
// channel blocks or the layer takes the small-channel path.  SFC_FORWARD_RECOMPUTE=0/1 forces
// one (A/B knob).
bool forward_recomputes(const sfc_layer* L, const ConvGeom& g) {
    if (const char* e = std::getenv("SFC_FORWARD_RECOMPUTE")) return e[0] == '1';
    return g.OCpad > g.BN || small_c(L, g);
}

void check_call(const sfc_layer* L, const void* x, int n, int h, int w, int pad) {
    if (!L) throw std::invalid_argument("null layer");
    if (!x) throw std::invalid_argument("null input");  // (the kept-V entry points pass the workspace)
    if (n <= 0 || h <= 0 || w <= 0 || pad < 0) throw std::invalid_argument("bad input shape");
    if (w > 16384 || h > 16384 || pad > 64) throw Unsupported("image sides above 16384 or padding above 64");
    if (h + 2 * pad - L->plan->R + 1 <= 0 || w + 2 * pad - L->plan->R + 1 <= 0)
        throw std::invalid_argument("filter larger than padded input");
    // tile counts, padded rows and every per-tile buffer size are formed in int / size_t
    // from these: refuse shapes whose tile count (rounded to the GEMM row block) or
    // per-frequency operand rows would not fit a signed 32-bit index
    const long long M = L->plan->M;
    const long long th = (h + 2 * pad - L->plan->R + 1 + M - 1) / M, tw = (w + 2 * pad - L->plan->R + 1 + M - 1) / M;
    const long long tiles = (long long)n * th * tw;
    if (tiles + 128 > 0x7fffffffLL || (long long)n * L->IC * h * w > 0x7fffffffffffLL)
        throw Unsupported("tile count above 2^31 - 128");
}

ConvGeom geom_of(const sfc_layer* L, int n, int h, int w, int pad) {
    ConvGeom g;
    geom_init(g, L->variant, n, L->IC, h, w, pad, L->OC);
    return g;
}

// The inspection / protocol entry points that only read a workspace a previous call filled:
// the same shape checks as a launch, and the workspace must be large enough for the shape.
WsView checked_carve(const sfc_layer* L, int n, int h, int w, int pad, void* ws, size_t ws_bytes) {
    check_call(L, ws, n, h, w, pad);
    const ConvGeom g = geom_of(L, n, h, w, pad);
    if (ws_bytes < workspace_bytes(g, L->F)) throw std::invalid_argument("workspace too small");
    return carve(ws, g, L->F);
}

// |y| <= (max_t sum_k |A[k,t]|)^2 * IC * qmax^2 (MinMax never clips, so |vq|,|uq| <= qmax):
// whether the exact y needs 64-bit accumulation; int32 y is then refused up front.
bool needs_y64(const sfc_layer* L, const sfc_outputs* o) {
    const double qmax = double((1 << (L->bits - 1)) - 1);
    const double bound = double(L->max_a_col_l1) * double(L->max_a_col_l1) * L->IC * qmax * qmax;
    const bool need64 = bound >= 2147483647.0;
    if (need64 && o && o->y_int32) throw Unsupported("y_int may exceed int32 for this layer; request y_int64 instead");
    return need64;
}

// Launch the per-call kernels.  `chained`: the previous operation on the stream is
// this call's absmax kernel, so the activation kernel may start under PDL.  Inside a
// full call every kernel after the first overlaps its predecessor's tail (PDL); the
// kernels themselves wait (griddepcontrol.wait) before consuming upstream results.
// mask & SFC_STAGE_KEPT: the activation stage quantizes the V kept in the workspace by
// sfc_act_transform (streaming) instead of recomputing the transform from x.
void run_conv(const sfc_layer* L, const int8_t* d_x, int n, int h, int w, int pad, const int32_t* d_vmax, void* ws,
              size_t ws_bytes, const sfc_outputs* o, unsigned mask, bool chained, cudaStream_t st) {
    const bool kept = (mask & SFC_STAGE_KEPT) != 0;
    mask &= SFC_STAGE_ALL;
    if (L && L->general)
        throw Unsupported("layers with a non-default QuantConfig run through sfc_conv_forward only (single GPU)");
    check_call(L, kept ? ws : static_cast<const void*>(d_x), n, h, w, pad);
    if (!d_vmax || !ws || !o) throw std::invalid_argument("null argument");
    ConvGeom g = geom_of(L, n, h, w, pad);
    g.p24 = p_layout_of(L, g);
    g.p2s = p2_sparse_wanted(g) ? 1 : 0;
    if (ws_bytes < workspace_bytes(g, L->F)) throw std::invalid_argument("workspace too small");
    const bool need64 = needs_y64(L, o);
    WsView v = carve(ws, g, L->F);
    const bool full = chained || (mask | SFC_STAGE_QPARAMS) == SFC_STAGE_ALL;
    static const bool no_pdl = std::getenv("SFC_DEBUG_NO_PDL") != nullptr;  // debugging knob
    const bool full_pdl = full && !no_pdl;
    bool pdl = chained && full_pdl;
    if (mask & SFC_STAGE_QPARAMS) {
        ck(cudaMemsetAsync(v.sat, 0, sizeof(unsigned long long), st), "memset sat");
        pdl = false;
    }
    // Kept V is quantized inside the GEMM by converter warps (the quantize launch and the vq
    // round trip disappear).  Default: the producer TMA-loads each stage's V tile into shared
    // memory next to A and B and the converters read it there (measured fastest on every
    // BASELINE config: config 2 0.067 ms, config 5 0.382 vs 0.407 streaming, ResNet-18 1.106
    // vs 1.187, VGG-16 15.38 vs 15.79).  SFC_QFUSE=0: streaming quantizer (vq through HBM);
    // 1: converters loading V through registers; 2: the default.
    bool qfuse = kept, qtma = kept;
    if (const char* q = std::getenv("SFC_QFUSE")) qfuse = kept && (q[0] == '1' || q[0] == '2'), qtma = q[0] == '2';
    const bool chunked = p_chunk(g, L->F).n > 1;
    qfuse = qfuse && !chunked;  // the converter GEMM covers the whole tile range
    if (!kept && !need64 && small_c(L, g)) {  // quantizing transform -> compact vq, fused dp4a epilogue
        ConvGeom gq = g;
        gq.Cpad = 4, gq.Tpad = g.T;  // vq [F][T][4]
        if (mask & SFC_STAGE_ACT) {
            ck(launch_act_quant(L->variant, d_x, gq, d_vmax, L->bits, v.qp, v.vq, v.sat, st, pdl), "act launch");
            pdl = full_pdl;
        }
        const OutPtrs op{o->y_int32, o->y_int64, o->out_f32, o->out_f64, o->out_i8, o->requant_scale};
        if (mask & SFC_STAGE_OUTPUT)
            ck(launch_output_smallc(L->variant, v.vq, L->d_uq, g, v.qp, L->d_sf, op, st, pdl), "output launch");
        return;
    }
    if (mask & SFC_STAGE_ACT) {
        if (!kept) {
            ck(launch_act_quant(L->variant, d_x, g, d_vmax, L->bits, v.qp, v.vq, v.sat, st, pdl), "act launch");
            pdl = full_pdl;
        } else if (!qfuse) {
            ck(launch_quant_kept(v.vkeep, g, L->F, d_vmax, L->bits, v.qp, v.vq, v.sat, st, pdl), "quantize launch");
            pdl = full_pdl;
        }
    }
    const OutPtrs op{o->y_int32, o->y_int64, o->out_f32, o->out_f64, o->out_i8, o->requant_scale};
    if (qfuse) {
        if (mask & SFC_STAGE_GEMM) {
            const QFuse qf{v.vkeep, d_vmax, qparams_table(false), v.qp, v.sat, L->bits};
            ck(qtma ? launch_gemm_qtma(qf, L->d_uq, v.P, g, L->F, st, pdl)
                    : launch_gemm_qfused(qf, L->d_uq, v.P, g, L->F, st, pdl),
               "fused quantize + gemm launch");
            pdl = full_pdl;
        }
        if (mask & SFC_STAGE_OUTPUT)
            ck(launch_output(L->variant, need64 ? 1 : 0, v.P, g, v.qp, L->d_sf, op, st, pdl), "output launch");
        return;
    }
    gemm_output(L, g, v, need64 ? 1 : 0, op, (mask & SFC_STAGE_GEMM) != 0, (mask & SFC_STAGE_OUTPUT) != 0, st, pdl,
                full_pdl);
}
}  // namespace

namespace {
// General QuantConfig (int8-valued inputs), in the steps a batch-sharded caller interleaves
// with its exchanges: prepare (absmax keeps V; this shard's activation maxima -> ws), [all-
// reduce(MAX) of the maxima; MseGrid: the rank-ordered chain of partial sums], conv (scales,
// quantize, contraction, fp64 epilogue).  quant.cpp:163-278.
void general_check(const sfc_layer* L, const sfc_outputs* o) {
    if (!L->general) throw Unsupported("the default QuantConfig shards through sfc_act_transform / sfc_conv_kept");
    if (o && (o->y_int32 || o->y_int64))
        throw Unsupported("y_int is defined only for PerTensor activation + PerChannel filter MinMax scales");
    if (L->act_scope == SFC_ACT_PER_FREQUENCY && L->F > 196) throw Unsupported("too many frequencies");
}

void general_prepare(const sfc_layer* L, const int8_t* d_x, const ConvGeom& g, const WsView& v, cudaStream_t st) {
    ck(cudaMemsetAsync(v.vmax, 0, kWsMaxima + sizeof(unsigned long long) * L->F, st), "memset header");
    ck(launch_act_absmax(L->variant, d_x, g, v.vmax, v.vkeep, st, false), "absmax launch");
    ck(launch_act_maxima(v.vkeep, g, L->F, L->act_scope == SFC_ACT_PER_FREQUENCY, v.vmaxf, st), "maxima launch");
}

void general_conv(const sfc_layer* L, const ConvGeom& g, const WsView& v, const double* err, const sfc_outputs* o,
                  cudaStream_t st) {
    const bool pf = L->act_scope == SFC_ACT_PER_FREQUENCY;
    ck(launch_act_pick(L->F, pf, v.vmaxf, L->bits, err, v.act_scale, st), "scale pick launch");
    OutPtrs op{nullptr, nullptr, o->out_f32, o->out_f64, o->out_i8, o->requant_scale};
    op.gen_act = v.act_scale, op.gen_per_freq = pf ? 1 : 0, op.gen_fil = L->d_fil;
    auto quantize = [&](void* vq) {
        ck(launch_act_quantize(v.vkeep, g, L->F, pf, v.act_scale, L->bits, vq, v.sat, st), "quantize launch");
    };
    if (L->bits > 8) return wide_tail(L, g, op, v.qp, quantize, st);
    quantize(v.vq);
    bool pdl = false;
    gemm_output(L, g, v, 2, op, true, true, st, pdl, false);
}
}  // namespace

extern "C" {

int sfc_general_prepare(sfc_layer_t L, const int8_t* d_x, int n, int h, int w, int pad, void* ws, size_t ws_bytes,
                        uint64_t** d_maxima, int* count, void* stream) {
    return guarded([&] {
        check_call(L, d_x, n, h, w, pad);
        if (!ws) throw std::invalid_argument("null workspace");
        general_check(L, nullptr);
        const ConvGeom g = geom_of(L, n, h, w, pad);
        if (ws_bytes < workspace_bytes(g, L->F)) throw std::invalid_argument("workspace too small");
        const WsView v = carve(ws, g, L->F);
        general_prepare(L, d_x, g, v, S(stream));
        if (d_maxima) *d_maxima = reinterpret_cast<uint64_t*>(v.vmaxf);
        if (count) *count = L->act_scope == SFC_ACT_PER_FREQUENCY ? L->F : 1;
    });
}

int sfc_general_mse_partial(sfc_layer_t L, int n, int h, int w, int pad, void* ws, size_t ws_bytes,
                            const double* d_err_in, double* d_err_out, void* stream) {
    return guarded([&] {
        if (!d_err_out) throw std::invalid_argument("null argument");
        const WsView v = checked_carve(L, n, h, w, pad, ws, ws_bytes);
        general_check(L, nullptr);
        if (L->search != SFC_SEARCH_MSE_GRID) throw std::invalid_argument("the layer's scale search is MinMax");
        const ConvGeom g = geom_of(L, n, h, w, pad);
        ck(launch_act_mse(v.vkeep, g, L->F, L->act_scope == SFC_ACT_PER_FREQUENCY, v.vmaxf, L->bits, d_err_in,
                          d_err_out, S(stream)),
           "mse launch");
    });
}

int sfc_general_conv(sfc_layer_t L, int n, int h, int w, int pad, void* ws, size_t ws_bytes, const double* d_err,
                     const sfc_outputs* o, void* stream) {
    return guarded([&] {
        if (!L || !ws || !o) throw std::invalid_argument("null argument");
        general_check(L, o);
        if ((L->search == SFC_SEARCH_MSE_GRID) != (d_err != nullptr))
            throw std::invalid_argument("d_err: the complete MseGrid sums for an MseGrid layer, NULL for MinMax");
        const ConvGeom g = geom_of(L, n, h, w, pad);
        if (ws_bytes < workspace_bytes(g, L->F)) throw std::invalid_argument("workspace too small");
        general_conv(L, g, carve(ws, g, L->F), d_err, o, S(stream));
    });
}

const char* sfc_last_error(void) { return g_err.c_str(); }
int sfc_version(void) { return 1; }

int sfc_catalog_json(char* buf, size_t cap, uint64_t* hash) {
    return guarded([&] {
        const std::string s = plan_export_json(plan_names());
        if (hash) *hash = fnv1a64(s);
        if (buf && cap) {
            const size_t n = std::min(cap - 1, s.size());
            std::memcpy(buf, s.data(), n);
            buf[n] = 0;
            if (s.size() >= cap) throw std::invalid_argument("buffer too small for catalog json");
        }
    });
}

int sfc_plan_create(const char* name, sfc_plan_t* out) {
    return guarded([&] {
        if (!name || !out) throw std::invalid_argument("null argument");
        *out = new sfc_plan{&plan_for(name)};
    });
}

int sfc_plan_destroy(sfc_plan_t plan) {
    delete plan;
    return SFC_OK;
}

int sfc_plan_dims(sfc_plan_t plan, int64_t* d) {
    return guarded([&] {
        if (!plan || !d) throw std::invalid_argument("null argument");
        const SfcPlan& p = *plan->p;
        const int64_t v[10] = {p.K, p.n_in, p.M, p.R, p.N, p.offset, p.a_denom, int64_t(p.corrections.size()),
                               p.mults_full(), p.mults_reduced()};
        std::memcpy(d, v, sizeof v);
    });
}

int sfc_plan_matrices(sfc_plan_t plan, int64_t* bt, int64_t* g, int64_t* a) {
    return guarded([&] {
        if (!plan) throw std::invalid_argument("null plan");
        const SfcPlan& p = *plan->p;
        if (bt) std::memcpy(bt, p.BT.data(), p.BT.size() * sizeof(int64_t));
        if (g) std::memcpy(g, p.G.data(), p.G.size() * sizeof(int64_t));
        if (a) std::memcpy(a, p.A.data(), p.A.size() * sizeof(int64_t));
    });
}

int sfc_layer_create(sfc_plan_t plan, const int8_t* d_w, int oc, int ic, int bits, int filter_scope, int search,
                     void* stream, sfc_layer_t* out) {
    return sfc_layer_create_ex(plan, d_w, oc, ic, bits, SFC_ACT_PER_TENSOR, filter_scope, search, stream, out);
}

int sfc_layer_create_ex(sfc_plan_t plan, const int8_t* d_w, int oc, int ic, int bits, int act_scope, int filter_scope,
                        int search, void* stream, sfc_layer_t* out) {
    sfc_layer* L = nullptr;
    int rc = guarded([&] {
        if (!plan || !d_w || !out) throw std::invalid_argument("null argument");
        if (bits < 2 || bits > 16) throw std::invalid_argument("quantization width must be between 2 and 16 bits");
        if (oc <= 0 || ic <= 0) throw std::invalid_argument("bad filter shape");
        if (act_scope < 0 || act_scope > 1 || filter_scope < 0 || filter_scope > 2 || search < 0 || search > 1)
            throw std::invalid_argument("bad quantization config");
        L = new sfc_layer();
        L->act_scope = act_scope, L->filter_scope = filter_scope, L->search = search;
        // bits 9-16 exceed the int8 operands: every scope then takes the fp64 parity path
        L->general = bits > 8 || !(act_scope == SFC_ACT_PER_TENSOR && filter_scope == SFC_FIL_PER_CHANNEL &&
                                   search == SFC_SEARCH_MINMAX);
        L->plan = plan->p;
        qparams_table(true);  // once per device; the kernels derive per CTA if this failed
        L->variant = plan->p->variant;
        L->OC = oc;
        L->IC = ic;
        L->bits = bits;
        L->F = plan->p->K * plan->p->K;
        ConvGeom g;
        geom_init(g, L->variant, 1, ic, 8, 8, 1, oc);
        L->BK = g.BK, L->Cpad = g.Cpad, L->BN = g.BN, L->OCpad = g.OCpad;
        for (int t = 0; t < plan->p->M; ++t) {
            int64_t l1 = 0;
            for (int k = 0; k < plan->p->K; ++k) l1 += std::abs(plan->p->a(k, t));
            L->max_a_col_l1 = std::max(L->max_a_col_l1, l1);
        }
        const size_t uq_bytes = size_t(L->F) * L->OCpad * L->Cpad;
        ck(cudaMalloc(&L->d_uq, uq_bytes), "cudaMalloc uq");
        ck(cudaMalloc(&L->d_sf, sizeof(double) * oc), "cudaMalloc sf");
        ck(cudaMalloc(&L->d_umax, sizeof(int) * oc), "cudaMalloc umax");
        ck(cudaMalloc(&L->d_sat, sizeof(unsigned long long)), "cudaMalloc sat");
        ck(cudaMemsetAsync(L->d_uq, 0, uq_bytes, S(stream)), "memset uq");
        ck(cudaMemsetAsync(L->d_sat, 0, sizeof(unsigned long long), S(stream)), "memset sat");
        if (!L->general) {
            ck(launch_filter_prepare(L->variant, d_w, oc, ic, L->Cpad, L->OCpad, bits, L->d_sf, L->d_umax, L->d_uq,
                                     L->d_sat, S(stream)),
               "filter prepare launch");
        } else {
            // U exactly, per-group scales in the reference's order, quantize (quant.cpp:183-229)
            const int F = L->F;
            L->n_fil_native = filter_scope == SFC_FIL_PER_CHANNEL ? oc : (filter_scope == SFC_FIL_PER_FREQUENCY ? F : oc * F);
            ck(cudaMalloc(&L->d_fil, sizeof(double) * size_t(oc) * F), "cudaMalloc fil");
            ck(cudaMalloc(&L->d_fil_native, sizeof(double) * L->n_fil_native), "cudaMalloc fil native");
            int32_t* U = nullptr;
            double* err = nullptr;
            ck(cudaMallocAsync(&U, sizeof(int32_t) * size_t(oc) * ic * F, S(stream)), "alloc U");
            ck(cudaMallocAsync(&err, sizeof(double) * size_t(L->n_fil_native) * 101, S(stream)), "alloc err");
            ck(launch_transform_filters(L->variant, d_w, oc, ic, U, S(stream)), "transform filters launch");
            void* uq_out = L->d_uq;
            if (bits > 8) {
                const size_t n = size_t(F) * L->OCpad * L->Cpad;
                ck(cudaMalloc(&L->d_uqw, n * sizeof(double)), "cudaMalloc wide uq");
                ck(cudaMemsetAsync(L->d_uqw, 0, n * sizeof(double), S(stream)), "memset wide uq");
                uq_out = L->d_uqw;
            }
            ck(launch_fil_general(U, oc, ic, F, filter_scope, search == SFC_SEARCH_MSE_GRID, bits, L->Cpad, L->OCpad,
                                  L->d_fil_native, err, uq_out, L->d_fil, L->d_sat, S(stream)),
               "general filter launch");
            ck(cudaFreeAsync(U, S(stream)), "free U");
            ck(cudaFreeAsync(err, S(stream)), "free err");
            ck(cudaMemsetAsync(L->d_umax, 0, sizeof(int) * oc, S(stream)), "memset umax");
            if (filter_scope == SFC_FIL_PER_CHANNEL)
                ck(cudaMemcpyAsync(L->d_sf, L->d_fil_native, sizeof(double) * oc, cudaMemcpyDeviceToDevice, S(stream)),
                   "copy sf");
            else
                ck(cudaMemsetAsync(L->d_sf, 0, sizeof(double) * oc, S(stream)), "memset sf");
        }
        ck(cudaStreamSynchronize(S(stream)), "filter prepare");
        *out = L;
    });
    if (rc != SFC_OK && L) sfc_layer_destroy(L);
    return rc;
}

int sfc_layer_destroy(sfc_layer_t L) {
    if (!L) return SFC_OK;
    cudaFree(L->d_uq);
    cudaFree(L->d_sf);
    cudaFree(L->d_umax);
    cudaFree(L->d_sat);
    cudaFree(L->d_fil);
    cudaFree(L->d_fil_native);
    cudaFree(L->d_uqw);
    delete L;
    return SFC_OK;
}

int sfc_layer_filter_scales_native(sfc_layer_t L, double* scales, int64_t* count) {
    return guarded([&] {
        if (!L || !count) throw std::invalid_argument("null argument");
        if (!L->general) {
            *count = L->OC;
            if (scales) ck(cudaMemcpy(scales, L->d_sf, sizeof(double) * L->OC, cudaMemcpyDeviceToHost), "copy sf");
            return;
        }
        *count = L->n_fil_native;
        if (scales)
            ck(cudaMemcpy(scales, L->d_fil_native, sizeof(double) * L->n_fil_native, cudaMemcpyDeviceToHost),
               "copy scales");
    });
}

int sfc_layer_filter_scales(sfc_layer_t L, double* sf, int32_t* umax) {
    return guarded([&] {
        if (!L) throw std::invalid_argument("null layer");
        if (sf) ck(cudaMemcpy(sf, L->d_sf, sizeof(double) * L->OC, cudaMemcpyDeviceToHost), "copy sf");
        if (umax) ck(cudaMemcpy(umax, L->d_umax, sizeof(int) * L->OC, cudaMemcpyDeviceToHost), "copy umax");
    });
}

int sfc_layer_saturations(sfc_layer_t L, int64_t* count) {
    return guarded([&] {
        if (!L || !count) throw std::invalid_argument("null argument");
        unsigned long long c = 0;
        ck(cudaMemcpy(&c, L->d_sat, sizeof c, cudaMemcpyDeviceToHost), "copy sat");
        *count = int64_t(c);
    });
}

int sfc_layer_uq(sfc_layer_t L, const int8_t** d_uq, int64_t* ic_pitch, int64_t* oc_pitch) {
    return guarded([&] {
        if (!L) throw std::invalid_argument("null layer");
        if (d_uq) *d_uq = L->d_uq;
        if (ic_pitch) *ic_pitch = L->Cpad;
        if (oc_pitch) *oc_pitch = L->OCpad;
    });
}

int sfc_conv_workspace_size(sfc_layer_t L, int n, int h, int w, int pad, size_t* bytes) {
    return guarded([&] {
        if (!L || !bytes) throw std::invalid_argument("null argument");
        if (n <= 0 || h <= 0 || w <= 0 || pad < 0) throw std::invalid_argument("bad input shape");
    if (w > 16384 || h > 16384 || pad > 64) throw Unsupported("image sides above 16384 or padding above 64");
        *bytes = workspace_bytes(geom_of(L, n, h, w, pad), L->F);
    });
}

int sfc_act_absmax(sfc_layer_t L, const int8_t* d_x, int n, int h, int w, int pad, int32_t* d_vmax, void* stream) {
    return guarded([&] {
        check_call(L, d_x, n, h, w, pad);
        if (!d_vmax) throw std::invalid_argument("null vmax");
        ck(launch_act_absmax(L->variant, d_x, geom_of(L, n, h, w, pad), d_vmax, nullptr, S(stream)), "absmax launch");
    });
}

int sfc_act_transform(sfc_layer_t L, const int8_t* d_x, int n, int h, int w, int pad, int32_t* d_vmax, void* ws,
                      size_t ws_bytes, void* stream) {
    return guarded([&] {
        check_call(L, d_x, n, h, w, pad);
        if (!d_vmax || !ws) throw std::invalid_argument("null argument");
        const ConvGeom g = geom_of(L, n, h, w, pad);
        if (ws_bytes < workspace_bytes(g, L->F)) throw std::invalid_argument("workspace too small");
        ck(launch_act_absmax(L->variant, d_x, g, d_vmax, carve(ws, g, L->F).vkeep, S(stream)), "absmax launch");
    });
}

int sfc_conv_kept(sfc_layer_t L, int n, int h, int w, int pad, const int32_t* d_vmax, void* ws, size_t ws_bytes,
                  const sfc_outputs* o, void* stream) {
    return guarded([&] {
        run_conv(L, nullptr, n, h, w, pad, d_vmax, ws, ws_bytes, o, SFC_STAGE_ALL | SFC_STAGE_KEPT, false, S(stream));
    });
}

int sfc_conv_int8(sfc_layer_t L, const int8_t* d_x, int n, int h, int w, int pad, const int32_t* d_vmax, void* ws,
                  size_t ws_bytes, const sfc_outputs* o, void* stream) {
    return sfc_conv_int8_stages(L, d_x, n, h, w, pad, d_vmax, ws, ws_bytes, o, SFC_STAGE_ALL, stream);
}

int sfc_conv_int8_stages(sfc_layer_t L, const int8_t* d_x, int n, int h, int w, int pad, const int32_t* d_vmax,
                         void* ws, size_t ws_bytes, const sfc_outputs* o, unsigned mask, void* stream) {
    return guarded([&] { run_conv(L, d_x, n, h, w, pad, d_vmax, ws, ws_bytes, o, mask, false, S(stream)); });
}

int sfc_conv_forward(sfc_layer_t L, const int8_t* d_x, int n, int h, int w, int pad, void* ws, size_t ws_bytes,
                     const sfc_outputs* o, void* stream) {
    return guarded([&] {
        check_call(L, d_x, n, h, w, pad);
        if (!ws) throw std::invalid_argument("null workspace");
        const ConvGeom g = geom_of(L, n, h, w, pad);
        if (ws_bytes < workspace_bytes(g, L->F)) throw std::invalid_argument("workspace too small");
        WsView v = carve(ws, g, L->F);
        if (!o) throw std::invalid_argument("null outputs");
        if (L->general) {  // non-default QuantConfig: fp64 parity path (quant.cpp:163-278)
            // the batch-sharded steps on the whole batch; the MseGrid sums use the (not yet
            // written) vq region of the workspace as scratch
            general_check(L, o);
            general_prepare(L, d_x, g, v, S(stream));
            double* err = reinterpret_cast<double*>(v.vq);
            const bool mse = L->search == SFC_SEARCH_MSE_GRID;
            if (mse) ck(launch_act_mse(v.vkeep, g, L->F, L->act_scope == SFC_ACT_PER_FREQUENCY, v.vmaxf, L->bits,
                                       nullptr, err, S(stream)),
                        "mse launch");
            general_conv(L, g, v, mse ? err : nullptr, o, S(stream));
            return;
        }
        needs_y64(L, o);  // refuse before anything is launched
        unsigned mask = SFC_STAGE_ALL & ~SFC_STAGE_QPARAMS;
        if (const char* dbg = std::getenv("SFC_DEBUG_FORWARD_MASK")) mask = unsigned(std::atoi(dbg));  // profiling only
        // Two schedules, bit-identical.  Kept V: the absmax pass keeps V (int16) and the GEMM's
        // converter warps quantize it into the A tiles.  Recompute: absmax only, then a
        // quantizing transform writes vq (int8) for a TMA-fed GEMM.  The converters quantize
        // every A tile once per output-channel block, so with several blocks (OCpad > BN) the
        // recompute schedule wins (config 5: 0.331 vs 0.359 ms); with one block the kept V
        // saves the second pass over x (ResNet-18 layer 0: 0.127 vs 0.150 ms, VGG-16 layer 2:
        // 1.31 vs 1.49 ms).  forward_recomputes() decides; sfc_conv_schedule reports it.
        const bool recompute = forward_recomputes(L, g);
        // vmax and the saturation counter share the first 16 bytes of the workspace
        ck(launch_zero_words(reinterpret_cast<uint32_t*>(v.vmax), 4, S(stream)), "workspace reset launch");
        ck(launch_act_absmax(L->variant, d_x, g, v.vmax, recompute ? nullptr : v.vkeep, S(stream), true),
           "absmax launch");
        run_conv(L, d_x, n, h, w, pad, v.vmax, ws, ws_bytes, o, recompute ? mask : mask | SFC_STAGE_KEPT, true,
                 S(stream));
    });
}

int sfc_conv_stats(sfc_layer_t L, int n, int h, int w, int pad, const void* ws, size_t ws_bytes, int64_t* stats,
                   void* stream) {
    return guarded([&] {
        if (!stats) throw std::invalid_argument("null argument");
        WsView v = checked_carve(L, n, h, w, pad, const_cast<void*>(ws), ws_bytes);
        const ConvGeom g = geom_of(L, n, h, w, pad);
        QuantParams qp;
        unsigned long long sat = 0;
        ck(cudaMemcpyAsync(&qp, v.qp, sizeof qp, cudaMemcpyDeviceToHost, S(stream)), "copy qp");
        ck(cudaMemcpyAsync(&sat, v.sat, sizeof sat, cudaMemcpyDeviceToHost, S(stream)), "copy sat");
        if (L->general) {  // the activation scale (first if per frequency) and the global max
            ck(cudaMemcpyAsync(&qp.sa, v.act_scale, sizeof(double), cudaMemcpyDeviceToHost, S(stream)), "copy sa");
            ck(cudaMemcpyAsync(&qp.vmax, v.vmax, sizeof(int), cudaMemcpyDeviceToHost, S(stream)), "copy vmax");
            qp.exact = 0;
        }
        ck(cudaStreamSynchronize(S(stream)), "stats sync");
        std::memcpy(&stats[0], &qp.sa, sizeof(double));
        stats[1] = qp.vmax;
        stats[2] = int64_t(sat);
        stats[3] = qp.exact;
        stats[4] = int64_t(L->OC) * L->IC * L->F + int64_t(g.T) * L->IC * L->F;
        stats[5] = g.T;
    });
}

int sfc_conv_act_scales(sfc_layer_t L, int n, int h, int w, int pad, const void* ws, size_t ws_bytes, double* scales,
                        int64_t* count, void* stream) {
    return guarded([&] {
        if (!count) throw std::invalid_argument("null argument");
        WsView v = checked_carve(L, n, h, w, pad, const_cast<void*>(ws), ws_bytes);
        *count = L->general && L->act_scope == SFC_ACT_PER_FREQUENCY ? L->F : 1;
        if (!scales) return;
        if (L->general) {
            ck(cudaMemcpyAsync(scales, v.act_scale, sizeof(double) * size_t(*count), cudaMemcpyDeviceToHost, S(stream)),
               "copy scales");
        } else {
            QuantParams qp;
            ck(cudaMemcpyAsync(&qp, v.qp, sizeof qp, cudaMemcpyDeviceToHost, S(stream)), "copy qp");
            ck(cudaStreamSynchronize(S(stream)), "sync");
            scales[0] = qp.sa;
        }
        ck(cudaStreamSynchronize(S(stream)), "sync");
    });
}

int sfc_conv_views(sfc_layer_t L, int n, int h, int w, int pad, void* ws, size_t ws_bytes, int8_t** d_vq,
                   int32_t** d_pacc, int64_t* geom) {
    return guarded([&] {
        WsView v = checked_carve(L, n, h, w, pad, ws, ws_bytes);
        const ConvGeom g = geom_of(L, n, h, w, pad);
        if (d_vq) *d_vq = v.vq;
        if (d_pacc) *d_pacc = p_chunk(g, L->F).n > 1 || small_c(L, g) ? nullptr : v.P;
        if (geom) {
            geom[0] = g.T, geom[1] = g.Tpad, geom[2] = g.Cpad, geom[3] = g.OCpad, geom[4] = g.th, geom[5] = g.tw;
        }
    });
}

int sfc_conv_schedule(sfc_layer_t L, int n, int h, int w, int pad, int* recompute, int* p_layout) {
    return guarded([&] {
        if (!L) throw std::invalid_argument("null argument");
        check_call(L, L, n, h, w, pad);
        const ConvGeom g = geom_of(L, n, h, w, pad);
        if (recompute) *recompute = forward_recomputes(L, g) ? 1 : 0;
        if (p_layout) *p_layout = small_c(L, g) ? 3 : p_layout_of(L, g);
    });
}

int sfc_direct_conv_int8(const int8_t* d_x, int n, int c, int h, int w, const int8_t* d_w, int oc, int r, int stride,
                         int pad, int32_t* d_out, void* stream) {
    return guarded([&] {
        if (!d_x || !d_w || !d_out) throw std::invalid_argument("null argument");
        if (stride < 1) throw std::invalid_argument("stride must be positive");
        if ((h + 2 * pad - r) / stride + 1 <= 0 || (w + 2 * pad - r) / stride + 1 <= 0 || h + 2 * pad < r ||
            w + 2 * pad < r)
            throw std::invalid_argument("filter larger than padded input");
        ck(launch_direct_conv(d_x, n, c, h, w, d_w, oc, r, stride, pad, d_out, S(stream)), "direct conv launch");
    });
}

int sfc_frequency_energy_int8(sfc_plan_t plan, const int8_t* d_x, int n, int c, int h, int w, int pad,
                              unsigned long long* d_sum, void* stream) {
    return guarded([&] {
        if (!plan || !d_x || !d_sum) throw std::invalid_argument("null argument");
        if (h + 2 * pad - plan->p->R + 1 <= 0 || w + 2 * pad - plan->p->R + 1 <= 0)
            throw std::invalid_argument("filter larger than padded input");
        ConvGeom g;
        geom_init(g, plan->p->variant, n, c, h, w, pad, 1);
        ck(launch_freq_energy(plan->p->variant, d_x, g, d_sum, S(stream)), "energy launch");
    });
}

int sfc_transform_filters_int8(sfc_plan_t plan, const int8_t* d_w, int oc, int ic, int32_t* d_u, void* stream) {
    return guarded([&] {
        if (!plan || !d_w || !d_u) throw std::invalid_argument("null argument");
        ck(launch_transform_filters(plan->p->variant, d_w, oc, ic, d_u, S(stream)), "transform filters launch");
    });
}

int sfc_transform_filters_f64(sfc_plan_t plan, const double* d_w, int oc, int ic, double* d_u, void* stream) {
    return guarded([&] {
        if (!plan || !d_w || !d_u) throw std::invalid_argument("null argument");
        if (oc <= 0 || ic <= 0) throw std::invalid_argument("bad filter shape");
        ck(launch_filters_f64(plan->p->variant, d_w, oc, ic, d_u, S(stream)), "fp64 filter transform launch");
    });
}

int sfc_report_sq_err(const double* d_out, const int32_t* d_ref, int64_t n, double* host_sums, void* stream) {
    return guarded([&] {
        if (!d_out || !d_ref || !host_sums || n < 0) throw std::invalid_argument("bad report arguments");
        void* d_sums = nullptr;
        ck(cudaMallocAsync(&d_sums, (2 + 2 * kSqErrBlocks) * sizeof(double), S(stream)), "alloc");
        ck(launch_sq_err(d_out, d_ref, n, static_cast<double*>(d_sums), S(stream)), "sq_err launch");
        ck(cudaMemcpyAsync(host_sums, d_sums, 2 * sizeof(double), cudaMemcpyDeviceToHost, S(stream)), "copy");
        ck(cudaFreeAsync(d_sums, S(stream)), "free");
        ck(cudaStreamSynchronize(S(stream)), "sync");
    });
}

int sfc_report_sq_err_f64(const double* d_out, const double* d_ref, int64_t n, double* host_sums, void* stream) {
    return guarded([&] {
        if (!d_out || !d_ref || !host_sums || n < 0) throw std::invalid_argument("bad report arguments");
        void* d_sums = nullptr;
        ck(cudaMallocAsync(&d_sums, (2 + 2 * kSqErrBlocks) * sizeof(double), S(stream)), "alloc");
        ck(launch_sq_err_f64(d_out, d_ref, n, static_cast<double*>(d_sums), S(stream)), "sq_err launch");
        ck(cudaMemcpyAsync(host_sums, d_sums, 2 * sizeof(double), cudaMemcpyDeviceToHost, S(stream)), "copy");
        ck(cudaFreeAsync(d_sums, S(stream)), "free");
        ck(cudaStreamSynchronize(S(stream)), "sync");
    });
}

int sfc_direct_conv_f64(const double* d_x, int n, int c, int h, int w, const double* d_weights, int oc, int r,
                        int stride, int pad, double* d_out, void* stream) {
    return guarded([&] {
        if (!d_x || !d_weights || !d_out) throw std::invalid_argument("null argument");
        if (n <= 0 || c <= 0 || h <= 0 || w <= 0 || oc <= 0 || r <= 0 || stride < 1 || pad < 0)
            throw std::invalid_argument("bad direct conv arguments");
        if ((h + 2 * pad - r) / stride + 1 <= 0 || (w + 2 * pad - r) / stride + 1 <= 0 || h + 2 * pad < r ||
            w + 2 * pad < r)
            throw std::invalid_argument("filter larger than padded input");
        ck(launch_direct_f64(d_x, n, c, h, w, d_weights, oc, r, stride, pad, d_out, S(stream)), "direct conv launch");
    });
}

int sfc_layer_create_f64(sfc_plan_t plan, const double* d_w, int oc, int ic, int bits, int act_scope,
                         int filter_scope, int search, void* stream, sfc_layer_t* out) {
    sfc_layer* L = nullptr;
    int rc = guarded([&] {
        if (!plan || !d_w || !out) throw std::invalid_argument("null argument");
        if (bits < 2 || bits > 16) throw std::invalid_argument("quantization width must be between 2 and 16 bits");
        if (oc <= 0 || ic <= 0) throw std::invalid_argument("bad filter shape");
        if (act_scope < 0 || act_scope > 1 || filter_scope < 0 || filter_scope > 2 || search < 0 || search > 1)
            throw std::invalid_argument("bad quantization config");
        L = new sfc_layer();
        L->act_scope = act_scope, L->filter_scope = filter_scope, L->search = search;
        L->general = true;  // real-valued tensors: the fp64 epilogue (no integer y)
        L->plan = plan->p;
        L->variant = plan->p->variant;
        L->OC = oc, L->IC = ic, L->bits = bits;
        L->F = plan->p->K * plan->p->K;
        ConvGeom g;
        geom_init(g, L->variant, 1, ic, 8, 8, 1, oc);
        L->BK = g.BK, L->Cpad = g.Cpad, L->BN = g.BN, L->OCpad = g.OCpad;
        const int F = L->F;
        L->n_fil_native = filter_scope == SFC_FIL_PER_CHANNEL ? oc : (filter_scope == SFC_FIL_PER_FREQUENCY ? F : oc * F);
        const size_t uq_bytes = size_t(F) * L->OCpad * L->Cpad;
        ck(cudaMalloc(&L->d_uq, uq_bytes), "cudaMalloc uq");
        ck(cudaMalloc(&L->d_sf, sizeof(double) * oc), "cudaMalloc sf");
        ck(cudaMalloc(&L->d_umax, sizeof(int) * oc), "cudaMalloc umax");
        ck(cudaMalloc(&L->d_sat, sizeof(unsigned long long)), "cudaMalloc sat");
        ck(cudaMalloc(&L->d_fil, sizeof(double) * size_t(oc) * F), "cudaMalloc fil");
        ck(cudaMalloc(&L->d_fil_native, sizeof(double) * L->n_fil_native), "cudaMalloc fil native");
        ck(cudaMemsetAsync(L->d_uq, 0, uq_bytes, S(stream)), "memset uq");
        ck(cudaMemsetAsync(L->d_sat, 0, sizeof(unsigned long long), S(stream)), "memset sat");
        ck(cudaMemsetAsync(L->d_umax, 0, sizeof(int) * oc, S(stream)), "memset umax");
        ck(cudaMemsetAsync(L->d_sf, 0, sizeof(double) * oc, S(stream)), "memset sf");
        double *U = nullptr, *err = nullptr;
        ck(cudaMallocAsync(&U, sizeof(double) * size_t(oc) * ic * F, S(stream)), "alloc U");
        ck(cudaMallocAsync(&err, sizeof(double) * size_t(L->n_fil_native) * 101, S(stream)), "alloc err");
        ck(launch_filters_f64(L->variant, d_w, oc, ic, U, S(stream)), "fp64 filter transform launch");
        void* uq_out = L->d_uq;
        if (bits > 8) {
            const size_t nw = size_t(F) * L->OCpad * L->Cpad;
            ck(cudaMalloc(&L->d_uqw, nw * sizeof(double)), "cudaMalloc wide uq");
            ck(cudaMemsetAsync(L->d_uqw, 0, nw * sizeof(double), S(stream)), "memset wide uq");
            uq_out = L->d_uqw;
        }
        ck(launch_fil_general_f64(U, oc, ic, F, filter_scope, search == SFC_SEARCH_MSE_GRID, bits, L->Cpad, L->OCpad,
                                  L->d_fil_native, err, uq_out, L->d_fil, L->d_sat, S(stream)),
           "general filter launch");
        ck(cudaFreeAsync(U, S(stream)), "free U");
        ck(cudaFreeAsync(err, S(stream)), "free err");
        if (filter_scope == SFC_FIL_PER_CHANNEL)
            ck(cudaMemcpyAsync(L->d_sf, L->d_fil_native, sizeof(double) * oc, cudaMemcpyDeviceToDevice, S(stream)),
               "copy sf");
        ck(cudaStreamSynchronize(S(stream)), "filter prepare");
        *out = L;
    });
    if (rc != SFC_OK && L) sfc_layer_destroy(L);
    return rc;
}

int sfc_conv_forward_f64(sfc_layer_t L, const double* d_x, int n, int h, int w, int pad, void* ws, size_t ws_bytes,
                         const sfc_outputs* o, void* stream) {
    return guarded([&] {
        check_call(L, d_x, n, h, w, pad);
        if (!ws || !o) throw std::invalid_argument("null argument");
        if (!L->general) throw Unsupported("real-valued inputs need a layer from sfc_layer_create_f64 / _ex");
        if (o->y_int32 || o->y_int64) throw Unsupported("y_int is not defined for real-valued tensors");
        const ConvGeom g = geom_of(L, n, h, w, pad);
        if (ws_bytes < workspace_bytes(g, L->F)) throw std::invalid_argument("workspace too small");
        WsView v = carve(ws, g, L->F);
        ck(cudaMemsetAsync(ws, 0, kWsMaxima + sizeof(unsigned long long) * L->F, S(stream)), "memset header");
        double* Vd = nullptr;
        ck(cudaMallocAsync(&Vd, sizeof(double) * size_t(L->F) * g.Tpad * g.Cpad, S(stream)), "alloc V");
        ck(launch_act_f64(L->variant, d_x, g, Vd, S(stream)), "fp64 input transform launch");
        const bool pf = L->act_scope == SFC_ACT_PER_FREQUENCY;
        OutPtrs op{nullptr, nullptr, o->out_f32, o->out_f64, o->out_i8, o->requant_scale};
        op.gen_act = v.act_scale, op.gen_per_freq = pf ? 1 : 0, op.gen_fil = L->d_fil;
        auto quantize = [&](void* vq) {
            ck(launch_act_general_f64(Vd, g, L->F, pf, L->search == SFC_SEARCH_MSE_GRID, L->bits, v.vmaxf, v.act_scale,
                                      vq, v.sat, reinterpret_cast<double*>(v.vq), S(stream)),
               "general activation launch");
        };
        if (L->bits > 8) {
            wide_tail(L, g, op, v.qp, quantize, S(stream));
            ck(cudaFreeAsync(Vd, S(stream)), "free V");
            return;
        }
        quantize(v.vq);
        ck(cudaFreeAsync(Vd, S(stream)), "free V");
        bool pdl = false;
        gemm_output(L, g, v, 2, op, true, true, S(stream), pdl, false);
    });
}

int sfc_fast_conv_f64(sfc_plan_t plan, const double* d_x, int n, int c, int h, int w, const double* d_weights,
                      int oc, int pad, int reduced, double* d_out, int64_t* counters, void* stream) {
    return guarded([&] {
        if (!plan || !d_x || !d_weights || !d_out) throw std::invalid_argument("null argument");
        if (n <= 0 || c <= 0 || h <= 0 || w <= 0 || oc <= 0 || pad < 0) throw std::invalid_argument("bad shape");
        const SfcPlan& P = *plan->p;
        if (h + 2 * pad - P.R + 1 <= 0 || w + 2 * pad - P.R + 1 <= 0)
            throw std::invalid_argument("filter larger than padded input");
        if (w > 16384 || h > 16384) throw Unsupported("image sides above 16384");
        ConvGeom g;
        geom_init(g, P.variant, n, c, h, w, pad, oc);
        const int F = P.K * P.K;
        const cudaStream_t st = S(stream);
        const size_t nv = size_t(F) * g.Tpad * g.Cpad, nu = size_t(oc) * c * F, nb = size_t(F) * g.OCpad * g.Cpad;
        const size_t np = size_t(F) * g.Tpad * g.OCpad;
        double *Vd = nullptr, *U = nullptr, *Ub = nullptr, *Pd = nullptr;
        void* dummy = nullptr;  // QuantParams / sf the epilogue reads but mode 3 ignores
        ck(cudaMallocAsync(&Vd, nv * sizeof(double), st), "alloc V");
        ck(cudaMallocAsync(&U, nu * sizeof(double), st), "alloc U");
        ck(cudaMallocAsync(&Ub, nb * sizeof(double), st), "alloc Ub");
        ck(cudaMallocAsync(&Pd, np * sizeof(double), st), "alloc P");
        ck(cudaMallocAsync(&dummy, 4096, st), "alloc");
        ck(cudaMemsetAsync(Vd, 0, nv * sizeof(double), st), "memset V");  // padding rows/channels are 0
        ck(cudaMemsetAsync(Ub, 0, nb * sizeof(double), st), "memset Ub");
        ck(cudaMemsetAsync(dummy, 0, 4096, st), "memset");
        ck(launch_act_f64(P.variant, d_x, g, Vd, st), "fp64 input transform launch");
        ck(launch_filters_f64(P.variant, d_weights, oc, c, U, st), "fp64 filter transform launch");
        ck(launch_pack_u_f64(U, oc, c, F, g.Cpad, g.OCpad, Ub, st), "pack launch");
        auto gemm = [&](const double* Ua, const double* Va, double* Pa, int batch) {
            dgemm_freq(Ua, Va, Pa, g, batch, st);
        };
        const PairedSchedule* ps = nullptr;
        if (reduced) {  // conv.cpp:399-403: no schedule (no triples) means the full product set
            const PairedSchedule& cand = paired_schedule(P);
            if (cand.available) ps = &cand;
        }
        long products = F;
        if (!ps) {
            gemm(Ub, Vd, Pd, F);
        } else {
            // reduced batch: the unpaired positions, then six evaluation products per block
            std::vector<PairSlice> slices;
            std::vector<PairFold> folds(size_t(F), PairFold{0, 0, {0, 0, 0, 0, 0, 0}});
            for (int f = 0; f < F; ++f)
                if (!ps->masked[size_t(f)]) {
                    folds[size_t(f)] = PairFold{1, int(slices.size()), {0, 0, 0, 0, 0, 0}};
                    slices.push_back(PairSlice{1, {f, 0, 0, 0}, {1, 0, 0, 0}, {1, 0, 0, 0}});
                }
            for (const PairBlock& b : ps->blocks) {
                const int base = int(slices.size());
                int corner[4];
                for (int q = 0; q < 4; ++q) corner[q] = b.r1[q >> 1] * P.K + b.r2[q & 1];
                for (int l = 0; l < 6; ++l) {
                    PairSlice sl{4, {corner[0], corner[1], corner[2], corner[3]}, {}, {}};
                    for (int q = 0; q < 4; ++q) sl.a[q] = b.alpha[l][q], sl.b[q] = b.beta[l][q];
                    slices.push_back(sl);
                }
                for (int q = 0; q < 4; ++q) {
                    PairFold& fd = folds[size_t(corner[q])];
                    fd.kind = 2, fd.src = base;
                    for (int l = 0; l < 6; ++l) fd.w[l] = b.fold[q][l];
                }
            }
            const int ns = int(slices.size());
            products = ns;
            const long long ev = (long long)g.Tpad * g.Cpad, eu = (long long)g.OCpad * g.Cpad,
                            ep = (long long)g.Tpad * g.OCpad;
            double *Vr = nullptr, *Ur = nullptr, *Pr = nullptr;
            PairSlice* dsl = nullptr;
            PairFold* dfd = nullptr;
            ck(cudaMallocAsync(&Vr, size_t(ns) * ev * sizeof(double), st), "alloc Vr");
            ck(cudaMallocAsync(&Ur, size_t(ns) * eu * sizeof(double), st), "alloc Ur");
            ck(cudaMallocAsync(&Pr, size_t(ns) * ep * sizeof(double), st), "alloc Pr");
            ck(cudaMallocAsync(&dsl, slices.size() * sizeof(PairSlice), st), "alloc slices");
            ck(cudaMallocAsync(&dfd, folds.size() * sizeof(PairFold), st), "alloc folds");
            ck(cudaMemcpyAsync(dsl, slices.data(), slices.size() * sizeof(PairSlice), cudaMemcpyHostToDevice, st),
               "copy slices");
            ck(cudaMemcpyAsync(dfd, folds.data(), folds.size() * sizeof(PairFold), cudaMemcpyHostToDevice, st),
               "copy folds");
            ck(launch_pair_gather(Vd, ev, dsl, ns, false, Vr, st), "pair gather launch");
            ck(launch_pair_gather(Ub, eu, dsl, ns, true, Ur, st), "pair gather launch");
            gemm(Ur, Vr, Pr, ns);
            ck(launch_pair_fold(Pr, ep, dfd, F, Pd, st), "pair fold launch");
            // the host tables are pageable: the copies above finished staging before returning
            for (void* p : {static_cast<void*>(Vr), static_cast<void*>(Ur), static_cast<void*>(Pr),
                            static_cast<void*>(dsl), static_cast<void*>(dfd)})
                ck(cudaFreeAsync(p, st), "free");
        }
        OutPtrs op{nullptr, nullptr, nullptr, d_out, nullptr, 0.0};
        ck(launch_output(P.variant, 3, Pd, g, static_cast<const QuantParams*>(dummy),
                         static_cast<const double*>(dummy), op, st, false),
           "output launch");
        for (void* p : {static_cast<void*>(Vd), static_cast<void*>(U), static_cast<void*>(Ub), static_cast<void*>(Pd),
                        dummy})
            ck(cudaFreeAsync(p, st), "free");
        if (counters) {  // conv.hpp ConvCounters: products actually formed, tiles
            counters[0] = int64_t(g.T) * oc * c * products;
            counters[1] = g.T;
        }
    });
}

int sfc_debug_timeline(uint64_t* out, int reset) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("null argument");
        ck(cudaDeviceSynchronize(), "sync");
        unsigned long long part[5][kTlCount][3];
        cudaError_t (*readers[5])(unsigned long long*, bool) = {tl_read_aux, tl_read_act, tl_read_reg, tl_read_gemm, tl_read_out};
        for (int u = 0; u < 5; ++u) {
            const cudaError_t e = readers[u](&part[u][0][0], reset != 0);
            if (e == cudaErrorNotSupported) throw Unsupported("not the timeline build (make TIMELINE=1)");
            ck(e, "timeline read");
        }
        for (int k = 0; k < kTlCount; ++k) {
            unsigned long long a = ~0ull, b = ~0ull, c = 0;
            for (int u = 0; u < 5; ++u) {
                a = std::min(a, part[u][k][0]);
                b = std::min(b, part[u][k][1]);
                c = std::max(c, part[u][k][2]);
            }
            out[3 * k] = a, out[3 * k + 1] = b, out[3 * k + 2] = c;
        }
    });
}

int sfc_debug_quantizer(int vmax, int bits, int32_t* d_q, int64_t* info, void* stream) {
    return guarded([&] {
        if (!d_q || vmax < 0 || bits < 2 || bits > 8) throw std::invalid_argument("bad quantizer probe");
        void* scratch = nullptr;
        ck(cudaMallocAsync(&scratch, 256, S(stream)), "alloc");
        int* d_vmax = static_cast<int*>(scratch);
        unsigned long long* sat = reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(scratch) + 8);
        QuantParams* qp = reinterpret_cast<QuantParams*>(static_cast<uint8_t*>(scratch) + 64);
        ck(cudaMemcpyAsync(d_vmax, &vmax, sizeof(int), cudaMemcpyHostToDevice, S(stream)), "copy vmax");
        qparams_table(true);
        ck(launch_quant_params(d_vmax, bits, qp, sat, S(stream)), "qparams");
        ck(launch_debug_quant(qp, vmax, d_q, sat, S(stream)), "debug quant");
        QuantParams h;
        ck(cudaMemcpyAsync(&h, qp, sizeof h, cudaMemcpyDeviceToHost, S(stream)), "copy qp");
        ck(cudaStreamSynchronize(S(stream)), "sync");
        ck(cudaFreeAsync(scratch, S(stream)), "free");
        if (info) {
            info[0] = h.exact;
            info[1] = h.shift;
            info[2] = h.mul;
            std::memcpy(&info[3], &h.sa, sizeof(double));
        }
    });
}

}  // extern "C"
