/* C-ABI of the B200 quantized SFC 3x3 convolution (libsfc_b200.so).
 *
 * This is the drop-in boundary a host binding (ctypes / cgo / JNI / the C++
 * `sfconv::` shim in include/sfconv/) calls.  Plain pointers, sizes and opaque
 * handles only.  Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj).
 *
 * Conventions
 *  - Return 0 on success, a negative SFC_ERR_* code otherwise; the message is
 *    in a thread-local buffer read with sfc_last_error().  The C++ shim maps
 *    the codes to the reference's exception types:
 *      SFC_ERR_INVALID     -> std::invalid_argument   (quant.cpp:155-156, conv.cpp:353-355, quant.cpp:49)
 *      SFC_ERR_DOMAIN      -> std::domain_error       (catalog.cpp:284-285)
 *      SFC_ERR_UNSUPPORTED -> std::invalid_argument   (configuration the device path does not cover)
 *      SFC_ERR_CUDA        -> std::runtime_error
 *  - Pointers named d_* are device pointers; `stream` is a cudaStream_t
 *    (NULL = legacy default stream).  Device calls are stream-ordered and
 *    asynchronous unless documented as synchronous.
 *  - Tensors are row-major NCHW like sfconv::DenseTensor (tensor.hpp:11-31);
 *    activations and weights are int8 (the integer values the reference
 *    receives as doubles); weights are [OC][IC][R][R] with R the algorithm's
 *    filter size (3 for the three 3x3 algorithms, 5 / 7 for sfc6-6x6-5x5 /
 *    sfc6-4x4-7x7).
 *  - Plans and layers are immutable after creation and may be shared across
 *    host threads; all per-call state lives in the caller's workspace, so
 *    concurrent calls on distinct streams need distinct workspaces.
 */
#ifndef SFC_B200_H
#define SFC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFC_OK 0
#define SFC_ERR_INVALID -1
#define SFC_ERR_DOMAIN -2
#define SFC_ERR_UNSUPPORTED -3
#define SFC_ERR_CUDA -4

/* Scope / search codes, numerically equal to the reference enums (quant.hpp:16-18). */
#define SFC_ACT_PER_TENSOR 0
#define SFC_ACT_PER_FREQUENCY 1
#define SFC_FIL_PER_CHANNEL 0
#define SFC_FIL_PER_FREQUENCY 1
#define SFC_FIL_PER_CHANNEL_FREQUENCY 2
#define SFC_SEARCH_MINMAX 0
#define SFC_SEARCH_MSE_GRID 1

typedef struct sfc_plan* sfc_plan_t;
typedef struct sfc_layer* sfc_layer_t;

const char* sfc_last_error(void);
int sfc_version(void);

/* ---- catalog: replaces catalog_algorithm / catalog_export_json / catalog_hash
 *      (include/sfconv/spec.hpp:76-79, src/catalog.cpp:275-287, 562-601) ----------- */

/* JSON of the five catalogued SFC algorithms (sfc4-4x4-3x3, sfc6-6x6-3x3, sfc6-7x7-3x3,
 * sfc6-6x6-5x5, sfc6-4x4-7x7) in the reference export layout; hash = FNV-1a 64 of it. */
int sfc_catalog_json(char* buf, size_t cap, uint64_t* hash);
/* Derive + exactness-gate + bind the compiled kernels for `name`
 * ("sfc4-4x4-3x3" | "sfc6-6x6-3x3" | "sfc6-7x7-3x3" | "sfc6-6x6-5x5" | "sfc6-4x4-7x7").
 * Every kernel serves all five; the register-resident transform (k_act_row), 24-bit P, the
 * small-channel (Cin <= 4) fused path and the persistent output kernel are 3x3-only fast
 * paths (the 5x5 / 7x7 algorithms take the shared-memory transforms and int32 P). */
int sfc_plan_create(const char* name, sfc_plan_t* out);
int sfc_plan_destroy(sfc_plan_t plan);
/* dims[10] = {K, n_in, M, R, N, offset, a_denom, n_corrections, mults_full, mults_reduced} */
int sfc_plan_dims(sfc_plan_t plan, int64_t* dims);
/* Row-major integer matrices BT[K][n_in], G[K][R], A[K][M] (any pointer may be NULL). */
int sfc_plan_matrices(sfc_plan_t plan, int64_t* bt, int64_t* g, int64_t* a);

/* ---- layer: offline filter stage of quantized_fast_conv2d
 *      (transform_filters src/conv.cpp:352-382 + filter scales/quantize src/quant.cpp:183-229) */

/* Runs U = G f G^T, the filter scales of `filter_scope` found by `search` and exact RNE
 * quantization on `stream` and keeps the quantized transformed filters on the
 * device.  Synchronous (returns once the layer is ready).  bits in [2, 16]; 9-16 bits
 * take the parity path below (operands exceed int8); activation scope PerTensor. */
int sfc_layer_create(sfc_plan_t plan, const int8_t* d_weights, int out_channels, int in_channels, int bits,
                     int filter_scope, int search, void* stream, sfc_layer_t* out);
/* The whole QuantConfig (quant.hpp:27-34): act_scope SFC_ACT_*, filter_scope SFC_FIL_*,
 * search SFC_SEARCH_*.  Anything but {PerTensor, PerChannel, MinMax} selects the parity
 * path: per-frequency dequantisation before the inverse transform in fp64 (quant.cpp:258-278),
 * scale searches in the reference's order; such layers run through sfc_conv_forward only
 * and produce out_f32 / out_f64 / out_i8 (y_int is not defined for them).  bits 9-16 (any
 * scope) keep vq / uq as integer-valued doubles and contract them with an exact fp64
 * batched GEMM (|pacc| <= C * 2^30 < 2^53, so pacc is the reference's int64 exactly). */
int sfc_layer_create_ex(sfc_plan_t plan, const int8_t* d_weights, int out_channels, int in_channels, int bits,
                        int act_scope, int filter_scope, int search, void* stream, sfc_layer_t* out);
int sfc_layer_destroy(sfc_layer_t layer);
/* Host copies of the filter scales sf[OC] (double) and per-oc max|U| (int32); synchronous. */
int sfc_layer_filter_scales(sfc_layer_t layer, double* sf, int32_t* umax);
/* The filter scales as the layer's scope defines them (quant.cpp:193-219): OC (PerChannel),
 * K*K (PerFrequency) or OC*K*K (PerChannelFrequency) doubles; *count receives the number
 * (pass scales = NULL to query it).  Synchronous. */
int sfc_layer_filter_scales_native(sfc_layer_t layer, double* scales, int64_t* count);
/* Filter-side saturation count (0 by construction for MinMax); synchronous. */
int sfc_layer_saturations(sfc_layer_t layer, int64_t* count);
/* Device view of the quantized transformed filters uq[f][oc][ic] with row pitch
 * `*ic_pitch` and plane pitch `*oc_pitch` rows. */
int sfc_layer_uq(sfc_layer_t layer, const int8_t** d_uq, int64_t* ic_pitch, int64_t* oc_pitch);

/* ---- per call: the activation stage, contraction and output stage of
 *      quantized_fast_conv2d (src/quant.cpp:163-181, 239-279) ------------------------- */

/* Bytes of caller-owned device workspace one sfc_conv_int8 call needs. */
int sfc_conv_workspace_size(sfc_layer_t layer, int n, int h, int w, int pad, size_t* bytes);

/* Absmax pre-pass: atomically max-accumulates max|B^T x B| over every tile
 * and channel of x into *d_vmax (caller zero-initialises it).  Multi-GPU
 * callers run this on their batch shard and all-reduce(MAX) d_vmax before
 * sfc_conv_int8, which makes the per-tensor scale global (quant.cpp:171-172). */
int sfc_act_absmax(sfc_layer_t layer, const int8_t* d_x, int n, int h, int w, int pad, int32_t* d_vmax,
                   void* stream);

/* sfc_act_absmax that also keeps the transformed activations V (int16) in the workspace,
 * so sfc_conv_kept quantizes them with one streaming pass instead of recomputing the
 * transform.  Multi-GPU: sfc_act_transform -> all-reduce(MAX) d_vmax -> sfc_conv_kept. */
int sfc_act_transform(sfc_layer_t layer, const int8_t* d_x, int n, int h, int w, int pad, int32_t* d_vmax,
                      void* d_workspace, size_t workspace_bytes, void* stream);

typedef struct {
    int32_t* y_int32;      /* [N][OC][HO][WO] integer output accumulator sum_kl A A pacc, or NULL */
    int64_t* y_int64;      /* same, 64-bit (required when the int32 bound does not hold), or NULL */
    float* out_f32;        /* dequantised output y * sa * sf[oc] / N^2, or NULL */
    double* out_f64;       /* the same in fp64 (what the sfconv:: DenseTensor shim returns), or NULL */
    int8_t* out_i8;        /* harness requant clamp(rint(out * requant_scale), 0, 127), or NULL */
    double requant_scale;
} sfc_outputs;

/* Quantize the transformed activations with the global scale derived from
 * *d_vmax, contract over channels on the tensor cores and apply the output
 * transform.  Asynchronous on `stream`. */
int sfc_conv_int8(sfc_layer_t layer, const int8_t* d_x, int n, int h, int w, int pad, const int32_t* d_vmax,
                  void* d_workspace, size_t workspace_bytes, const sfc_outputs* outs, void* stream);

/* Same as sfc_conv_int8 but launches only the kernels selected by `stage_mask`
 * (profiling / per-kernel timing; stages must still run in order on one stream). */
#define SFC_STAGE_QPARAMS 1u   /* reset the activation saturation counter  */
#define SFC_STAGE_ACT 2u       /* scale + exact quantizer from *d_vmax, input transform, quantize -> vq */
#define SFC_STAGE_GEMM 4u      /* per-frequency int8 contraction -> pacc   */
#define SFC_STAGE_OUTPUT 8u    /* output transform + dequant / requant     */
#define SFC_STAGE_ALL 15u
#define SFC_STAGE_KEPT 16u     /* with SFC_STAGE_ACT: quantize the V kept by sfc_act_transform */
int sfc_conv_int8_stages(sfc_layer_t layer, const int8_t* d_x, int n, int h, int w, int pad, const int32_t* d_vmax,
                         void* d_workspace, size_t workspace_bytes, const sfc_outputs* outs, unsigned stage_mask,
                         void* stream);

/* sfc_conv_int8 after sfc_act_transform on the same workspace and input shape: quantizes
 * the kept V (no input pointer needed), contracts and applies the output transform. */
int sfc_conv_kept(sfc_layer_t layer, int n, int h, int w, int pad, const int32_t* d_vmax, void* d_workspace,
                  size_t workspace_bytes, const sfc_outputs* outs, void* stream);

/* Convenience (single GPU): zero the workspace's vmax slot, sfc_act_transform, sfc_conv_kept. */
int sfc_conv_forward(sfc_layer_t layer, const int8_t* d_x, int n, int h, int w, int pad, void* d_workspace,
                     size_t workspace_bytes, const sfc_outputs* outs, void* stream);

/* Inspection of the last call's workspace (synchronous on `stream`):
 * stats[0..5] = {sa (as double bits), vmax, activation saturations, fast-quantizer-exact flag,
 *                values_quantized, tiles}. */
/* Activation scales of the last call: 1 (PerTensor) or K*K (PerFrequency) doubles in *count;
 * scales may be NULL to query the count.  Synchronous on `stream`. */
int sfc_conv_act_scales(sfc_layer_t layer, int n, int h, int w, int pad, const void* d_workspace,
                        size_t workspace_bytes, double* scales, int64_t* count, void* stream);
int sfc_conv_stats(sfc_layer_t layer, int n, int h, int w, int pad, const void* d_workspace, size_t workspace_bytes,
                   int64_t* stats, void* stream);
/* Device views into the workspace after sfc_conv_int8:
 *   vq   int8  [F][Tpad][Cpad]   quantized transformed activations
 *   pacc                         per-frequency channel contractions in the storage
 *                                sfc_conv_schedule reports as p_layout; NULL when P is
 *                                chunked (opt-in SFC_PCHUNK_MB budget exceeded: each chunk
 *                                is consumed from L2 and never materialised whole)
 * geom[6] = {T, Tpad, Cpad, OCpad, th, tw}. */
int sfc_conv_views(sfc_layer_t layer, int n, int h, int w, int pad, void* d_workspace, size_t workspace_bytes,
                   int8_t** d_vq, int32_t** d_pacc, int64_t* geom);
/* The schedule sfc_conv_forward picks for this layer and geometry (either may be NULL):
 *   *recompute  0: the absmax pass keeps V and the GEMM quantizes it (sfc_act_transform +
 *                  sfc_conv_kept); 1: absmax only, then a quantizing transform writes vq
 *                  (sfc_act_absmax + sfc_conv_int8).  Both are bit-identical.
 *   *p_layout   storage of pacc in the workspace: 0 = int32 [F][Tpad][OCpad]; 1 = 24-bit
 *               [F][Tpad] rows of 3*OCpad bytes (byte planes b0 | b1 | b2, P = b0 + 2^8 b1 +
 *               2^16 b2 with b2 signed; exact as qmax^2 * Cin < 2^23; SFC_P24=0 keeps int32);
 *               2 = the same 24-bit values unit-major for the tensor-core output transform
 *               ([OCpad/32][3 planes][F][Tpad/4][128 B]: 32 channels x 4 tiles per 128-byte
 *               row, 16-byte chunk c of row f at c ^ (f & 7); the default for the 3x3 variants
 *               on grids of >= 2 units per SM, SFC_OUT_MMA=0 keeps layout 1).  Layout 2 holds
 *               P + 2^15 and its plane 2 is sparse: row (f, unit) of plane 2 is written only
 *               when one of its 128 values leaves 16 bits, and a flag byte per (unit, f) --
 *               [OCpad/32][Tpad/32][F][8] at byte offset 3*F*Tpad*OCpad -- says so (unflagged
 *               rows of plane 2 are undefined and stand for zeros; SFC_P2_DENSE=1 writes every
 *               row); 3 = no P:
 *               Cin <= 4 layers contract with dp4a inside the output transform and the vq
 *               view is compact [F][T][4] (SFC_SMALLC=0 keeps the tensor-core GEMM).
 *               sfc_conv_views returns the raw P storage in this layout (the Python
 *               SfcLayer.views() decodes every layout to int32 [F][T][OC]). */
int sfc_conv_schedule(sfc_layer_t layer, int n, int h, int w, int pad, int* recompute, int* p_layout);

/* Exact int8 direct correlation (int32 accumulate), the report baseline
 * of quantized_fast_conv2d (quant.cpp:282) and direct_conv2d (conv.cpp:320-350). */
int sfc_direct_conv_int8(const int8_t* d_x, int n, int c, int h, int w, const int8_t* d_weights, int oc, int r,
                         int stride, int pad, int32_t* d_out, void* stream);

/* Exact per-frequency energy sum_{tiles,channels} V^2 (frequency_energy, quant.cpp:136-150).
 * d_sum[K*K] (uint64, caller zeroes) accumulates; divide by n*th*tw*c on the host. */
int sfc_frequency_energy_int8(sfc_plan_t plan, const int8_t* d_x, int n, int c, int h, int w, int pad,
                              unsigned long long* d_sum, void* stream);

/* U = G f G^T for every (oc, ic) as exact int32 [OC][IC][K][K] (transform_filters, conv.cpp:352-382). */
int sfc_transform_filters_int8(sfc_plan_t plan, const int8_t* d_weights, int oc, int ic, int32_t* d_u,
                               void* stream);

/* U = G f G^T for real-valued fp64 filters in the reference's accumulation order, fp64
 * [OC][IC][K][K] (transform_filters, conv.cpp:352-382, for non-integer filters). */
int sfc_transform_filters_f64(sfc_plan_t plan, const double* d_weights, int oc, int ic, double* d_u,
                              void* stream);

/* Report sums of quantized_fast_conv2d (quant.cpp:283-291) on the device: host_sums[0] =
 * sum (out - ref)^2, host_sums[1] = sum ref^2 over n elements (ref = sfc_direct_conv_int8 output).
 * Synchronous. */
int sfc_report_sq_err(const double* d_out, const int32_t* d_ref, int64_t n, double* host_sums, void* stream);

/* Test hook: run the device activation quantizer for every integer v in [-vmax, vmax]
 * (d_q has 2*vmax+1 int32 slots); info[4] = {fast path exact flag, shift, multiplier,
 * sa as double bits}.  Synchronous. */
int sfc_debug_quantizer(int vmax, int bits, int32_t* d_q, int64_t* info, void* stream);

/* ---- real-valued (fp64) tensors, the reference API's DenseTensor values ---------------- */
/* sfc_layer_create_ex for fp64 filters [OC][IC][R][R]: U = G f G^T in transform_filters'
 * arithmetic order (conv.cpp:352-382), then the QuantConfig's scales and quantization. */
int sfc_layer_create_f64(sfc_plan_t plan, const double* d_weights, int out_channels, int in_channels, int bits,
                         int act_scope, int filter_scope, int search, void* stream, sfc_layer_t* out);
/* sfc_conv_forward for fp64 inputs: V = B^T x B in gather_tiles' order (quant.cpp:44-93),
 * scales, exact quantization, the int8 contraction and the fp64 epilogue (out_f32 / out_f64 /
 * out_i8; no y_int).  Needs a layer from sfc_layer_create_f64 or a non-default
 * sfc_layer_create_ex config.  Temporary V buffer stream-ordered (cudaMallocAsync). */
int sfc_conv_forward_f64(sfc_layer_t layer, const double* d_x, int n, int h, int w, int pad, void* d_workspace,
                         size_t workspace_bytes, const sfc_outputs* outs, void* stream);
/* direct_conv2d (conv.cpp:320-350) in fp64 with the reference's summation order. */
int sfc_direct_conv_f64(const double* d_x, int n, int c, int h, int w, const double* d_weights, int oc, int r,
                        int stride, int pad, double* d_out, void* stream);
/* sfc_report_sq_err against an fp64 reference. */
int sfc_report_sq_err_f64(const double* d_out, const double* d_ref, int64_t n, double* host_sums, void* stream);

/* fast_conv2d (conv.cpp:384-553), the fp64 float path, on the device: V and U in the
 * reference's order, the K^2 per-frequency products as one strided-batched fp64 GEMM,
 * y = A^T P A / N^2.  reduced != 0 is FastConvOptions::reduced_products (conv.cpp:399-403,
 * 466-509): each (triple x triple) block's nine products become six evaluation products
 * folded onto its corners, so the batch shrinks to mults_reduced() slices (88 of 100 for
 * sfc6-6x6-3x3).  d_out [N][OC][HO][WO] fp64.  counters[2] (optional) = {products formed,
 * tiles}.  Temporary buffers are stream-ordered (cudaMallocAsync). */
int sfc_fast_conv_f64(sfc_plan_t plan, const double* d_x, int n, int c, int h, int w, const double* d_weights,
                      int oc, int pad, int reduced, double* d_out, int64_t* counters, void* stream);

/* ---- the general QuantConfig on a batch shard: the full batch's activation
 *      scales from per-shard steps.  Layers from sfc_layer_create_ex with a non-default config
 *      (int8-valued inputs), one workspace per shard.  Sequence per rank:
 *        sfc_general_prepare       absmax keeps V; this shard's activation maxima -> *d_maxima
 *                                  (count = 1 or F uint64: fp64 bit patterns of non-negative
 *                                  values, so an integer all-reduce(MAX) is the exact global max)
 *        all-reduce(MAX) of d_maxima
 *        MseGrid only: sfc_general_mse_partial with d_err_in = the previous rank's d_err_out
 *                                  (NULL on rank 0), sent on to the next rank: the reference's
 *                                  one sequential fp64 sum per candidate (quant.cpp:19-30,
 *                                  168-181) continued shard by shard in batch order; the last
 *                                  rank's sums [count][101] are broadcast to every rank
 *        sfc_general_conv          scales (MinMax from the maxima / the MseGrid pick over d_err),
 *                                  quantize, contraction, fp64 epilogue -> out_f32 / out_f64 / i8
 *      The result equals sfc_conv_forward on the whole batch bit for bit. */
int sfc_general_prepare(sfc_layer_t layer, const int8_t* d_x, int n, int h, int w, int pad, void* d_workspace,
                        size_t workspace_bytes, uint64_t** d_maxima, int* count, void* stream);
int sfc_general_mse_partial(sfc_layer_t layer, int n, int h, int w, int pad, void* d_workspace,
                            size_t workspace_bytes, const double* d_err_in, double* d_err_out, void* stream);
int sfc_general_conv(sfc_layer_t layer, int n, int h, int w, int pad, void* d_workspace, size_t workspace_bytes,
                     const double* d_err, const sfc_outputs* outputs, void* stream);

/* Profiling hook of the timeline build (libsfc_b200_tl.so, `make TIMELINE=1`): out[8][3] =
 * per kernel {first CTA entry, first CTA past its dependency wait, last CTA exit} in
 * %globaltimer ns (0 / UINT64_MAX when the kernel did not run); reset re-arms the stamps.
 * Kernel ids: 0 workspace reset, 1 absmax, 2 quantize, 3 GEMM, 4 output.
 * Synchronous.  Returns SFC_ERR_UNSUPPORTED in the normal build. */
int sfc_debug_timeline(uint64_t* out, int reset);

#ifdef __cplusplus
}
#endif
#endif /* SFC_B200_H */
