/* TEST INFRASTRUCTURE ONLY -- the CPU oracle for the quantized SFC 3x3 path.
 *
 * A plain-C restatement of the reference's quantized fast convolution
 * (proj/src/quant.cpp:44-293 with transform_filters, proj/src/conv.cpp:352-382,
 * and direct_conv2d, conv.cpp:320-350) that additionally exposes the integer
 * intermediates the reference keeps private: the quantized transformed
 * activations vq, the quantized transformed filters uq, the per-frequency
 * integer contractions pacc and the integer output accumulator
 * y_int = A^T pacc A.  Floating-point work is done in the reference's exact
 * fp64 operation order so its `out` is bitwise equal to the reference's
 * QuantReport::output (pinned in tests/test_oracle.py against oracle/_ref).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may load
 * this library.  The product (paper_2407_02913_b200) never does.
 */
#ifndef SFC_ORACLE_H
#define SFC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dims[10] = {K, n_in, M, R, N, offset, a_denom, n_corrections, mults_full, mults_reduced}.
 * Matrices are row-major int64: BT[K][n_in], G[K][R], A[K][M]. */
int sfo_spec(const char* name, int64_t* dims, int64_t* bt, int64_t* g, int64_t* a);

int64_t sfo_quantize_value(double v, double scale, int bits, int64_t* saturated);
double sfo_scale_minmax(const double* v, int64_t n, int bits);
double sfo_scale_mse_grid(const double* v, int64_t n, int bits);

/* Scope / search codes follow the reference enums (quant.hpp:16-18). */
enum { SFO_ACT_PER_TENSOR = 0, SFO_ACT_PER_FREQUENCY = 1 };
enum { SFO_FIL_PER_CHANNEL = 0, SFO_FIL_PER_FREQUENCY = 1, SFO_FIL_PER_CHANNEL_FREQUENCY = 2 };
enum { SFO_SEARCH_MINMAX = 0, SFO_SEARCH_MSE_GRID = 1 };

typedef struct {
    int bits, act_scope, filter_scope, search;
    int threads;      /* worker threads for the tile loop (results are thread-count independent) */
    int want_report;  /* 1: run the fp64 direct conv for mse / signal_energy / snr_db */
    int64_t vmax_override; /* >= 0: use this max|V| for the PerTensor MinMax scale instead of the
                              local one (a batch shard quantized with the global batch scale) */
    const double* act_scale_override; /* non-NULL: the activation scales (1 or F) to quantize with,
                                         any scope / search (a shard with the full batch's scales) */
} sfo_config;

typedef struct {
    double mse, signal_energy, snr_db;
    int64_t saturations, values_quantized;
    int64_t vmax;      /* max |V| over the whole batch (PerTensor) */
    int64_t tiles;     /* T = B * th * tw */
    int th, tw, HO, WO;
} sfo_report;

/* Quantized SFC convolution on int8-valued inputs (the values the reference
 * receives as doubles).  x: [B][C][H][W], w: [OC][C][R][R] (R = 3).
 * Optional outputs (pass NULL to skip):
 *   out    double  [B][OC][HO][WO]  bitwise equal to the reference output
 *   y_int  int64   [B][OC][HO][WO]  sum_kl A[k,t1] A[l,t2] pacc[k,l]
 *   pacc   int64   [T][OC][K*K]
 *   vq     int32   [T][C][K*K]
 *   uq     int32   [OC][C][K*K]
 *   act_scale double [1 or K*K], fil_scale double [OC | K*K | OC*K*K]
 * Returns 0, or -1 for invalid arguments (message via sfo_last_error). */
int sfo_quantized_conv(const int8_t* x, int B, int C, int H, int W, const int8_t* w, int OC,
                       const char* spec, int pad, const sfo_config* cfg, double* out,
                       int64_t* y_int, int64_t* pacc, int32_t* vq, int32_t* uq,
                       double* act_scale, double* fil_scale, sfo_report* rep);

/* Same pipeline, but only the fp64 direct conv (proj/src/conv.cpp:320-350). */
int sfo_direct_conv(const int8_t* x, int B, int C, int H, int W, const int8_t* w, int OC, int R,
                    int pad, int threads, double* out);

/* Exact integer single-tile execution (catalog.cpp:324-381) and the
 * exhaustive exactness identity sum_k A[k,t] BT[k,i] G[k,j] == a_denom [i == t + j]. */
int sfo_execute_tile(const char* spec, const int64_t* x, const int64_t* f, int64_t* y);
int sfo_check_identity(const char* spec);

const char* sfo_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
