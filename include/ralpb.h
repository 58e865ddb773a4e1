/*
 * ralpb.h — C ABI of libralpb200.so, the B200-native execution backend for the
 * resource-aware layer-placement (RALP) training step of arXiv 1901.05803.
 *
 * The reference (`ralp`, pkg/src/ralp) has no FFI: its drop-in surface is the
 * Python package API (pkg/src/ralp/__init__.py:3-91).  The execution entry it
 * offers is `simulate_run(Scenario) -> SimReport` (pkg/src/ralp/simulator.py:743-770),
 * whose per-job schedule is `_JobRun._ralp_worker/_ralp_ps`
 * (simulator.py:669-715) and `_baseline_worker/_baseline_ps` (simulator.py:637-665).
 * This library executes that schedule for real; the Python package
 * `paper_1901_05803_b200` binds it with ctypes.
 *
 * Conventions: every function returns 0 on success and a nonzero code on
 * failure; ralpb_last_error() returns a thread-local message.  Pointers are
 * device pointers unless a parameter name says `host_`.  `stream` is a
 * cudaStream_t (NULL = legacy default stream).  No torch types cross the ABI.
 */
#ifndef RALPB_H_
#define RALPB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status */
const char* ralpb_last_error(void);
int ralpb_version(void);

/* ------------------------------------------------------------ kernels
 * Dense contraction on tcgen05 tensor cores (bf16 operands, fp32 accumulate).
 *   out[m*s_m + n*s_n] = epi( sum_k A[m,k] * B[n,k] )
 * A is [a_rows][a_cols] row-major with leading dim a_ld; a_mn=0 means rows=M, cols=K
 * (K-major), a_mn=1 means rows=K, cols=M (MN-major).  Same for B with N.
 * out_kind: 0 = bf16 store, 1 = fp32 store, 2 = fp32 atomic add (allows k_splits).
 * bias (fp32, per n) and relu apply before the store; mask (bf16, mask[m*mask_s+n] > 0)
 * multiplies by the ReLU derivative.  k_splits=0 picks a split for the atomic epilogue;
 * block_n=0 picks the N tile.  Replaces the FC forward/backward compute the
 * reference models as `back_batch_s` (simulator.py:542) and infer_fc (layers.py:117-123). */
int ralpb_gemm_bf16(const void* a, long long a_rows, long long a_cols, long long a_ld, int a_mn,
                    const void* b, long long b_rows, long long b_cols, long long b_ld, int b_mn,
                    int M, int N, long long K, void* out, int out_kind, long long s_m,
                    long long s_n, const float* bias, int relu, const void* mask, long long mask_s,
                    int k_splits, int block_n, void* stream);

/* Implicit-GEMM convolution (stride 1, k = 2*pad+1) over the padded NHWC layout
 * [n][h+2pad][w+2pad][c] bf16 with zero borders.  Implements infer_conv
 * (layers.py:87-103) with ReLU fused.
 *   w:  [cout][k*k][cin] bf16      wd: [cin][k*k][cout] bf16 (tap-reversed transpose)
 *   dw: [cout][k*k][cin] fp32, accumulated (caller zeroes). */
int ralpb_conv_fwd(const void* x_pad, const void* w, const float* bias, void* y_pad, int n, int h,
                   int w_, int cin, int cout, int k, int pad, int relu, void* stream);
int ralpb_conv_dgrad(const void* dy_pad, const void* wd, const void* mask_pad, void* dx_pad, int n,
                     int h, int w_, int cin, int cout, int k, int pad, void* stream);
int ralpb_conv_wgrad(const void* x_pad, const void* dy_pad, float* dw, int n, int h, int w_,
                     int cin, int cout, int k, int pad, void* stream);

/* fp32 NHWC images -> bf16 padded NHWC with cp >= c channels (zero fill). */
int ralpb_pack_input(const float* x, int n, int h, int w, int c, void* out, int cp, int pad,
                     void* stream);
/* Max pool (infer_pool, layers.py:106-114; stride defaults to window). */
int ralpb_maxpool_fwd(const void* x, int n, int h, int w, int c, int pad_in, int k, int stride,
                      void* y, int pad_out, void* stream);
int ralpb_maxpool_bwd(const void* x, const void* dy, int n, int h, int w, int c, int pad_in, int k,
                      int stride, int pad_out, void* dx, void* stream);
/* Softmax cross-entropy (the LOSS layer, layers.py:161-163): per-row loss and
 * dlogits = (softmax - onehot) * scale (bf16). */
int ralpb_softmax_xent(const float* logits, int rows, int classes, long long ld,
                       const int32_t* labels, float scale, float* row_loss, void* dlogits,
                       long long ld_d, void* stream);
/* SGD with momentum, PyTorch form: v = mu*v + gscale*g; p -= lr*v. */
int ralpb_sgd_momentum(float* p, float* v, const float* g, long long n, float lr, float mu,
                       float gscale, void* stream);
/* db[c] += sum_r dy[r*ld + c] (bf16 in, fp32 atomics). */
int ralpb_colsum_bf16(const void* dy, long long rows, int c, long long ld, float* db, void* stream);
/* fp32 [co][taps][ci] -> bf16 forward copy and bf16 [ci][taps-1-t][co] dgrad copy (wd may be NULL). */
int ralpb_conv_weight_prep(const float* w, int co, int taps, int ci, void* wf, void* wd, void* stream);
int ralpb_cast_bf16(const float* x, long long n, void* y, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RALPB_H_ */
