// HBM-bound kernels of the step: input packing, max-pool fwd/bwd, softmax
// cross-entropy, SGD-momentum, bias-gradient column sums, weight re-layouts.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ralpb {

// fp32 NHWC [n][h][w][c] -> bf16 [n][h+2p][w+2p][cp] (zero border, zero channels c..cp).
cudaError_t pack_input(const float* x, int n, int h, int w, int c, __nv_bfloat16* out, int cp,
                       int pad, cudaStream_t s);

// im2col of an fp32 NHWC image batch for the first convolution (k x k, stride st, pad p):
// out[(img, oy+po, ox+po)][j] for the padded output grid [n][ho+2po][wo+2po][kpad], with
// j = (r*k + s)*c + ch the filter tap, column k*k*c = 1 (bias folded into the GEMM) and zeros
// elsewhere (incl. every border row).
cudaError_t pack_im2col(const float* x, int n, int h, int w, int c, int k, int st, int p, int ho, int wo,
                        int po, int kpad, __nv_bfloat16* out, cudaStream_t s);

// out[r][c] = act(sum_p parts[p][r*ld + c] + bias[c]) -> bf16 (out_bf16) or fp32 (out_f32),
// row stride ld_out; the reduction of row-/column-parallel partial results (RALP_MPS).
struct PartialSum {
  const float* part[8];
  int n;
};
cudaError_t sum_partials(const PartialSum& ps, int rows, int cols, long long ld, const float* bias, int relu,
                         __nv_bfloat16* out_bf16, float* out_f32, long long ld_out, cudaStream_t s);

// Max pool, window k, stride st (no pool padding).  x: [n][h+2pi][w+2pi][c]; y:
// [n][oh+2po][ow+2po][c] with zero border.  Ties resolve to the first maximum
// in row-major window order.  idx (optional, [n][oh][ow][c] uint8): window position of the
// first max, 255 where it is not > 0 (input of maxpool_bwd_gather).
cudaError_t maxpool_fwd(const __nv_bfloat16* x, int n, int h, int w, int c, int pad_in, int k,
                        int st, __nv_bfloat16* y, int pad_out, cudaStream_t s, uint8_t* idx = nullptr);
// dx[i] = sum over windows containing i where i is the (first) argmax: dy[window],
// then times (x[i] > 0) (the ReLU of the producing conv).  dx has x's padded layout,
// border written as zero.  colsum (optional, c <= 1024): colsum[ch] += sum of the stored dx
// maxpool_bwd_idx: the same for a 2x2/2 pool from the argmax bytes of the fused conv+pool
// forward (idx [n][oh][ow][c], 255 = no gradient); dy [n][oh+2po][ow+2po][c], dx interior.
cudaError_t maxpool_bwd_idx(const uint8_t* idx, const __nv_bfloat16* dy, int n, int oh, int ow, int c, int pad_out,
                            int pad_in, __nv_bfloat16* dx, float* colsum, cudaStream_t s);
// Any k/stride (overlapping windows): gather from the argmax bytes of maxpool_fwd(..., idx)
// (idx [n][oh][ow][c]: window position ky*k+kx of the first max, 255 = max not > 0).
cudaError_t maxpool_bwd_gather(const uint8_t* idx, const __nv_bfloat16* dy, int n, int h, int w, int c, int pad_in,
                               int k, int st, int pad_out, __nv_bfloat16* dx, float* colsum, cudaStream_t s);
// (the producing conv's bias gradient).
cudaError_t maxpool_bwd(const __nv_bfloat16* x, const __nv_bfloat16* dy, int n, int h, int w,
                        int c, int pad_in, int k, int st, int pad_out, __nv_bfloat16* dx, float* colsum,
                        cudaStream_t s);

// Softmax cross-entropy over rows of fp32 logits (row stride ld).  Writes per-row
// loss (natural log) to row_loss and dlogits = (softmax - onehot) * scale as bf16
// (row stride ld_d).
cudaError_t softmax_xent(const float* logits, int rows, int classes, long long ld,
                         const int32_t* labels, float scale, float* row_loss,
                         __nv_bfloat16* dlogits, long long ld_d, cudaStream_t s);
// out[0] = scale * sum(x[0..n)) (single block, deterministic).
cudaError_t reduce_sum(const float* x, int n, float scale, float* out, cudaStream_t s);

// v = mu*v + gscale*g ; p -= lr*v  (PyTorch SGD-momentum form, no dampening/decay).
cudaError_t sgd_momentum(float* p, float* v, const float* g, long long n, float lr, float mu,
                         float gscale, cudaStream_t s);
// Same, also writing bf16(p) to `out` (may be null).
cudaError_t sgd_momentum_bf16(float* p, float* v, const float* g, long long n, float lr, float mu,
                              float gscale, __nv_bfloat16* out, cudaStream_t s);

// db[c] += sum_r dy[r][c]   (bf16 input, fp32 atomics into db).
cudaError_t colsum_bf16(const __nv_bfloat16* dy, long long rows, int c, long long ld, float* db,
                        cudaStream_t s);

// Conv weights fp32 [co][t][ci] -> bf16 forward copy [co][t][ci] and bf16
// backward-data copy [ci][taps-1-t][co].  wd may be null.
struct WeightPrepJob {
  const float* w;
  __nv_bfloat16* wf;
  __nv_bfloat16* wd;     // may be null
  int co, taps, ci;
  int tiles_co, tiles_ci;   // filled by conv_weight_prep_batch
  long long block0;
};
constexpr int kMaxPrepJobs = 24;
struct WeightPrepBatch {
  WeightPrepJob job[kMaxPrepJobs];
  int n;
  long long total_blocks;
};
// conv_weight_prep for several layers in one launch.
cudaError_t conv_weight_prep_batch(const WeightPrepJob* jobs, int n, cudaStream_t s);
cudaError_t conv_weight_prep(const float* w, int co, int taps, int ci, __nv_bfloat16* wf,
                             __nv_bfloat16* wd, cudaStream_t s);
// out = act(acc + bias) [* (mask > 0)] -> bf16 (out_bf16) and/or fp32 (out_f32); finishes a
// split-K GEMM whose fp32 partial sums were accumulated atomically into `acc`.
cudaError_t gemm_finalize(const float* acc, int rows, int cols, long long ld_acc, const float* bias, int relu,
                          const __nv_bfloat16* mask, long long ld_mask, __nv_bfloat16* out_bf16, float* out_f32,
                          long long ld_out, cudaStream_t s);
// fp32 -> bf16 cast.
cudaError_t cast_bf16(const float* x, long long n, __nv_bfloat16* y, cudaStream_t s);
// Several fp32 -> bf16 casts in one launch (x and y 16-byte / 8-byte aligned: parameter offsets are
// multiples of 4 floats), up to kMaxCastJobs per launch.
struct CastJob {
  const float* x;
  __nv_bfloat16* y;
  long long n;
};
constexpr int kMaxCastJobs = 64;
cudaError_t cast_bf16_batch(const CastJob* jobs, int n, cudaStream_t s);

}  // namespace ralpb
