// HBM-bound kernels of the branchy model (ResNet-50 bottleneck blocks): training-mode
// batch normalisation over each worker's batch, strided operand layouts for the strided
// convolutions, padded max pool, global average pool.  The contractions themselves run on the
// tcgen05 engine (gemm / slab conv kernels).  Tensors are bf16 NHWC [n][h + 2*pad][w + 2*pad][c];
// every kernel takes each tensor's own padding and touches interior pixels only.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ralpb {

// ld: pixel stride in elements (0 = the tensor's channel count); a channel slice of a wider
// tensor (a branch of a concatenation) has ld = the wide tensor's channels.  Honoured by the
// batch-norm kernels and add_act.
struct Act4 {
  const __nv_bfloat16* p = nullptr;
  int pad = 0;
  int ld = 0;
};
struct MutAct4 {
  __nv_bfloat16* p = nullptr;
  int pad = 0;
  int ld = 0;
};

// Batch statistics over the n*h*w interior pixels: mean[c], rstd[c] = 1/sqrt(var + eps) (biased
// variance, training mode; torch.nn.functional.batch_norm(training=True)).  `work` is the
// kBnWorkFloats scratch (zeroed once at allocation): [2][2048] accumulators the reduction's last
// block finishes and zeroes again, [2][2048] finished sums (backward), a block ticket.
// groups > 1: the n images form `groups` equal consecutive groups, each normalised with its own
// statistics (mean / rstd of group g at + g * stat_stride): per-worker batch statistics for layers
// the PS runs over every worker's gathered rows.
constexpr int kBnWorkFloats = 4 * 2048 + 64;
cudaError_t bn_stats(Act4 x, int n, int h, int w, int c, float eps, float* work, float* mean, float* rstd,
                     cudaStream_t s, int groups = 1, long long stat_stride = 0);

// y = act((x - mean) * rstd * gamma + beta + residual), act = ReLU if relu; residual: none
// (res_kind 0), a raw tensor r (1), or the batch norm of r with its own statistics (2).
struct BnApply {
  Act4 x;
  const float *mean, *rstd, *gamma, *beta;
  int res_kind;
  Act4 r;
  const float *r_mean, *r_rstd, *r_gamma, *r_beta;
  int relu;
  MutAct4 y;
  int n, h, w, c;
  uint8_t* mask_out = nullptr;   // optional (relu): [n*h*w][c/8] bytes, bit j of byte (p, g) = the
                                 // stored y[p][8g + j] > 0 -- the ReLU mask its backward reads
  int groups = 1;                // per-group statistics (see bn_stats)
  long long stat_stride = 0;
};
cudaError_t bn_apply(const BnApply& a, cudaStream_t s);

// Backward of y = act(bn(x) [+ residual]): dz = dy * (y > 0 if relu_mask);  dbeta = sum dz,
// dgamma = sum dz * xhat  (accumulated into dgamma / dbeta);  then
// dx = gamma * rstd * (dz - dbeta / M - xhat * dgamma / M)  (M = n*h*w);  dz_out (optional)
// receives dz itself (the identity shortcut's gradient).  `work` fp32 [2c] scratch.
struct BnBackward {
  Act4 dy;
  Act4 y;            // the forward output (ReLU mask), ignored unless relu_mask
  int relu_mask;
  Act4 x;            // the forward input of the batch norm
  const float *mean, *rstd, *gamma;
  float *dgamma, *dbeta;  // parameter gradients (accumulated)
  MutAct4 dx;
  MutAct4 dz_out;    // optional
  int n, h, w, c;
  const uint8_t* mask_in = nullptr;   // relu_mask from BnApply::mask_out bits instead of reading y
                                      // (1/16 of its bytes, read twice per backward)
  int groups = 1;                     // per-group statistics (see bn_stats); dgamma / dbeta summed
  long long stat_stride = 0;
};
cudaError_t bn_backward(const BnBackward& b, float* work, cudaStream_t s);

// Patch matrix of a padded bf16 activation for a k x k convolution with stride st and padding p
// (reading the zero borders of x, x.pad >= p): out [n*ho*wo][k*k*c], column (r*k + q)*c + ch.
cudaError_t im2col_bf16(Act4 x, int n, int h, int w, int c, int k, int st, int p, int ho, int wo,
                        __nv_bfloat16* out, cudaStream_t s);
// out[n][ho][wo][c] = x[n][st*oy][st*ox][c]  (the 1x1 stride-st projection's input)
cudaError_t subsample(Act4 x, int n, int h, int w, int c, int st, __nv_bfloat16* out, cudaStream_t s);
// y[n][st*oy][st*ox][c] = bf16(y + g[n][oy][ox][c]) (its backward, accumulated into y)
cudaError_t add_strided(const __nv_bfloat16* g, int n, int ho, int wo, int c, int st, MutAct4 y, cudaStream_t s);
// out (interior, zero elsewhere) = dy placed at stride-st positions of the (h x w) grid: the
// stride-1 form of a strided convolution's backward-data input
cudaError_t dilate(const __nv_bfloat16* dy, int n, int ho, int wo, int c, int st, MutAct4 out, int h, int w,
                   cudaStream_t s);
// y = bf16(a + b) elementwise over n*h*w*c (interiors)
cudaError_t add_act(Act4 a, Act4 b, MutAct4 y, int n, int h, int w, int c, cudaStream_t s);

// Max pool with zero padding p (inputs are ReLU outputs >= 0, so a zero border never changes the
// maximum): window k, stride st; idx [n][oh][ow][c] = window position of the first max, 255
// where the max is not > 0.  Backward: gather form.
cudaError_t maxpool_pad_fwd(Act4 x, int n, int h, int w, int c, int k, int st, int p, MutAct4 y, int oh, int ow,
                            uint8_t* idx, cudaStream_t s);
cudaError_t maxpool_pad_bwd(const uint8_t* idx, Act4 dy, int n, int h, int w, int c, int k, int st, int p, int oh,
                            int ow, MutAct4 dx, cudaStream_t s);

// Global average pool: y[n][c] = mean over h*w of x; backward dx = dy / (h*w) broadcast.
cudaError_t avgpool_fwd(Act4 x, int n, int h, int w, int c, __nv_bfloat16* y, cudaStream_t s);
cudaError_t avgpool_bwd(const __nv_bfloat16* dy, int n, int h, int w, int c, MutAct4 dx, cudaStream_t s);

}  // namespace ralpb
