// fp32 values as P bf16 pieces: the data format of the parity precision (RALPB_PRECISION_FP32,
// include/ralpb.h).
//
// A value v is carried as pieces p_0 = bf16_rn(v), p_a = bf16_rn(v - p_0 - ... - p_{a-1}).  With
// P = 3 the pieces hold all 24 significand bits: hi + mid + lo == v EXACTLY for every fp32 v (each
// remainder fits the next 8-bit piece), so storage loses nothing against fp32.  (P = 2 keeps 16-17
// bits, |v - p_0 - p_1| <= 2^-17 |v|: too coarse for the 1e-4 parity target on AlexNet, where
// the oracle emulating it drifts 2e-2 of the update from plain fp32 in 3 steps.)
// A tensor is a sequence of G groups of C values stored as [G][P][C] -- per group the C most
// significant pieces, then the next C, ...:
//   activations      group = one pixel of the padded NHWC layout, C = channels (border pixels 0)
//   FC rows          group = one pixel of the HWC-flattened cut (C = channels), or the whole
//                    row of a hidden FC output (G = 1, C = its padded width)
// so a piece tensor IS a bf16 tensor with P*C channels, and every contraction runs unchanged on
// the tcgen05 GEMM engine with the other operand laid out to match:
//   forward       B[(a, n)][(g, b, c)] = w_a[n][g*C + c]   ->  out[m][(a, n)] = (x . w_a)[m][n]
//   backward-data B[(a, n)][(g, b, c)] = w_b[n][g*C + c]   ->  out[m][(g, b, c)] = (dy . w_b)[m][..]
//   weight grad   S[(a, n)][(g, b, c)] = sum_m dy_a[m][n] x_b[m][g*C + c]
// (w_a the pieces of the fp32 master), and a finishing pass sums the pieces (all P*P products of
// the pieces, each exact in fp32, fp32 accumulation -- the BF16x9 emulation of an fp32 GEMM at
// P = 3) before bias / ReLU / mask and the split of the result into the next pieces.  Semantics are
// those of the bf16 path (layers.py:87-123).  Names say "pair" for brevity.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ralpb {

// im2col of fp32 NHWC images for a first (RGB) convolution as a piece matrix: rows = the conv's
// padded output grid [n][ho+2po][wo+2po], each row [P][kpad]: column j = (r*k+s)*c+ch, column
// k*k*c = 1 (bias), zero elsewhere and on border rows.
cudaError_t pair_pack_im2col(const float* x, int n, int h, int w, int c, int k, int st, int p, int ho, int wo, int po,
                             int kpad, __nv_bfloat16* out, int P, cudaStream_t s);

// Convolution operands from the fp32 master w [co][taps][ci]:
//   wf2 [P*co][taps][P*ci]: wf2[(a,o)][t][(b,c)] = piece_a(w[o][t][c])             (forward)
//   wd2 [P*ci][taps][P*co]: wd2[(a,c)][t][(b,o)] = piece_a(w[o][taps-1-t][c])      (backward-data)
// wd2 may be null.
cudaError_t pair_prep_conv(const float* w, int co, int taps, int ci, __nv_bfloat16* wf2, __nv_bfloat16* wd2, int P,
                           cudaStream_t s);
// Matrix operands from the fp32 master w [out][in] (in = G groups of C), rows padded to ld_out:
//   bf [P*ld_out][P*in]: bf[(a,n)][(g,b,c)] = piece_a(w[n][g*C+c])  (forward; zero rows n >= out)
//   bd [P*ld_out][P*in]: bd[(a,n)][(g,b,c)] = piece_b(w[n][g*C+c])  (backward-data; may be null)
cudaError_t pair_prep_mat(const float* w, int out, int ld_out, int groups, int c, __nv_bfloat16* bf,
                          __nv_bfloat16* bd, int P, cudaStream_t s);

// Finish a contraction whose pieces sit side by side: for rows q of a [rows][P*ld] fp32 matrix
// (pieces at columns a*ld + n):
//   v = sum_a acc[q][a*ld + n] (+ bias[n]); relu; times (mask_hi[q][n] > 0) if mask
//   out2 (pieces, row [P][ld]) and/or out_f32 (row stride ld_f32)
// Geometry: rows are `rows`; if border (padded NHWC grid img_rows = hp*wp, wp, pad, h, w) only
// interior rows are written.  mask: a pair tensor with the same row layout (its hi half is used).
struct PairFinish {
  int pieces;
  const float* acc;
  long long rows;
  int n, ld;
  const float* bias;
  int relu;
  const __nv_bfloat16* mask;
  __nv_bfloat16* out2;
  float* out_f32;
  int ld_f32;
  int border, img_rows, wp, pad, h, w;
};
cudaError_t pair_finish(const PairFinish& f, cudaStream_t s);

// Backward-data finish for the (g, b, c) column layout (pieces per group): for rows q, groups g:
//   v = sum_b acc[q][g][b][c]; times (mask_hi > 0) if mask; -> out2[q][g][pieces][c]
// (acc row = groups*P*c fp32, out2 row = groups*P*c bf16).  border as above (rows = pixels, g = 1).
struct PairFinishGroups {
  int pieces;
  const float* acc;
  long long rows;
  int groups, c;
  const __nv_bfloat16* mask;
  __nv_bfloat16* out2;
  int border, img_rows, wp, pad, h, w;
};
cudaError_t pair_finish_groups(const PairFinishGroups& f, cudaStream_t s);

// Max pool on pieces (window k, stride st, no pool padding): x [n][h+2pi][w+2pi][P][c] ->
// y [n][oh+2po][ow+2po][P][c] (interior), first maximum of the carried value in row-major window
// order; idx [n][oh][ow][c] = its window position, 255 where the maximum is not > 0.
cudaError_t pair_maxpool_fwd(const __nv_bfloat16* x, int n, int h, int w, int c, int pi, int k, int st,
                             __nv_bfloat16* y, int po, uint8_t* idx, int P, cudaStream_t s);
// Its backward (gather form, any window / stride): dx[i] = sum of dy over the windows whose
// recorded maximum is i (0 elsewhere: the ReLU mask is in the 255 marks), written as pieces on the
// interior of [n][h+2pi][w+2pi][P][c]; colsum (optional): colsum[ch] += sum of dx (the producing
// conv's bias gradient).
cudaError_t pair_maxpool_bwd(const uint8_t* idx, const __nv_bfloat16* dy, int n, int h, int w, int c, int pi, int k,
                             int st, int po, __nv_bfloat16* dx, float* colsum, int P, cudaStream_t s);

// db[c] += sum over rows of the value carried by a piece tensor with rows [P][ld] (first n columns).
cudaError_t pair_colsum(const __nv_bfloat16* x2, long long rows, int n, int ld, float* db, int P, cudaStream_t s);

// Weight-gradient finish: g[m][t][c] = sum_{a,b} S[(a,m)][t][(b,c)] for m < m_valid, where S is
// fp32 [P*m_rows][t_count][P*c] (the GEMM's [PM] x [T][PC] output); g is [m_valid][t_count][c]
// with row stride (floats) g_ld per m (t_count * c when dense).
cudaError_t pair_reduce_wgrad(const float* S, int m_rows, int m_valid, int t_count, int c, float* g, long long g_ld,
                              int P, cudaStream_t s);

// Softmax cross-entropy on fp32 logits (row stride ld): per-row loss and
// dlogits = (softmax - onehot) * scale as pieces [rows][P][ld] (padding columns untouched).
cudaError_t pair_softmax_xent(const float* logits, int rows, int classes, int ld, const int32_t* labels, float scale,
                              float* row_loss, __nv_bfloat16* dlogits2, int P, cudaStream_t s);

}  // namespace ralpb
