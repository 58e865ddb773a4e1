// fp32-accurate (hi, lo) bf16 pairs: the data format of the parity precision
// (RALPB_PRECISION_FP32, include/ralpb.h).
//
// A value v is carried as hi = bf16_rn(v), lo = bf16_rn(v - hi): |v - (hi + lo)| <= 2^-17 |v|
// (hi + lo is exact in fp32).  A tensor is a sequence of G groups of C values stored as
// [G][2][C] -- per group the C hi values, then the C lo values:
//   activations      group = one pixel of the padded NHWC layout, C = channels (border pixels 0)
//   FC rows          group = one pixel of the HWC-flattened cut (C = channels), or the whole
//                    row of a hidden FC output (G = 1, C = its padded width)
// so a pair tensor IS a bf16 tensor with 2C channels, and every contraction runs unchanged on
// the tcgen05 GEMM engine with the other operand laid out to match:
//   forward       B[(a, n)][(g, b, c)] = w_a[n][g*C + c]   ->  out[m][(a, n)] = (x . w_a)[m][n]
//   backward-data B[(a, n)][(g, b, c)] = w_b[n][g*C + c]   ->  out[m][(g, b, c)] = (dy . w_b)[m][..]
//   weight grad   S[(a, n)][(g, b, c)] = sum_m dy_a[m][n] x_b[m][g*C + c]
// (w_0 / w_1 the hi / lo pieces of the fp32 master), and a finishing pass sums the two pieces
// (hi*hi + hi*lo + lo*hi + lo*lo, fp32 accumulation) before bias / ReLU / mask and the split of the
// result into the next pair.  Semantics are those of the bf16 path (layers.py:87-123).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ralpb {

// im2col of fp32 NHWC images for a first (RGB) convolution as a pair matrix: rows = the conv's
// padded output grid [n][ho+2po][wo+2po], each row [2][kpad]: column j = (r*k+s)*c+ch, column
// k*k*c = 1 (bias: hi 1, lo 0), zero elsewhere and on border rows.
cudaError_t pair_pack_im2col(const float* x, int n, int h, int w, int c, int k, int st, int p, int ho, int wo, int po,
                             int kpad, __nv_bfloat16* out, cudaStream_t s);

// Convolution operands from the fp32 master w [co][taps][ci]:
//   wf2 [2co][taps][2ci]: wf2[(a,o)][t][(b,c)] = piece_a(w[o][t][c])             (forward)
//   wd2 [2ci][taps][2co]: wd2[(a,c)][t][(b,o)] = piece_a(w[o][taps-1-t][c])      (backward-data)
// wd2 may be null.
cudaError_t pair_prep_conv(const float* w, int co, int taps, int ci, __nv_bfloat16* wf2, __nv_bfloat16* wd2,
                           cudaStream_t s);
// Matrix operands from the fp32 master w [out][in] (in = G groups of C), rows padded to ld_out:
//   bf [2*ld_out][2*in]: bf[(a,n)][(g,b,c)] = piece_a(w[n][g*C+c])  (forward; zero rows n >= out)
//   bd [2*ld_out][2*in]: bd[(a,n)][(g,b,c)] = piece_b(w[n][g*C+c])  (backward-data; may be null)
cudaError_t pair_prep_mat(const float* w, int out, int ld_out, int groups, int c, __nv_bfloat16* bf,
                          __nv_bfloat16* bd, cudaStream_t s);

// Finish a contraction whose pieces sit side by side: for rows q of a [rows][2*ld] fp32 matrix
// (row stride 2*ld; pieces at columns n and ld + n):
//   v = acc[q][n] + acc[q][ld + n] (+ bias[n]); relu; times (mask_hi[q][n] > 0) if mask
//   out2 (pair, row [2][ld]) and/or out_f32 (row stride ld_f32)
// Geometry: rows are `rows`; if border (padded NHWC grid img_rows = hp*wp, wp, pad, h, w) only
// interior rows are written.  mask: a pair tensor with the same row layout (its hi half is used).
struct PairFinish {
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
//   v = acc[q][g][0][c] + acc[q][g][1][c]; times (mask_hi > 0) if mask; -> out2[q][g][{hi,lo}][c]
// (acc row = groups*2*c fp32, out2 row = groups*2*c bf16).  border as above (rows = pixels, g = 1).
struct PairFinishGroups {
  const float* acc;
  long long rows;
  int groups, c;
  const __nv_bfloat16* mask;
  __nv_bfloat16* out2;
  int border, img_rows, wp, pad, h, w;
};
cudaError_t pair_finish_groups(const PairFinishGroups& f, cudaStream_t s);

// Max pool on pairs (window k, stride st, no pool padding): x [n][h+2pi][w+2pi][2][c] ->
// y [n][oh+2po][ow+2po][2][c] (interior), first maximum of hi+lo in row-major window order;
// idx [n][oh][ow][c] = its window position, 255 where the maximum is not > 0.
cudaError_t pair_maxpool_fwd(const __nv_bfloat16* x, int n, int h, int w, int c, int pi, int k, int st,
                             __nv_bfloat16* y, int po, uint8_t* idx, cudaStream_t s);
// Its backward (gather form, any window / stride): dx[i] = sum of dy over the windows whose
// recorded maximum is i (0 elsewhere: the ReLU mask is in the 255 marks), written as pairs on the
// interior of [n][h+2pi][w+2pi][2][c]; colsum (optional): colsum[ch] += sum of dx (the producing
// conv's bias gradient).
cudaError_t pair_maxpool_bwd(const uint8_t* idx, const __nv_bfloat16* dy, int n, int h, int w, int c, int pi, int k,
                             int st, int po, __nv_bfloat16* dx, float* colsum, cudaStream_t s);

// db[c] += sum over rows of (hi + lo) of a pair tensor with rows [2][ld] (the first n columns).
cudaError_t pair_colsum(const __nv_bfloat16* x2, long long rows, int n, int ld, float* db, cudaStream_t s);

// Weight-gradient finish: g[m][t][c] = sum_{a,b} S[(a,m)][t][(b,c)] for m < m_valid, where S is
// fp32 [2*m_rows][t_count][2*c] (the GEMM's [2M] x [T][2C] output); g is [m_valid][t_count][c]
// with row stride (floats) g_ld per m (t_count * c when dense).
cudaError_t pair_reduce_wgrad(const float* S, int m_rows, int m_valid, int t_count, int c, float* g, long long g_ld,
                              cudaStream_t s);

// Softmax cross-entropy on fp32 logits (row stride ld): per-row loss and
// dlogits = (softmax - onehot) * scale as a pair [rows][2][ld] (padding columns untouched).
cudaError_t pair_softmax_xent(const float* logits, int rows, int classes, int ld, const int32_t* labels, float scale,
                              float* row_loss, __nv_bfloat16* dlogits2, cudaStream_t s);

}  // namespace ralpb
