// Implicit-GEMM convolution over the padded-flattened NHWC layout.
//
// An activation of spatial size HxW with padding p is stored as
// [N][H+2p][W+2p][C] bf16 with zero borders and viewed as a 2-D matrix of
// Q = N*(H+2p)*(W+2p) rows.  For a stride-1 "same" convolution (k = 2p+1)
// output row q (same index space) is
//     y[q] = sum_t x[q + off(t)] * W[t],   off(r,s) = (r-p)*(W+2p) + (s-p)
// so every tap is a plain row-shifted 2-D TMA load of the input matrix; rows
// that fall on padding positions are computed and then zeroed by the epilogue.
// Backward-data is the same GEMM with the tap order reversed and the filter
// transposed; backward-filter contracts over q with both operands MN-major.
// Reference semantics: infer_conv (pkg/src/ralp/layers.py:87-103).
#pragma once
#include "gemm_host.cuh"

namespace ralpb {

struct ConvGeom {
  int n, h, w, cin, cout, k, pad;
  int hp() const { return h + 2 * pad; }
  int wp() const { return w + 2 * pad; }
  long long q() const { return static_cast<long long>(n) * hp() * wp(); }
  int taps() const { return k * k; }
};

// Every conv entry point takes the padded layout; the slab kernels (the default)
// write interior pixels only, so output buffers must be allocated with zero borders
// (the executor zero-initialises every activation/gradient buffer once).
//
// y_pad = relu?(conv(x_pad, w) + bias).  w: [cout][k*k][cin] bf16.
cudaError_t conv_fwd(const ConvGeom& g, const void* x_pad, const void* w, const float* bias,
                     void* y_pad, int relu, cudaStream_t s, std::string* why);
// ... and the 2x2/2 max pool of y written to pool_out ([n][h/2+2pp][w/2+2pp][cout], interior),
// fused into the epilogue (slab kernels; returns an error where they do not apply).
bool conv_fwd_pool_ok(const ConvGeom& g);
// pool_idx (optional, [n][h/2][w/2][cout] uint8): window position of the first max (0..3 row-major),
// 255 where the max is not > 0 -- everything maxpool_bwd_idx needs (no re-read of y).
cudaError_t conv_fwd_pool(const ConvGeom& g, const void* x_pad, const void* w, const float* bias, void* y_pad,
                          int relu, void* pool_out, int pool_pad, cudaStream_t s, std::string* why,
                          void* pool_idx = nullptr);
// dx_pad = conv_transpose(dy_pad, w) * (mask_pad > 0 if mask_pad).
// wd: [cin][k*k][cout] bf16, wd[ci][t][co] = w[co][k*k-1-t][ci].
// colsum (optional): colsum[ci] += sum over pixels of the stored bf16 dx -- the bias gradient of
// the previous convolution, fused into this producer so the wgrad kernel needs no bias pass.
cudaError_t conv_dgrad(const ConvGeom& g, const void* dy_pad, const void* wd, const void* mask_pad,
                       void* dx_pad, float* colsum, cudaStream_t s, std::string* why);
// dw[co][t][ci] += sum_q dy[q][co] * x[q + off(t)][ci];  db[co] += sum_q dy[q][co] if db.
cudaError_t conv_wgrad(const ConvGeom& g, const void* x_pad, const void* dy_pad, float* dw, float* db,
                       cudaStream_t s, std::string* why);

// Padded-flattened single-tap-load variants (write the full padded buffer, zero borders).
cudaError_t conv_fwd_flat(const ConvGeom& g, const void* x_pad, const void* w, const float* bias,
                          void* y_pad, int relu, cudaStream_t s, std::string* why);
cudaError_t conv_dgrad_flat(const ConvGeom& g, const void* dy_pad, const void* wd, const void* mask_pad,
                            void* dx_pad, cudaStream_t s, std::string* why);
cudaError_t conv_wgrad_flat(const ConvGeom& g, const void* x_pad, const void* dy_pad, float* dw,
                            cudaStream_t s, std::string* why);

// Tensor maps (conv_slab.cu): padded activation [n][hp][wp][c] as a 4-D tensor with box
// {bc, bw, bh, 1}, and a row-major [rows][cols] bf16 matrix with box {bc, br}; swz = 32/64/128.
bool encode_act(CUtensorMap* tm, const void* ptr, long long c, long long wp, long long hp, long long n, int bc, int bw,
                int bh, int swz, std::string* why);
bool encode_mat(CUtensorMap* tm, const void* ptr, long long rows, long long cols, int bc, int br, int swz,
                std::string* why);
// Interior view of a padded activation (pixel (pad, pad) onward, clipped at the image edge),
// box {32, bw, bh, 1}, 64-byte swizzle: TMA stores through it never touch the zero borders.
bool encode_interior(CUtensorMap* tm, void* ptr, long long c, long long w, long long h, long long wp, long long hp,
                     long long n, int pad, std::string* why);
bool encode_interior_box(CUtensorMap* tm, void* ptr, long long c, long long w, long long h, long long wp, long long hp,
                         long long n, int pad, int bw, int bh, std::string* why);

// First (RGB) convolution fused with its im2col (conv_first.cu): 3x3/1/pad 1, cin = 3,
// 64 output channels, h % 8 == 0, w % 16 == 0.  img: fp32 NHWC; wf: [64][32] bf16 with the bias
// in column 9*cin; y_pad / dy_pad: [n][h+2p][w+2p][64]; dw: [64][32] fp32 (accumulated).
bool conv_first_ok(int h, int w, int cin, int cout, int k, int stride, int pad);
cudaError_t conv_first_fwd(const float* img, int n, int h, int w, int cin, const void* wf, void* y_pad, int pad_out,
                           cudaStream_t s, std::string* why);
cudaError_t conv_first_wgrad(const float* img, int n, int h, int w, int cin, const void* dy_pad, int pad_out,
                             float* dw, cudaStream_t s, std::string* why);

// Slab-tiled kernels (conv_slab.cu).  `c` = contracted channels, `cout` = produced channels.
bool slab_fwd_ok(const ConvGeom& g, int c, int cout);
double slab_fwd_bytes(const ConvGeom& g, int c, int cout, bool mask, bool pool, bool idx);
double wgrad_bytes(const ConvGeom& g);
bool slab_wgrad_ok(const ConvGeom& g);
// Row-streamed 64 -> 64 channel 3x3 kernel (conv_row.cu), used by conv_slab_fwd when it applies
// (RALPB_ROW64=0 disables).
bool row64_ok(const ConvGeom& g, int c, int cout, const void* pool_idx);
cudaError_t conv_row64_fwd(const ConvGeom& g, const void* x_pad, const void* w, const float* bias, int relu,
                           const void* mask_pad, void* y_pad, float* colsum, void* pool_out, int pool_pad,
                           cudaStream_t s, std::string* why);
cudaError_t conv_slab_fwd(const ConvGeom& g, const void* x_pad, const void* w, int c, int cout, const float* bias,
                          int relu, const void* mask_pad, void* y_pad, float* colsum, cudaStream_t s,
                          std::string* why, void* pool_out = nullptr, int pool_pad = 0, void* pool_idx = nullptr);
cudaError_t conv_slab_wgrad(const ConvGeom& g, const void* x_pad, const void* dy_pad, float* dw, float* db,
                            cudaStream_t s, std::string* why);

}  // namespace ralpb
