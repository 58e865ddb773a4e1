// C-ABI entry points for the individual step kernels (used by the parity tests
// and by the executor's unit checks).  All pointers are device pointers; all
// calls are asynchronous on `stream` (a cudaStream_t, or NULL for the legacy
// default stream).  Return 0 on success, nonzero on error (see ralpb_last_error).
#include <string>
#include "../../include/ralpb.h"
#include "conv.cuh"
#include "elementwise.cuh"
#include "status.cuh"

using namespace ralpb;

extern "C" {

int ralpb_gemm_bf16(const void* a, long long a_rows, long long a_cols, long long a_ld, int a_mn,
                    const void* b, long long b_rows, long long b_cols, long long b_ld, int b_mn,
                    int M, int N, long long K, void* out, int out_kind, long long s_m,
                    long long s_n, const float* bias, int relu, const void* mask, long long mask_s,
                    int k_splits, int block_n, void* stream) {
  GemmDesc d;
  d.M = M;
  d.N = N;
  d.K = K;
  d.a_mode = a_mn ? LD_MN : LD_K;
  d.b_mode = b_mn ? LD_MN : LD_K;
  d.a = Operand2D{a, a_rows, a_cols, a_ld};
  d.b = Operand2D{b, b_rows, b_cols, b_ld};
  // narrow K-major contractions use a 32/16-wide k-block (64B/32B swizzle) instead of
  // zero-filling a 64-wide one
  d.kb = (!a_mn && !b_mn && K <= 16) ? 16 : (!a_mn && !b_mn && K <= 32) ? 32 : 64;
  d.block_n = block_n;
  d.k_splits = k_splits;
  d.epi = out_kind;
  d.out = out;
  d.s_m = s_m;
  d.s_n = s_n;
  d.bias = bias;
  d.relu = relu;
  d.mask = mask;
  d.mask_s = mask_s;
  std::string why;
  return set_status(gemm_launch(d, static_cast<cudaStream_t>(stream), &why), why);
}

int ralpb_conv_fwd(const void* x_pad, const void* w, const float* bias, void* y_pad, int n, int h,
                   int w_, int cin, int cout, int k, int pad, int relu, void* stream) {
  std::string why;
  ConvGeom g{n, h, w_, cin, cout, k, pad};
  return set_status(conv_fwd(g, x_pad, w, bias, y_pad, relu, static_cast<cudaStream_t>(stream), &why), why);
}

int ralpb_conv_fwd_pool(const void* x_pad, const void* w, const float* bias, void* y_pad, void* pool_out,
                        int pool_pad, void* pool_idx, int n, int h, int w_, int cin, int cout, int k, int pad,
                        int relu, void* stream) {
  std::string why;
  ConvGeom g{n, h, w_, cin, cout, k, pad};
  return set_status(conv_fwd_pool(g, x_pad, w, bias, y_pad, relu, pool_out, pool_pad,
                                  static_cast<cudaStream_t>(stream), &why, pool_idx), why);
}

int ralpb_maxpool_bwd_idx(const void* idx, const void* dy, int n, int oh, int ow, int c, int pad_out, int pad_in,
                          void* dx, float* colsum, void* stream) {
  return set_status(maxpool_bwd_idx(static_cast<const uint8_t*>(idx), static_cast<const __nv_bfloat16*>(dy), n, oh,
                                    ow, c, pad_out, pad_in, static_cast<__nv_bfloat16*>(dx), colsum,
                                    static_cast<cudaStream_t>(stream)),
                    "maxpool_bwd_idx");
}

int ralpb_conv_dgrad(const void* dy_pad, const void* wd, const void* mask_pad, void* dx_pad, float* colsum,
                     int n, int h, int w_, int cin, int cout, int k, int pad, void* stream) {
  std::string why;
  ConvGeom g{n, h, w_, cin, cout, k, pad};
  return set_status(conv_dgrad(g, dy_pad, wd, mask_pad, dx_pad, colsum, static_cast<cudaStream_t>(stream), &why),
                    why);
}

int ralpb_conv_first_fwd(const float* img, int n, int h, int w, const void* wf, void* y_pad, int pad_out,
                         void* stream) {
  std::string why;
  if (!conv_first_ok(h, w, 3, 64, 3, 1, 1)) return set_status(cudaErrorInvalidValue, "conv_first: unsupported shape");
  return set_status(conv_first_fwd(img, n, h, w, 3, wf, y_pad, pad_out, static_cast<cudaStream_t>(stream), &why), why);
}

int ralpb_conv_first_wgrad(const float* img, int n, int h, int w, const void* dy_pad, int pad_out, float* dw,
                           void* stream) {
  std::string why;
  if (!conv_first_ok(h, w, 3, 64, 3, 1, 1)) return set_status(cudaErrorInvalidValue, "conv_first: unsupported shape");
  return set_status(conv_first_wgrad(img, n, h, w, 3, dy_pad, pad_out, dw, static_cast<cudaStream_t>(stream), &why),
                    why);
}

int ralpb_conv_wgrad(const void* x_pad, const void* dy_pad, float* dw, float* db, int n, int h, int w_,
                     int cin, int cout, int k, int pad, void* stream) {
  std::string why;
  ConvGeom g{n, h, w_, cin, cout, k, pad};
  return set_status(conv_wgrad(g, x_pad, dy_pad, dw, db, static_cast<cudaStream_t>(stream), &why), why);
}

}  // extern "C"
