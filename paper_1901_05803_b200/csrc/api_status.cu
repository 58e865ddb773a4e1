#include <string>
#include "../../include/ralpb.h"
#include "elementwise.cuh"
#include "status.cuh"

namespace ralpb {
std::string& last_error_slot() {
  thread_local std::string slot;
  return slot;
}
}  // namespace ralpb

using namespace ralpb;

extern "C" {

const char* ralpb_last_error(void) { return last_error_slot().c_str(); }
int ralpb_version(void) { return 1; }

#define RALPB_S(st) static_cast<cudaStream_t>(st)
#define RALPB_BF(p) reinterpret_cast<__nv_bfloat16*>(p)
#define RALPB_CBF(p) reinterpret_cast<const __nv_bfloat16*>(p)

int ralpb_pack_input(const float* x, int n, int h, int w, int c, void* out, int cp, int pad,
                     void* stream) {
  return set_status(pack_input(x, n, h, w, c, RALPB_BF(out), cp, pad, RALPB_S(stream)), "pack_input");
}
int ralpb_maxpool_fwd(const void* x, int n, int h, int w, int c, int pad_in, int k, int stride,
                      void* y, int pad_out, void* stream) {
  return set_status(maxpool_fwd(RALPB_CBF(x), n, h, w, c, pad_in, k, stride, RALPB_BF(y), pad_out,
                                RALPB_S(stream)), "maxpool_fwd");
}
int ralpb_maxpool_fwd_idx(const void* x, int n, int h, int w, int c, int pad_in, int k, int stride, void* y,
                          int pad_out, void* idx, void* stream) {
  return set_status(maxpool_fwd(RALPB_CBF(x), n, h, w, c, pad_in, k, stride, RALPB_BF(y), pad_out, RALPB_S(stream),
                                static_cast<uint8_t*>(idx)),
                    "maxpool_fwd_idx");
}
int ralpb_maxpool_bwd_gather(const void* idx, const void* dy, int n, int h, int w, int c, int pad_in, int k,
                             int stride, int pad_out, void* dx, float* colsum, void* stream) {
  return set_status(maxpool_bwd_gather(static_cast<const uint8_t*>(idx), RALPB_CBF(dy), n, h, w, c, pad_in, k, stride,
                                       pad_out, RALPB_BF(dx), colsum, RALPB_S(stream)),
                    "maxpool_bwd_gather");
}
int ralpb_maxpool_bwd(const void* x, const void* dy, int n, int h, int w, int c, int pad_in, int k,
                      int stride, int pad_out, void* dx, float* colsum, void* stream) {
  return set_status(maxpool_bwd(RALPB_CBF(x), RALPB_CBF(dy), n, h, w, c, pad_in, k, stride, pad_out,
                                RALPB_BF(dx), colsum, RALPB_S(stream)), "maxpool_bwd");
}
int ralpb_softmax_xent(const float* logits, int rows, int classes, long long ld,
                       const int32_t* labels, float scale, float* row_loss, void* dlogits,
                       long long ld_d, void* stream) {
  return set_status(softmax_xent(logits, rows, classes, ld, labels, scale, row_loss,
                                 RALPB_BF(dlogits), ld_d, RALPB_S(stream)), "softmax_xent");
}
int ralpb_sgd_momentum(float* p, float* v, const float* g, long long n, float lr, float mu,
                       float gscale, void* stream) {
  return set_status(sgd_momentum(p, v, g, n, lr, mu, gscale, RALPB_S(stream)), "sgd_momentum");
}
int ralpb_colsum_bf16(const void* dy, long long rows, int c, long long ld, float* db, void* stream) {
  return set_status(colsum_bf16(RALPB_CBF(dy), rows, c, ld, db, RALPB_S(stream)), "colsum_bf16");
}
int ralpb_conv_weight_prep(const float* w, int co, int taps, int ci, void* wf, void* wd, void* stream) {
  return set_status(conv_weight_prep(w, co, taps, ci, RALPB_BF(wf), RALPB_BF(wd), RALPB_S(stream)),
                    "conv_weight_prep");
}
int ralpb_cast_bf16(const float* x, long long n, void* y, void* stream) {
  return set_status(cast_bf16(x, n, RALPB_BF(y), RALPB_S(stream)), "cast_bf16");
}

}  // extern "C"

extern "C" int ralpb_pack_im2col(const float* x, int n, int h, int w, int c, int k, int stride, int pad, int ho,
                                 int wo, int po, int kpad, void* out, void* stream) {
  return set_status(pack_im2col(x, n, h, w, c, k, stride, pad, ho, wo, po, kpad, RALPB_BF(out), RALPB_S(stream)),
                    "pack_im2col");
}
