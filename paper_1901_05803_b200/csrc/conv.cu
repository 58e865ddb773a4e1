#include <algorithm>
#include <cstdlib>
#include <cstring>
#include "conv.cuh"
#include "elementwise.cuh"

namespace ralpb {

static bool check_geom(const ConvGeom& g, std::string* why) {
  if (g.k != 2 * g.pad + 1) { *why = "implicit conv needs a stride-1 'same' filter (k == 2*pad+1)"; return false; }
  if (g.taps() > kMaxTaps) { *why = "filter too large"; return false; }
  if (g.cin % 16 != 0 || g.cout % 16 != 0) { *why = "channels must be multiples of 16"; return false; }
  if (g.q() >= (1LL << 31)) { *why = "activation too large for 32-bit row coordinates"; return false; }
  return true;
}

// K-block of the implicit-GEMM A operand: the widest of 64 / 32 / 16 channels dividing c
static int kb_for(int c) { return c % 64 == 0 ? 64 : (c % 32 == 0 ? 32 : 16); }

static void fill_taps(const ConvGeom& g, GemmDesc* d) {
  d->taps = g.taps();
  for (int r = 0; r < g.k; ++r)
    for (int s = 0; s < g.k; ++s) d->tap_off[r * g.k + s] = (r - g.pad) * g.wp() + (s - g.pad);
}

static void fill_border(const ConvGeom& g, GemmDesc* d) {
  d->border = 1;
  d->img_rows = g.hp() * g.wp();
  d->wp = g.wp();
  d->pad = g.pad;
  d->h = g.h;
  d->w = g.w;
}

cudaError_t conv_fwd_flat(const ConvGeom& g, const void* x_pad, const void* w, const float* bias,
                          void* y_pad, int relu, cudaStream_t s, std::string* why) {
  if (!check_geom(g, why)) return cudaErrorInvalidValue;
  GemmDesc d;
  d.M = static_cast<int>(g.q());
  d.N = g.cout;
  d.kb = kb_for(g.cin);
  d.K = static_cast<long long>(g.taps()) * g.cin;
  d.a_mode = LD_K_CONV;
  d.a = Operand2D{x_pad, g.q(), g.cin, g.cin};
  d.cblks = g.cin / d.kb;
  d.b_mode = LD_K;
  d.b = Operand2D{w, g.cout, static_cast<long long>(g.taps()) * g.cin, static_cast<long long>(g.taps()) * g.cin};
  fill_taps(g, &d);
  d.epi = EPI_BF16;
  d.relu = relu;
  d.bias = bias;
  d.out = y_pad;
  d.s_m = g.cout;
  d.s_n = 1;
  fill_border(g, &d);
  return gemm_launch(d, s, why);
}

cudaError_t conv_dgrad_flat(const ConvGeom& g, const void* dy_pad, const void* wd, const void* mask_pad,
                            void* dx_pad, cudaStream_t s, std::string* why) {
  if (!check_geom(g, why)) return cudaErrorInvalidValue;
  GemmDesc d;
  d.M = static_cast<int>(g.q());
  d.N = g.cin;
  d.kb = kb_for(g.cout);
  d.K = static_cast<long long>(g.taps()) * g.cout;
  d.a_mode = LD_K_CONV;
  d.a = Operand2D{dy_pad, g.q(), g.cout, g.cout};
  d.cblks = g.cout / d.kb;
  d.b_mode = LD_K;
  d.b = Operand2D{wd, g.cin, static_cast<long long>(g.taps()) * g.cout, static_cast<long long>(g.taps()) * g.cout};
  fill_taps(g, &d);
  d.epi = EPI_BF16;
  d.mask = mask_pad;
  d.mask_s = g.cin;
  d.out = dx_pad;
  d.s_m = g.cin;
  d.s_n = 1;
  fill_border(g, &d);
  return gemm_launch(d, s, why);
}

cudaError_t conv_wgrad_flat(const ConvGeom& g, const void* x_pad, const void* dy_pad, float* dw,
                            cudaStream_t s, std::string* why) {
  if (!check_geom(g, why)) return cudaErrorInvalidValue;
  GemmDesc d;
  d.M = g.taps() * g.cin;
  d.N = g.cout;
  d.K = g.q();
  d.a_mode = LD_MN_CONV;
  d.a = Operand2D{x_pad, g.q(), g.cin, g.cin};
  d.a_cin = g.cin;
  d.b_mode = LD_MN;
  d.b = Operand2D{dy_pad, g.q(), g.cout, g.cout};
  fill_taps(g, &d);
  d.block_n = g.cout >= 256 ? 256 : (g.cout >= 128 ? 128 : (g.cout >= 64 ? 64 : 32));
  d.k_splits = 0;
  d.epi = EPI_F32_ATOMIC;
  d.out = dw;
  d.s_m = 1;
  d.s_n = static_cast<long long>(g.taps()) * g.cin;
  return gemm_launch(d, s, why);
}

// Kernel family per call: RALPB_CONV=slab|flat forces one (A/B comparisons); the default
// uses the slab kernels wherever they apply (they win at every VGG-16 shape once the MMA
// issue loop uses compile-time descriptor offsets; tools/probe_conv.py).
enum class Family { kAuto, kSlab, kFlat };
static Family family() {
  const char* e = getenv("RALPB_CONV");
  if (e != nullptr && std::strcmp(e, "flat") == 0) return Family::kFlat;
  if (e != nullptr && std::strcmp(e, "slab") == 0) return Family::kSlab;
  return Family::kAuto;
}
static bool pick_slab(bool eligible, bool auto_choice) {
  if (!eligible) return false;
  switch (family()) {
    case Family::kFlat: return false;
    case Family::kSlab: return true;
    default: return auto_choice;
  }
}

cudaError_t conv_fwd(const ConvGeom& g, const void* x_pad, const void* w, const float* bias, void* y_pad,
                     int relu, cudaStream_t s, std::string* why) {
  if (pick_slab(slab_fwd_ok(g, g.cin, g.cout), true))
    return conv_slab_fwd(g, x_pad, w, g.cin, g.cout, bias, relu, nullptr, y_pad, nullptr, s, why);
  return conv_fwd_flat(g, x_pad, w, bias, y_pad, relu, s, why);
}

bool conv_fwd_pool_ok(const ConvGeom& g) {
  return pick_slab(slab_fwd_ok(g, g.cin, g.cout), true) && g.h % 2 == 0 && g.w % 2 == 0;
}

cudaError_t conv_fwd_pool(const ConvGeom& g, const void* x_pad, const void* w, const float* bias, void* y_pad,
                          int relu, void* pool_out, int pool_pad, cudaStream_t s, std::string* why, void* pool_idx) {
  if (!conv_fwd_pool_ok(g)) { *why = "conv_fwd_pool: shape not supported by the slab kernels"; return cudaErrorInvalidValue; }
  return conv_slab_fwd(g, x_pad, w, g.cin, g.cout, bias, relu, nullptr, y_pad, nullptr, s, why, pool_out, pool_pad,
                       pool_idx);
}

cudaError_t conv_dgrad(const ConvGeom& g, const void* dy_pad, const void* wd, const void* mask_pad,
                       void* dx_pad, float* colsum, cudaStream_t s, std::string* why) {
  if (pick_slab(slab_fwd_ok(g, g.cout, g.cin), true))
    return conv_slab_fwd(g, dy_pad, wd, g.cout, g.cin, nullptr, 0, mask_pad, dx_pad, colsum, s, why);
  cudaError_t e = conv_dgrad_flat(g, dy_pad, wd, mask_pad, dx_pad, s, why);
  if (e != cudaSuccess || colsum == nullptr) return e;
  return colsum_bf16(static_cast<const __nv_bfloat16*>(dx_pad), g.q(), g.cin, g.cin, colsum, s);
}

cudaError_t conv_wgrad(const ConvGeom& g, const void* x_pad, const void* dy_pad, float* dw, float* db,
                       cudaStream_t s, std::string* why) {
  if (pick_slab(slab_wgrad_ok(g), true)) return conv_slab_wgrad(g, x_pad, dy_pad, dw, db, s, why);
  cudaError_t e = conv_wgrad_flat(g, x_pad, dy_pad, dw, s, why);
  if (e != cudaSuccess || db == nullptr) return e;
  return colsum_bf16(static_cast<const __nv_bfloat16*>(dy_pad), g.q(), g.cout, g.cout, db, s);
}

}  // namespace ralpb
