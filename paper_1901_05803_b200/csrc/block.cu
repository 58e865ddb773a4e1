// ResNet bottleneck blocks and the batch-normalised stem convolution on the tcgen05 engine
// (branchy models executed).  Semantics (torchvision v1.5, the geometry behind the
// reference catalog's resnet-50 entries, pkg/tools/build_catalog.py:286-333):
//   a_pre = x Wa^T (1x1);  a = relu(bn_a(a_pre))
//   b_pre = conv3x3(a, Wb, stride s, pad 1);  b = relu(bn_b(b_pre))
//   c_pre = b Wc^T (1x1);  y = relu(bn_c(c_pre) + shortcut),
//   shortcut = x, or bn_d(subsample_s(x) Wd^T) (1x1 projection) on a stage's first block.
// Batch norm uses each worker's batch statistics (training mode, biased variance, eps 1e-5), scale
// and shift are learnable (the catalog's "+2*Cout" parameters).  The 1x1 convolutions are GEMMs over
// the NHWC rows; the stride-1 3x3 is the slab implicit-GEMM kernel (conv_slab.cuh); the stride-2
// 3x3 runs as an im2col GEMM forward / backward-filter, and its backward-data as the stride-1
// kernel over the gradient dilated with zeros.  Storage is bf16 everywhere; every reduction fp32.
#include <algorithm>
#include <cstdlib>
#include "block.cuh"
#include "elementwise.cuh"
#include "gemm_host.cuh"
#include "resnet.cuh"

namespace ralpb {

bool res_epilogue() {
  static const bool on = [] {
    const char* e = getenv("RALPB_RES_EPI");
    return e != nullptr && e[0] == '1';
  }();
  return on;
}

namespace {

constexpr float kBnEps = 1e-5f;

#define RALPB_TRY(expr)                                   \
  do {                                                    \
    cudaError_t _e = (expr);                              \
    if (_e != cudaSuccess) {                              \
      if (why->empty()) *why = std::string(#expr);        \
      *why += std::string(": ") + cudaGetErrorString(_e); \
      return 1;                                           \
    }                                                     \
  } while (0)

// out[rows][n] = a[rows][k] . w[n][k]^T  (bf16 out)
int mm_fwd(Model* m, const bf16* a, long long rows, int k, const bf16* w, int n, bf16* out, std::string* why) {
  GemmDesc d;
  d.M = static_cast<int>(rows); d.N = n; d.K = k;
  d.a = Operand2D{a, rows, k, k};
  d.b = Operand2D{w, n, k, k};
  d.epi = EPI_BF16; d.out = out; d.s_m = n;
  RALPB_TRY(gemm_launch(d, m->stream, why));
  ++m->launches;
  return 0;
}
// out[rows][k] = dy[rows][n] . w[n][k] (+ residual[rows][k]: a gradient summed in the epilogue; may be out)
int mm_dgrad(Model* m, const bf16* dy, long long rows, int n, const bf16* w, int k, bf16* out, std::string* why,
             const bf16* residual = nullptr) {
  GemmDesc d;
  d.M = static_cast<int>(rows); d.N = k; d.K = n;
  d.a_mode = LD_K; d.a = Operand2D{dy, rows, n, n};
  d.b_mode = LD_MN; d.b = Operand2D{w, n, k, k};
  d.epi = EPI_BF16; d.out = out; d.s_m = k;
  d.residual = residual; d.res_s = k;
  RALPB_TRY(gemm_launch(d, m->stream, why));
  ++m->launches;
  return 0;
}
// g[n][k] += dy[rows][n]^T . x[rows][k]  (fp32, split-K atomics; g zeroed by the step)
int mm_wgrad(Model* m, const bf16* dy, long long rows, int n, const bf16* x, int k, float* g, std::string* why) {
  GemmDesc d;
  d.M = n; d.N = k; d.K = rows;
  d.a_mode = LD_MN; d.a = Operand2D{dy, rows, n, n};
  d.b_mode = LD_MN; d.b = Operand2D{x, rows, k, k};
  d.k_splits = 0;
  d.epi = EPI_F32_ATOMIC; d.out = g; d.s_m = k; d.s_n = 1;
  RALPB_TRY(gemm_launch(d, m->stream, why));
  ++m->launches;
  return 0;
}

ConvGeom geom_b(const BlockBufs& k) { return ConvGeom{k.n, k.h, k.w, k.width, k.width, 3, 1}; }

float* mean_of(BlockBufs& k, int which) { return k.stats + static_cast<size_t>(which) * 2 * k.cmax; }
float* rstd_of(BlockBufs& k, int which) { return k.stats + static_cast<size_t>(which) * 2 * k.cmax + k.cmax; }

template <class T>
T* balloc(Model* m, size_t count, std::string* why, bool zero = false) {
  void* p = nullptr;
  if (cudaMalloc(&p, std::max<size_t>(count * sizeof(T), 16)) != cudaSuccess) {
    *why = "cudaMalloc failed (" + std::to_string(count * sizeof(T)) + " bytes)";
    return nullptr;
  }
  if (zero) cudaMemset(p, 0, std::max<size_t>(count * sizeof(T), 16));
  m->owned.push_back(p);
  return static_cast<T*>(p);
}

}  // namespace

int block_alloc(Model* m, BlockBufs& k, std::string* why) {
  const long long rin = static_cast<long long>(k.n) * k.h * k.w;
  const long long rout = static_cast<long long>(k.n) * k.ho * k.wo;
  const long long rpad = static_cast<long long>(k.n) * (k.h + 2) * (k.w + 2);   // the 3x3's padded input grid
  const bool s1 = k.stride == 1;
  k.cmax = std::max(k.width, k.cout);
#define BA(ptr, count, zero) \
  if (!((ptr) = balloc<bf16>(m, static_cast<size_t>(count), why, zero))) return 1
  BA(k.wa, static_cast<long long>(k.width) * k.cin, false);
  BA(k.wbf, 9LL * k.width * k.width, false);
  BA(k.wbd, 9LL * k.width * k.width, false);
  BA(k.wc, static_cast<long long>(k.cout) * k.width, false);
  if (k.down) BA(k.wd, static_cast<long long>(k.cout) * k.cin, false);
  BA(k.a_pre, rin * k.width, false);
  BA(k.a, rpad * k.width, true);                                  // zero borders
  BA(k.b_pre, (s1 ? rpad : rout) * k.width, s1);
  BA(k.b, rout * k.width, false);
  BA(k.c_pre, rout * k.cout, false);
  if (k.down) {
    if (!s1) BA(k.d_in, rout * k.cin, false);
    BA(k.d_pre, rout * k.cout, false);
    BA(k.dd_pre, rout * k.cout, false);
    BA(k.dxs, rout * k.cin, false);
  }
  if (!s1) {
    BA(k.col, rout * 9 * k.width, false);
    BA(k.dil, rpad * k.width, true);
  }
  BA(k.dc_pre, rout * k.cout, false);
  BA(k.dz, rout * k.cout, false);
  BA(k.db, rout * k.width, false);
  BA(k.db_pre, (s1 ? rpad : rout) * k.width, s1);
  BA(k.da, rpad * k.width, true);
  BA(k.da_pre, rin * k.width, false);
#undef BA
  if (!(k.stats = balloc<float>(m, 8 * static_cast<size_t>(k.cmax) * k.groups, why, true))) return 1;
  if (!(k.ma = balloc<uint8_t>(m, static_cast<size_t>(rin) * k.width / 8, why)) ||
      !(k.mb = balloc<uint8_t>(m, static_cast<size_t>(rout) * k.width / 8, why)) ||
      !(k.mc = balloc<uint8_t>(m, static_cast<size_t>(rout) * k.cout / 8, why)))
    return 1;
  return 0;
}

int block_prep(Model* m, BlockBufs& k, cudaStream_t s, std::string* why, std::vector<CastJob>* casts,
               std::vector<WeightPrepJob>* preps) {
  if (casts != nullptr && preps != nullptr) {
    casts->push_back(CastJob{m->P + k.wa_off, k.wa, static_cast<long long>(k.width) * k.cin});
    casts->push_back(CastJob{m->P + k.wc_off, k.wc, static_cast<long long>(k.cout) * k.width});
    if (k.down) casts->push_back(CastJob{m->P + k.wd_off, k.wd, static_cast<long long>(k.cout) * k.cin});
    WeightPrepJob j{};
    j.w = m->P + k.wb_off; j.wf = k.wbf; j.wd = k.wbd; j.co = k.width; j.taps = 9; j.ci = k.width;
    preps->push_back(j);
    return 0;
  }
  RALPB_TRY(cast_bf16(m->P + k.wa_off, static_cast<long long>(k.width) * k.cin, k.wa, s));
  RALPB_TRY(conv_weight_prep(m->P + k.wb_off, k.width, 9, k.width, k.wbf, k.wbd, s));
  RALPB_TRY(cast_bf16(m->P + k.wc_off, static_cast<long long>(k.cout) * k.width, k.wc, s));
  if (k.down) RALPB_TRY(cast_bf16(m->P + k.wd_off, static_cast<long long>(k.cout) * k.cin, k.wd, s));
  m->launches += k.down ? 4 : 3;
  return 0;
}

int block_forward(Model* m, BlockBufs& k, const bf16* x, bf16* y, std::string* why) {
  cudaStream_t s = m->stream;
  const long long rin = static_cast<long long>(k.n) * k.h * k.w;
  const long long rout = static_cast<long long>(k.n) * k.ho * k.wo;
  const bool s1 = k.stride == 1;
  float* P = m->P;
  // conv a (1x1) + bn_a + ReLU -> a (padded for the 3x3)
  if (mm_fwd(m, x, rin, k.cin, k.wa, k.width, k.a_pre, why)) return 1;
  RALPB_TRY(bn_stats(Act4{k.a_pre, 0}, k.n, k.h, k.w, k.width, kBnEps, m->bn_work, mean_of(k, 0), rstd_of(k, 0), s,
                     k.groups, 8LL * k.cmax));
  {
    BnApply ap{};
    ap.x = Act4{k.a_pre, 0}; ap.mean = mean_of(k, 0); ap.rstd = rstd_of(k, 0);
    ap.gamma = P + k.ga_off; ap.beta = P + k.ga_off + k.width; ap.relu = 1; ap.y = MutAct4{k.a, 1};
    ap.mask_out = k.ma;
    ap.groups = k.groups; ap.stat_stride = 8LL * k.cmax;
    ap.n = k.n; ap.h = k.h; ap.w = k.w; ap.c = k.width;
    RALPB_TRY(bn_apply(ap, s));
  }
  // conv b (3x3, stride s) + bn_b + ReLU -> b
  if (s1) {
    RALPB_TRY(conv_fwd(geom_b(k), k.a, k.wbf, nullptr, k.b_pre, 0, s, why));
  } else {
    RALPB_TRY(im2col_bf16(Act4{k.a, 1}, k.n, k.h, k.w, k.width, 3, k.stride, 1, k.ho, k.wo, k.col, s));
    if (mm_fwd(m, k.col, rout, 9 * k.width, k.wbf, k.width, k.b_pre, why)) return 1;
  }
  const Act4 bpre{k.b_pre, s1 ? 1 : 0};
  RALPB_TRY(bn_stats(bpre, k.n, k.ho, k.wo, k.width, kBnEps, m->bn_work, mean_of(k, 1), rstd_of(k, 1), s,
                     k.groups, 8LL * k.cmax));
  {
    BnApply ap{};
    ap.x = bpre; ap.mean = mean_of(k, 1); ap.rstd = rstd_of(k, 1);
    ap.gamma = P + k.gb_off; ap.beta = P + k.gb_off + k.width; ap.relu = 1; ap.y = MutAct4{k.b, 0};
    ap.mask_out = k.mb;
    ap.groups = k.groups; ap.stat_stride = 8LL * k.cmax;
    ap.n = k.n; ap.h = k.ho; ap.w = k.wo; ap.c = k.width;
    RALPB_TRY(bn_apply(ap, s));
  }
  // conv c (1x1), the shortcut, bn_c + add + ReLU -> y
  if (mm_fwd(m, k.b, rout, k.width, k.wc, k.cout, k.c_pre, why)) return 1;
  RALPB_TRY(bn_stats(Act4{k.c_pre, 0}, k.n, k.ho, k.wo, k.cout, kBnEps, m->bn_work, mean_of(k, 2), rstd_of(k, 2), s,
                     k.groups, 8LL * k.cmax));
  if (k.down) {
    const bf16* xin = x;
    if (!s1) {
      RALPB_TRY(subsample(Act4{x, 0}, k.n, k.h, k.w, k.cin, k.stride, k.d_in, s));
      xin = k.d_in;
    }
    if (mm_fwd(m, xin, rout, k.cin, k.wd, k.cout, k.d_pre, why)) return 1;
    RALPB_TRY(bn_stats(Act4{k.d_pre, 0}, k.n, k.ho, k.wo, k.cout, kBnEps, m->bn_work, mean_of(k, 3), rstd_of(k, 3), s,
                       k.groups, 8LL * k.cmax));
  }
  {
    BnApply ap{};
    ap.x = Act4{k.c_pre, 0}; ap.mean = mean_of(k, 2); ap.rstd = rstd_of(k, 2);
    ap.gamma = P + k.gc_off; ap.beta = P + k.gc_off + k.cout;
    if (k.down) {
      ap.res_kind = 2; ap.r = Act4{k.d_pre, 0}; ap.r_mean = mean_of(k, 3); ap.r_rstd = rstd_of(k, 3);
      ap.r_gamma = P + k.gd_off; ap.r_beta = P + k.gd_off + k.cout;
    } else {
      ap.res_kind = 1; ap.r = Act4{x, 0};
    }
    ap.relu = 1; ap.y = MutAct4{y, 0};
    ap.mask_out = k.mc;
    ap.groups = k.groups; ap.stat_stride = 8LL * k.cmax;
    ap.n = k.n; ap.h = k.ho; ap.w = k.wo; ap.c = k.cout;
    RALPB_TRY(bn_apply(ap, s));
  }
  m->launches += k.down ? 16 : 12;
  return 0;
}

int block_backward(Model* m, BlockBufs& k, const bf16* x, const bf16* y, const bf16* dy, bf16* dx, std::string* why) {
  cudaStream_t s = m->stream;
  const long long rin = static_cast<long long>(k.n) * k.h * k.w;
  const long long rout = static_cast<long long>(k.n) * k.ho * k.wo;
  const bool s1 = k.stride == 1;
  float *P = m->P, *G = m->G;
  // bn_c (ReLU on the block output): dc_pre, and dz = the masked dy (the shortcut's gradient)
  {
    BnBackward bb{};
    bb.dy = Act4{dy, 0}; bb.y = Act4{y, 0}; bb.relu_mask = 1; bb.x = Act4{k.c_pre, 0};
    bb.mask_in = k.mc;
    bb.mean = mean_of(k, 2); bb.rstd = rstd_of(k, 2); bb.gamma = P + k.gc_off;
    bb.dgamma = G + k.gc_off; bb.dbeta = G + k.gc_off + k.cout;
    bb.dx = MutAct4{k.dc_pre, 0}; bb.dz_out = MutAct4{k.dz, 0};
    bb.groups = k.groups; bb.stat_stride = 8LL * k.cmax;
    bb.n = k.n; bb.h = k.ho; bb.w = k.wo; bb.c = k.cout;
    RALPB_TRY(bn_backward(bb, m->bn_work, s));
  }
  // conv c
  if (mm_wgrad(m, k.dc_pre, rout, k.cout, k.b, k.width, G + k.wc_off, why)) return 1;
  if (mm_dgrad(m, k.dc_pre, rout, k.cout, k.wc, k.width, k.db, why)) return 1;
  // bn_b (ReLU mask b): -> db_pre (padded for the stride-1 3x3's kernels)
  const MutAct4 dbpre{k.db_pre, s1 ? 1 : 0};
  {
    BnBackward bb{};
    bb.dy = Act4{k.db, 0}; bb.y = Act4{k.b, 0}; bb.relu_mask = 1; bb.x = Act4{k.b_pre, s1 ? 1 : 0};
    bb.mask_in = k.mb;
    bb.mean = mean_of(k, 1); bb.rstd = rstd_of(k, 1); bb.gamma = P + k.gb_off;
    bb.dgamma = G + k.gb_off; bb.dbeta = G + k.gb_off + k.width;
    bb.dx = dbpre;
    bb.groups = k.groups; bb.stat_stride = 8LL * k.cmax;
    bb.n = k.n; bb.h = k.ho; bb.w = k.wo; bb.c = k.width;
    RALPB_TRY(bn_backward(bb, m->bn_work, s));
  }
  // conv b: backward-filter and backward-data (-> da, padded)
  if (s1) {
    RALPB_TRY(conv_wgrad(geom_b(k), k.a, k.db_pre, G + k.wb_off, nullptr, s, why));
    RALPB_TRY(conv_dgrad(geom_b(k), k.db_pre, k.wbd, nullptr, k.da, nullptr, s, why));
  } else {
    if (mm_wgrad(m, k.db_pre, rout, k.width, k.col, 9 * k.width, G + k.wb_off, why)) return 1;
    RALPB_TRY(dilate(k.db_pre, k.n, k.ho, k.wo, k.width, k.stride, MutAct4{k.dil, 1}, k.h, k.w, s));
    RALPB_TRY(conv_dgrad(geom_b(k), k.dil, k.wbd, nullptr, k.da, nullptr, s, why));
  }
  // bn_a (ReLU mask a) -> da_pre
  {
    BnBackward bb{};
    bb.dy = Act4{k.da, 1}; bb.y = Act4{k.a, 1}; bb.relu_mask = 1; bb.x = Act4{k.a_pre, 0};
    bb.mask_in = k.ma;
    bb.mean = mean_of(k, 0); bb.rstd = rstd_of(k, 0); bb.gamma = P + k.ga_off;
    bb.dgamma = G + k.ga_off; bb.dbeta = G + k.ga_off + k.width;
    bb.dx = MutAct4{k.da_pre, 0};
    bb.groups = k.groups; bb.stat_stride = 8LL * k.cmax;
    bb.n = k.n; bb.h = k.h; bb.w = k.w; bb.c = k.width;
    RALPB_TRY(bn_backward(bb, m->bn_work, s));
  }
  // conv a
  if (mm_wgrad(m, k.da_pre, rin, k.width, x, k.cin, G + k.wa_off, why)) return 1;
  // dx = Wa^T da_pre (+ the identity shortcut's gradient dz, summed in the GEMM epilogue)
  const bool fuse = res_epilogue();
  if (dx != nullptr &&
      mm_dgrad(m, k.da_pre, rin, k.width, k.wa, k.cin, dx, why, k.down || !fuse ? nullptr : k.dz))
    return 1;
  // the shortcut
  if (k.down) {
    BnBackward bb{};
    bb.dy = Act4{k.dz, 0}; bb.relu_mask = 0; bb.x = Act4{k.d_pre, 0};
    bb.mean = mean_of(k, 3); bb.rstd = rstd_of(k, 3); bb.gamma = P + k.gd_off;
    bb.dgamma = G + k.gd_off; bb.dbeta = G + k.gd_off + k.cout;
    bb.dx = MutAct4{k.dd_pre, 0};
    bb.groups = k.groups; bb.stat_stride = 8LL * k.cmax;
    bb.n = k.n; bb.h = k.ho; bb.w = k.wo; bb.c = k.cout;
    RALPB_TRY(bn_backward(bb, m->bn_work, s));
    if (mm_wgrad(m, k.dd_pre, rout, k.cout, s1 ? x : k.d_in, k.cin, G + k.wd_off, why)) return 1;
    if (dx != nullptr) {
      if (s1 && fuse) {   // the projection's gradient accumulated into dx in the GEMM epilogue
        if (mm_dgrad(m, k.dd_pre, rout, k.cout, k.wd, k.cin, dx, why, dx)) return 1;
      } else if (s1) {
        if (mm_dgrad(m, k.dd_pre, rout, k.cout, k.wd, k.cin, k.dxs, why)) return 1;
        RALPB_TRY(add_act(Act4{dx, 0}, Act4{k.dxs, 0}, MutAct4{dx, 0}, k.n, k.h, k.w, k.cin, s));
      } else {
        if (mm_dgrad(m, k.dd_pre, rout, k.cout, k.wd, k.cin, k.dxs, why)) return 1;
        RALPB_TRY(add_strided(k.dxs, k.n, k.ho, k.wo, k.cin, k.stride, MutAct4{dx, 0}, s));
      }
    }
  } else if (dx != nullptr && !fuse) {
    RALPB_TRY(add_act(Act4{dx, 0}, Act4{k.dz, 0}, MutAct4{dx, 0}, k.n, k.h, k.w, k.cin, s));
  }
  m->launches += fuse && !(k.down && !s1) ? 23 : 24;
  return 0;
}

// The batch-normalised stem (im2col GEMM without a bias column): pre = patches . W^T;
// y = relu(bn(pre)).
int bn_stem_forward(Model* m, FrontLayer& f, const ActBuf& in, const ActBuf& out, std::string* why) {
  cudaStream_t s = m->stream;
  const long long rows = in.rows();
  if (mm_fwd(m, in.ptr, rows, f.kpad, f.wf, f.g.cout, f.pre, why)) return 1;
  const int c = f.g.cout;
  RALPB_TRY(bn_stats(Act4{f.pre, 0}, out.n, out.h, out.w, c, kBnEps, m->bn_work, f.bn_stats, f.bn_stats + c, s));
  BnApply ap{};
  ap.x = Act4{f.pre, 0}; ap.mean = f.bn_stats; ap.rstd = f.bn_stats + c;
  ap.gamma = m->P + f.b_off; ap.beta = m->P + f.b_off + c; ap.relu = 1; ap.y = MutAct4{out.ptr, out.pad};
  ap.mask_out = f.bn_mask;
  ap.n = out.n; ap.h = out.h; ap.w = out.w; ap.c = c;
  RALPB_TRY(bn_apply(ap, s));
  m->launches += 3;
  return 0;
}

int bn_stem_backward(Model* m, FrontLayer& f, const ActBuf& in, const ActBuf& out, const bf16* dy, std::string* why) {
  cudaStream_t s = m->stream;
  const int c = f.g.cout;
  BnBackward bb{};
  bb.dy = Act4{dy, out.pad}; bb.y = Act4{out.ptr, out.pad}; bb.relu_mask = 1; bb.x = Act4{f.pre, 0};
  bb.mask_in = f.bn_mask;
  bb.mean = f.bn_stats; bb.rstd = f.bn_stats + c; bb.gamma = m->P + f.b_off;
  bb.dgamma = m->G + f.b_off; bb.dbeta = m->G + f.b_off + c;
  bb.dx = MutAct4{f.dpre, 0};
  bb.n = out.n; bb.h = out.h; bb.w = out.w; bb.c = c;
  RALPB_TRY(bn_backward(bb, m->bn_work, s));
  if (mm_wgrad(m, f.dpre, in.rows(), c, in.ptr, f.kpad, m->G + f.w_off, why)) return 1;
  m->launches += 3;
  return 0;
}

}  // namespace ralpb
