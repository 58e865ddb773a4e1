// Host planning / launch of the slab-tiled conv kernels (see conv_slab.cuh).
#include <cudaTypedefs.h>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include "conv.cuh"
#include "elementwise.cuh"
#include "conv_slab.cuh"

namespace ralpb {

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

static CUtensorMapSwizzle swz_mode(int bytes) {
  return bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
}

// Padded activation [n][hp][wp][c] as a 4-D tensor, box {bc, bw, bh, 1}.
bool encode_act(CUtensorMap* tm, const void* ptr, long long c, long long wp, long long hp, long long n, int bc, int bw,
                int bh, int swz, std::string* why) {
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(wp), static_cast<cuuint64_t>(hp),
                        static_cast<cuuint64_t>(n)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(c) * 2, static_cast<cuuint64_t>(wp * c) * 2,
                           static_cast<cuuint64_t>(hp * wp * c) * 2};
  cuuint32_t box[4] = {static_cast<cuuint32_t>(bc), static_cast<cuuint32_t>(bw), static_cast<cuuint32_t>(bh), 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = encoder()(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, swz_mode(swz), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { *why = "3-D tensor map encode failed (" + std::to_string(static_cast<int>(r)) + ")"; return false; }
  return true;
}

bool encode_mat(CUtensorMap* tm, const void* ptr, long long rows, long long cols, int bc, int br, int swz,
                std::string* why) {
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(bc), static_cast<cuuint32_t>(br)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encoder()(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, swz_mode(swz), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { *why = "2-D tensor map encode failed (" + std::to_string(static_cast<int>(r)) + ")"; return false; }
  return true;
}

// Interior view of a padded activation [n][hp][wp][c]: dims {c, w, h, n} starting at pixel
// (pad, pad) with the padded strides, box {32, 8, 16, 1}, 64B swizzle -- TMA stores through it
// clip at the image edge, so the zero borders are never written.
bool encode_interior(CUtensorMap* tm, void* ptr, long long c, long long w, long long h, long long wp, long long hp,
                     long long n, int pad, std::string* why) {
  return encode_interior_box(tm, ptr, c, w, h, wp, hp, n, pad, 8, 16, why);
}

bool encode_interior_box(CUtensorMap* tm, void* ptr, long long c, long long w, long long h, long long wp, long long hp,
                         long long n, int pad, int bw, int bh, std::string* why) {
  char* base = static_cast<char*>(ptr) + (static_cast<long long>(pad) * wp + pad) * c * 2;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(w), static_cast<cuuint64_t>(h),
                        static_cast<cuuint64_t>(n)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(c) * 2, static_cast<cuuint64_t>(wp * c) * 2,
                           static_cast<cuuint64_t>(hp * wp * c) * 2};
  cuuint32_t box[4] = {32, static_cast<cuuint32_t>(bw), static_cast<cuuint32_t>(bh), 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = encoder()(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { *why = "interior tensor map encode failed (" + std::to_string(static_cast<int>(r)) + ")"; return false; }
  return true;
}

namespace {

int align1k(int x) { return (x + 1023) & ~1023; }
constexpr int kSmemBudget = 227 * 1024 - 1024 - 512 - 2048;

}  // namespace

bool slab_fwd_ok(const ConvGeom& g, int c, int cout) {
  // cout % 32: the TMA-store epilogue writes 32-channel boxes
  return g.k == 2 * g.pad + 1 && (g.k == 3 || g.k == 5) && (c == 16 || c == 32 || c % 64 == 0) && cout % 32 == 0 &&
         g.q() < (1LL << 31);
}

bool slab_wgrad_ok(const ConvGeom& g) {
  return ((g.k == 3 && g.pad == 1) || (g.k == 5 && g.pad == 2)) && g.cin % 64 == 0 && g.cout % 64 == 0 &&
         g.q() < (1LL << 31);
}

// Algorithmic DRAM bytes of one launch (each operand once): input interior, filters, output
// interior (+ the ReLU mask it reads, the fused pool's output / argmax bytes).
double slab_fwd_bytes(const ConvGeom& g, int c, int cout, bool mask, bool pool, bool idx) {
  const double px = static_cast<double>(g.n) * g.h * g.w;
  double b = px * c * 2.0 + static_cast<double>(g.taps()) * c * cout * 2.0 + px * cout * 2.0;
  if (mask) b += px * cout * 2.0;
  if (pool) b += px / 4.0 * cout * 2.0;
  if (idx) b += px / 4.0 * cout;
  return b;
}
double wgrad_bytes(const ConvGeom& g) {
  const double px = static_cast<double>(g.n) * g.h * g.w;
  return px * (g.cin + g.cout) * 2.0 + static_cast<double>(g.taps()) * g.cin * g.cout * 4.0;
}

cudaError_t conv_slab_fwd(const ConvGeom& g, const void* x_pad, const void* w, int c, int cout, const float* bias,
                          int relu, const void* mask_pad, void* y_pad, float* colsum, cudaStream_t s,
                          std::string* why, void* pool_out, int pool_pad, void* pool_idx) {
  if (pool_out != nullptr && (g.h % 2 != 0 || g.w % 2 != 0)) { *why = "fused pool needs even h, w"; return cudaErrorInvalidValue; }
  if (row64_ok(g, c, cout, pool_idx))   // 64 -> 64 channels: row-streamed kernel (conv_row.cu)
    return conv_row64_fwd(g, x_pad, w, bias, relu, mask_pad, y_pad, colsum, pool_out, pool_pad, s, why);
  if (colsum != nullptr && cout > 512) { *why = "slab conv: fused colsum supports <= 512 channels"; return cudaErrorInvalidValue; }
  SlabConvParams p;
  std::memset(&p, 0, sizeof(p));
  p.n = g.n; p.h = g.h; p.w = g.w; p.hp = g.hp(); p.wp = g.wp(); p.pad = g.pad; p.k = g.k; p.taps = g.taps();
  p.c = c; p.cout = cout;
  p.kb = std::min(64, c);
  p.row_bytes = p.kb * 2;
  p.bn = cout >= 256 ? 256 : cout >= 128 ? 128 : cout >= 64 ? 64 : 32;
  p.macc = p.bn >= 256 ? 1 : p.bn >= 128 ? 2 : 4;
  // CTA pairs for 128/256-wide filter tiles: each SM loads half of every filter tile (the
  // 256-wide tiles' filter stream is ~60 B/cycle/SM from L2 on a single CTA).  Measured +5-8 %
  // (tools/probe_conv.py); not for the 64-wide filter-resident conv1_2 shape (-20 %) nor where
  // stacking two row blocks pads the image further (14x14: -35 %).
  // RALPB_FWD_PAIR=0 disables.
  const char* penv = getenv("RALPB_FWD_PAIR");
  const int rows1 = (g.h + 16 * p.macc - 1) / (16 * p.macc) * 16 * p.macc;
  const int rows2 = (g.h + 32 * p.macc - 1) / (32 * p.macc) * 32 * p.macc;
  // 64-wide tiles pair up only outside the filter-resident mode (conv2_1 dgrad: +10 %)
  const char* nwe = getenv("RALPB_NO_WRES");
  const bool no_wres = nwe != nullptr && nwe[0] == '1';
  const bool wres_shape = c == p.kb && cout <= p.bn && !no_wres;
  const bool pair = (p.bn == 128 || p.bn == 256 || (p.bn == 64 && !wres_shape)) && rows2 == rows1 &&
                    !(penv != nullptr && penv[0] == '0');
  const int ncta = pair ? 2 : 1;
  const int brows = p.bn / ncta;   // filter rows per CTA
  p.sw = 8 + g.k - 1;
  p.b_load = brows * p.row_bytes;
  p.b_stage = align1k(p.b_load);
  p.na = 2;
  int staging = 0, budget = 0;
  int nb_cap = 8;
  if (const char* e = getenv("RALPB_NB")) nb_cap = std::max(2, std::min(16, atoi(e)));
  // M accumulators per tile: shrink until two slab stages, two filter stages and the output
  // staging (2 x 8 KB per epilogue warpgroup, TMA-store epilogue) fit in shared memory
  for (;;) {
    p.sh = 16 * p.macc + g.k - 1;
    p.slab_load = p.row_bytes * p.sw * p.sh;
    p.slab_stage = align1k(p.slab_load);
    staging = (p.macc >= 2 ? 2 : 1) * kOutBufs * 8192;
    budget = kSmemBudget - staging;
    p.nb = std::min(nb_cap, (budget - p.na * p.slab_stage) / p.b_stage);
    if (p.nb >= 2 || p.macc == 1) break;
    p.macc /= 2;
  }
  // as many TMEM accumulator buffers (<= 4) as fit: the MMA runs ahead of the epilogue
  p.acc_bufs = std::max(1, std::min(4, 512 / (p.macc * p.bn)));
  if (const char* ae = getenv("RALPB_ACC_BUFS")) p.acc_bufs = std::max(1, std::min(p.acc_bufs, atoi(ae)));
  const int used = p.macc * p.bn * p.acc_bufs;
  p.tmem_cols = used <= 32 ? 32 : used <= 64 ? 64 : used <= 128 ? 128 : used <= 256 ? 256 : 512;
  // Filters resident in shared memory when one channel block and one N tile cover the layer
  // (e.g. 64->64 at 224x224): the per-tile filter reloads disappear.
  if (wres_shape && p.macc >= 2) {
    const int macc2 = 2;
    const int slab2 = align1k(p.row_bytes * p.sw * (16 * macc2 + g.k - 1));
    const int na2 = g.taps() * p.b_stage + 3 * slab2 <= budget ? 3 : 2;
    if (g.taps() * p.b_stage + na2 * slab2 <= budget && g.taps() <= 16) {
      p.wres = 1;
      p.macc = macc2;
      p.sh = 16 * macc2 + g.k - 1;
      p.slab_load = p.row_bytes * p.sw * p.sh;
      p.slab_stage = slab2;
      p.na = na2;
      p.nb = g.taps();
      p.acc_bufs = std::max(1, std::min(4, 512 / (p.macc * p.bn)));
      if (const char* ae = getenv("RALPB_ACC_BUFS")) p.acc_bufs = std::max(1, std::min(p.acc_bufs, atoi(ae)));
      const int used2 = p.macc * p.bn * p.acc_bufs;
      p.tmem_cols = used2 <= 256 ? 256 : 512;
    }
  }
  if (p.nb < 2) { *why = "slab conv: tile does not fit in shared memory"; return cudaErrorInvalidValue; }
  p.n_hb = (g.h + 16 * p.macc * ncta - 1) / (16 * p.macc * ncta);
  p.n_wb = (g.w + 7) / 8;
  p.n_nt = (cout + p.bn - 1) / p.bn;
  p.idesc = umma_idesc_bf16(128 * ncta, p.bn, false, false);
  p.out = static_cast<__nv_bfloat16*>(y_pad);
  p.bias = bias;
  p.relu = relu;
  p.mask = static_cast<const __nv_bfloat16*>(mask_pad);
  p.colsum = colsum;
  p.pool_out = static_cast<__nv_bfloat16*>(pool_out);
  p.pool_pad = pool_pad;
  p.pool_idx = static_cast<uint8_t*>(pool_idx);
  if (const char* e = getenv("RALPB_DEBUG")) p.dbg = atoi(e);
  if (!encode_act(&p.tmX, x_pad, c, g.wp(), g.hp(), g.n, p.kb, p.sw, p.sh, p.row_bytes, why))
    return cudaErrorInvalidValue;
  if (!encode_mat(&p.tmB, w, cout, static_cast<long long>(g.taps()) * c, p.kb, brows, p.row_bytes, why))
    return cudaErrorInvalidValue;
  if (!encode_interior(&p.tmY, y_pad, cout, g.w, g.h, g.wp(), g.hp(), g.n, g.pad, why)) return cudaErrorInvalidValue;
  const int smem = 1024 + p.na * p.slab_stage + p.nb * p.b_stage + staging + 512 + 2048;  // barriers, colsum
  const long long total = static_cast<long long>(g.n) * p.n_hb * p.n_wb * p.n_nt;
  const int grid = pair ? 2 * static_cast<int>(std::min<long long>(total, num_sms() / 2))
                        : static_cast<int>(std::min<long long>(total, num_sms()));
  const int ks = p.kb / 16;
  bool launched = false;
  auto go = [&](auto kern, int threads, bool cluster) {
    static_cast<void>(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    launch_timed([&] {
      static_cast<void>(launch_pdl(kern, dim3(grid), dim3(threads), smem, s, cluster ? 2 : 1, p));
    }, s, cluster ? KIND_CONV_FWD_PAIR : KIND_CONV_FWD, 2.0 * g.n * g.h * g.w * static_cast<double>(g.taps()) * c * cout,
       slab_fwd_bytes(g, c, cout, mask_pad != nullptr, pool_out != nullptr, pool_idx != nullptr));
    launched = true;
  };
#define RALPB_SLAB_CASE(KK, KS, MA)                                                                   \
  if (g.k == KK && ks == KS && p.macc == MA) {                                                        \
    if (pair) {                                                                                       \
      go(conv_slab_fwd_kernel<KK, KS, MA, true>, 128 + 128 * (MA >= 2 ? 2 : 1), true);                \
    } else {                                                                                          \
      go(conv_slab_fwd_kernel<KK, KS, MA, false>, 128 + 128 * (MA >= 2 ? 2 : 1), false);              \
    }                                                                                                 \
  }
  RALPB_SLAB_CASE(3, 4, 1) RALPB_SLAB_CASE(3, 4, 2) RALPB_SLAB_CASE(3, 4, 4)
  RALPB_SLAB_CASE(3, 2, 1) RALPB_SLAB_CASE(3, 2, 2) RALPB_SLAB_CASE(3, 2, 4)
  RALPB_SLAB_CASE(3, 1, 1) RALPB_SLAB_CASE(3, 1, 2) RALPB_SLAB_CASE(3, 1, 4)
  RALPB_SLAB_CASE(5, 4, 1) RALPB_SLAB_CASE(5, 4, 2) RALPB_SLAB_CASE(5, 4, 4)
  RALPB_SLAB_CASE(5, 2, 1) RALPB_SLAB_CASE(5, 2, 2) RALPB_SLAB_CASE(5, 2, 4)
  RALPB_SLAB_CASE(5, 1, 1) RALPB_SLAB_CASE(5, 1, 2) RALPB_SLAB_CASE(5, 1, 4)
#undef RALPB_SLAB_CASE
  if (!launched) { *why = "slab conv: no kernel instance for this filter/channel/tile shape"; return cudaErrorInvalidValue; }
  return cudaGetLastError();
}

cudaError_t conv_slab_wgrad(const ConvGeom& g, const void* x_pad, const void* dy_pad, float* dw, float* db,
                            cudaStream_t s, std::string* why) {
  SlabConvParams p;
  std::memset(&p, 0, sizeof(p));
  p.n = g.n; p.h = g.h; p.w = g.w; p.hp = g.hp(); p.wp = g.wp(); p.pad = g.pad; p.k = g.k; p.taps = g.taps();
  p.c = g.cin; p.cout = g.cout;
  p.kb = 64;
  p.row_bytes = 128;
  p.bn = 64;
  // pixel blocks of bh rows x 8 columns; 14 divides every VGG feature-map height
  const int bh = g.h % 14 == 0 ? 14 : 16;
  p.sw = 8 + g.k - 1;
  p.sh = bh + g.k - 1;
  p.slab_load = 128 * p.sw * p.sh;
  p.slab_stage = align1k(p.slab_load);
  p.b_load = 128 * 8 * bh;
  p.b_stage = align1k(p.b_load);
  p.na = std::min(8, (kSmemBudget - 4096) / (p.slab_stage + p.b_stage));
  p.tmem_cols = 512;  // 5 tap-pair accumulators + bias = 384 columns
  p.n_hb = (g.h + bh - 1) / bh;
  p.n_wb = (g.w + 7) / 8;
  p.n_pix_blocks = g.n * p.n_hb * p.n_wb;
  p.n_ci_blocks = g.cin / 64;
  p.n_co_blocks = g.cout / 64;
  p.idesc = umma_idesc_bf16(128, 64, true, true);
  p.n_splits = g.k == 5 ? 2 : 1;   // tap groups: 25 taps = 16 + 9 (8 tap-pair accumulators per pass)
  p.dw = dw;
  p.db = db;
  if (!encode_act(&p.tmX, x_pad, g.cin, g.wp(), g.hp(), g.n, 64, p.sw, p.sh, 128, why)) return cudaErrorInvalidValue;
  if (!encode_act(&p.tmB, dy_pad, g.cout, g.wp(), g.hp(), g.n, 64, 8, bh, 128, why)) return cudaErrorInvalidValue;
  const int smem = 1024 + 4096 + p.na * (p.slab_stage + p.b_stage) + 512;
  const long long units = static_cast<long long>(p.n_ci_blocks) * p.n_co_blocks * p.n_splits * p.n_pix_blocks;
  const int grid = static_cast<int>(std::min<long long>(units, num_sms()));
  // CTA-pair kernel (M=256 x N=128 UMMAs, 3x3) when the output channels come in 128s
  const char* wenv = getenv("RALPB_WGRAD");
  const bool pair = g.k == 3 && g.cout % 128 == 0 && !(wenv != nullptr && std::strcmp(wenv, "single") == 0);
  if (pair) {
    p.n_co_blocks = g.cout / 128;
    p.idesc = umma_idesc_bf16(256, 128, true, true);
    const int smem2 = 1024 + p.na * (p.slab_stage + p.b_stage) + 512;
    const long long units2 = static_cast<long long>(p.n_ci_blocks) * p.n_co_blocks * p.n_pix_blocks;
    const int clusters = static_cast<int>(std::min<long long>(units2, num_sms() / 2));
    auto go2 = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      launch_timed([&] { static_cast<void>(launch_pdl(kern, dim3(2 * clusters), dim3(256), smem2, s, 1, p)); }, s, KIND_WGRAD_PAIR,
                   2.0 * g.n * g.h * g.w * static_cast<double>(g.taps()) * g.cin * g.cout, wgrad_bytes(g));
    };
    if (bh == 14) go2(conv_slab_wgrad_pair_kernel<14>); else go2(conv_slab_wgrad_pair_kernel<16>);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || db == nullptr) return e;
    return colsum_bf16(static_cast<const __nv_bfloat16*>(dy_pad), g.q(), g.cout, g.cout, db, s);
  }
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    launch_timed([&] { static_cast<void>(launch_pdl(kern, dim3(grid), dim3(256), smem, s, 1, p)); }, s, KIND_WGRAD,
                 2.0 * g.n * g.h * g.w * static_cast<double>(g.taps()) * g.cin * g.cout, wgrad_bytes(g));
  };
  if (g.k == 5) {
    go(bh == 14 ? conv_slab_wgrad_kernel<14, 5> : conv_slab_wgrad_kernel<16, 5>);
    cudaError_t e = cudaGetLastError();   // no bias accumulator for 5x5: db from dY's column sums
    if (e != cudaSuccess || db == nullptr) return e;
    return colsum_bf16(static_cast<const __nv_bfloat16*>(dy_pad), g.q(), g.cout, g.cout, db, s);
  }
  if (bh == 14) go(conv_slab_wgrad_kernel<14, 3>); else go(conv_slab_wgrad_kernel<16, 3>);
  return cudaGetLastError();
}

}  // namespace ralpb
