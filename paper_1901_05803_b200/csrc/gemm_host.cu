#include <cudaTypedefs.h>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include "gemm_host.cuh"
#include "gemm.cuh"

namespace ralpb {

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode;
}

static thread_local GemmTimer* g_timer = nullptr;
void set_gemm_timer(GemmTimer* t) { g_timer = t; }
GemmTimer* current_gemm_timer() { return g_timer; }

int num_sms() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

static bool encode_2d(CUtensorMap* tm, const Operand2D& op, int box_cols, int box_rows, int swz,
                      std::string* why) {
  auto fn = encode_fn();
  if (!fn) { *why = "cuTensorMapEncodeTiled unavailable"; return false; }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(op.cols), static_cast<cuuint64_t>(op.rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(op.ld) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMapSwizzle sw = swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                      : CU_TENSOR_MAP_SWIZZLE_32B;
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(op.ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *why = "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ") rows=" +
           std::to_string(op.rows) + " cols=" + std::to_string(op.cols) + " ld=" +
           std::to_string(op.ld) + " box=" + std::to_string(box_cols) + "x" + std::to_string(box_rows);
    return false;
  }
  return true;
}

static bool is_k(int mode) { return mode == LD_K || mode == LD_K_CONV; }

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("RALPB_PDL");
    return e == nullptr || e[0] != '0';
  }();
  return on;
}

cudaError_t gemm_launch(const GemmDesc& d, cudaStream_t stream, std::string* why) {
  static bool attr_set = false;
  if (d.M <= 0 || d.N <= 0 || d.K <= 0) return cudaSuccess;
  GemmParams p;
  std::memset(&p, 0, sizeof(p));
  p.M = d.M;
  p.N = d.N;
  // ---- tile shape
  int bn = d.block_n;
  if (bn == 0) {
    bn = d.N >= 256 ? 256 : (d.N > 64 ? 128 : (d.N > 32 ? 64 : 32));
  }
  if (!(bn == 32 || bn == 64 || bn == 128 || bn == 256)) { *why = "bad block_n"; return cudaErrorInvalidValue; }
  if (!is_k(d.b_mode) && bn < 32) { *why = "MN-major B needs BN>=32"; return cudaErrorInvalidValue; }
  p.block_n = bn;
  const bool a_k = is_k(d.a_mode), b_k = is_k(d.b_mode);
  if (a_k != b_k && (a_k ? d.kb : 64) != 64) { *why = "mixed-major GEMM needs kb=64"; return cudaErrorInvalidValue; }
  int kb = a_k ? d.kb : 64;
  if (!(kb == 16 || kb == 32 || kb == 64)) { *why = "kb must be 16/32/64"; return cudaErrorInvalidValue; }
  p.kb = kb;
  // ---- swizzles
  // LD_MN_CONV: the widest swizzle atom that divides one tap's channel row (e.g. 96 channels -> 64 B)
  const int conv_row = d.a_cin * 2;
  p.a_swz = a_k ? kb * 2
                : (d.a_mode == LD_MN_CONV ? (conv_row % 128 == 0 ? 128 : (conv_row % 64 == 0 ? 64 : 32)) : 128);
  p.b_swz = b_k ? kb * 2 : std::min(128, bn * 2);
  if (d.a_mode == LD_MN_CONV && (d.a_cin * 2) % p.a_swz != 0) { *why = "a_cin must be a multiple of the atom"; return cudaErrorInvalidValue; }
  p.a_bytes = a_k ? kBM * kb * 2 : kBM * 64 * 2;
  p.b_bytes = b_k ? bn * kb * 2 : bn * 64 * 2;
  p.b_stage_bytes = std::max(1024, bn * 128);
  // ---- tensor maps
  if (a_k) {
    if (!encode_2d(&p.tmA, d.a, kb, kBM, p.a_swz, why)) return cudaErrorInvalidValue;
  } else {
    if (!encode_2d(&p.tmA, d.a, p.a_swz / 2, 64, p.a_swz, why)) return cudaErrorInvalidValue;
  }
  if (b_k) {
    if (!encode_2d(&p.tmB, d.b, kb, bn, p.b_swz, why)) return cudaErrorInvalidValue;
  } else {
    if (!encode_2d(&p.tmB, d.b, p.b_swz / 2, 64, p.b_swz, why)) return cudaErrorInvalidValue;
  }
  // ---- grid
  p.n_mt = (d.M + kBM - 1) / kBM;
  p.n_nt = (d.N + bn - 1) / bn;
  const long long kblocks = a_k ? (d.K + kb - 1) / kb : (d.K + 63) / 64;
  p.kblocks_total = static_cast<int>(kblocks);
  const int sms = num_sms();
  int splits = d.k_splits;
  if (splits == 0) {
    // split-K minimising (waves of the persistent grid) x (k-blocks per unit + a per-unit
    // epilogue/setup cost of ~8 k-blocks), >= 4 k-blocks per split.  Wave quantisation is what
    // matters at the FC shapes: M=512 x N=4096 (64 tiles) runs best at 2 splits, M=1024 (128
    // tiles) unsplit (tools/probe_fc_gemm.py); the old "~2 waves" rule picked 5 and 3.
    const long long tiles = static_cast<long long>(p.n_mt) * p.n_nt;
    const long long maxs = std::max<long long>(1, std::min<long long>(kblocks / 4, 4LL * sms));
    long long best = -1;
    splits = 1;
    for (long long sp = 1; sp <= maxs; ++sp) {
      const long long waves = (tiles * sp + sms - 1) / sms;
      const long long cost = waves * ((kblocks + sp - 1) / sp + 8);
      if (best < 0 || cost < best) { best = cost; splits = static_cast<int>(sp); }
    }
  }
  if (splits > 1 && d.epi != EPI_F32_ATOMIC) { *why = "split-K needs the atomic epilogue"; return cudaErrorInvalidValue; }
  p.kblocks_per_split = static_cast<int>((kblocks + splits - 1) / splits);
  p.n_ks = static_cast<int>((kblocks + p.kblocks_per_split - 1) / p.kblocks_per_split);
  // ---- TMA epilogue: coalesced 128x32 boxes (store, or reduce-add for split-K) instead of
  // per-thread row stores (RALPB_GEMM_TMA_EPI=0 disables)
  {
    const char* te = getenv("RALPB_GEMM_TMA_EPI");
    const bool allowed = !(te != nullptr && te[0] == '0');
    const int esz = d.epi == EPI_BF16 ? 2 : 4;
    const bool shape_ok = d.s_n == 1 && !d.border && d.N >= 32 &&
                          (reinterpret_cast<uintptr_t>(d.out) & 15) == 0 && (d.s_m * esz) % 16 == 0;
    if (allowed && shape_ok && (d.epi == EPI_F32 || d.epi == EPI_BF16 || d.epi == EPI_F32_ATOMIC)) {
      auto fn = encode_fn();
      cuuint64_t dims[2] = {static_cast<cuuint64_t>(d.N), static_cast<cuuint64_t>(d.M)};
      cuuint64_t strides[1] = {static_cast<cuuint64_t>(d.s_m) * esz};
      cuuint32_t box[2] = {32, 128};
      cuuint32_t estr[2] = {1, 1};
      CUresult r = fn(&p.tmC, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                      d.out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      esz == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r == CUDA_SUCCESS) p.tma_epi = d.epi == EPI_F32_ATOMIC ? 2 : 1;
    }
  }
  // ---- stages
  const int stage_bytes = kAStage + p.b_stage_bytes;
  const int staging = p.tma_epi ? 2 * 16384 : 0;
  const int budget = 227 * 1024 - 1024 - 256 - staging;
  static const int max_stages = [] { const char* e = getenv("RALPB_GEMM_MAX_STAGES"); return e ? atoi(e) : 8; }();
  p.stages = std::min(max_stages, budget / stage_bytes);
  if (const char* e = getenv("RALPB_STAGES")) p.stages = std::max(1, std::min(p.stages, atoi(e)));
  const int smem = 1024 + p.stages * stage_bytes + staging + 256;
  // RALPB_GEMM_PRODUCERS=2 keeps two producer warps for the MN-major modes too (A/B)
  static const int mn_producers = [] {
    const char* e = getenv("RALPB_GEMM_PRODUCERS");
    return e != nullptr ? std::max(2, std::min(3, atoi(e))) : 3;
  }();
  // RALPB_GEMM_PRODUCERS_K=3: the K-major modes too (Inception / GoogLeNet / ResNet-50 steps
  // -0.3-0.6 %, the VGG-16 step within noise, -0.3 %: left at 2)
  static const int k_producers = [] {
    const char* e = getenv("RALPB_GEMM_PRODUCERS_K");
    return e != nullptr ? std::max(2, std::min(3, atoi(e))) : 2;
  }();
  p.producers = (d.a_mode == LD_MN || d.a_mode == LD_MN_CONV) ? mn_producers : k_producers;
  p.idesc = umma_idesc_bf16(kBM, bn, !a_k, !b_k);
  p.a_mode = d.a_mode;
  p.b_mode = d.b_mode;
  p.cblks = d.cblks;
  p.a_cin = d.a_cin;
  p.taps = d.taps;
  if (d.taps > kMaxTaps) { *why = "too many taps"; return cudaErrorInvalidValue; }
  for (int i = 0; i < d.taps; ++i) p.tap_off[i] = d.tap_off[i];
  p.epi = d.epi;
  p.relu = d.relu;
  p.out = d.out;
  p.s_m = d.s_m;
  p.s_n = d.s_n;
  p.bias = d.bias;
  p.sgd_mom = d.sgd_mom;
  p.sgd_bf16 = d.sgd_bf16;
  p.sgd_lr = d.sgd_lr;
  p.sgd_mu = d.sgd_mu;
  p.mask = reinterpret_cast<const __nv_bfloat16*>(d.mask);
  p.mask_s = d.mask_s;
  p.residual = reinterpret_cast<const __nv_bfloat16*>(d.residual);
  p.res_s = d.res_s;
  if (d.residual != nullptr && d.epi != EPI_BF16) { *why = "residual: EPI_BF16 only"; return cudaErrorInvalidValue; }
  p.border = d.border;
  p.img_rows = d.img_rows;
  p.wp = d.wp;
  p.pad = d.pad;
  p.h = d.h;
  p.w = d.w;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_sm100_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_set = true;
  }
  const long long total = static_cast<long long>(p.n_mt) * p.n_nt * p.n_ks;
  const int grid = static_cast<int>(std::min<long long>(total, sms));
  const double esz_out = d.epi == EPI_BF16 ? 2.0 : 4.0;
  launch_timed([&] { static_cast<void>(launch_pdl(gemm_sm100_kernel, dim3(grid), dim3(kThreads), smem, stream, 1, p)); },
               stream, KIND_GEMM, 2.0 * d.M * d.N * static_cast<double>(d.K),
               2.0 * (static_cast<double>(d.M) + d.N) * static_cast<double>(d.K) + esz_out * d.M * static_cast<double>(d.N));
  return cudaGetLastError();
}

}  // namespace ralpb
