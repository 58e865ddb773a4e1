// The first (RGB) convolution of a 224x224 network, fused with its im2col.
//
// conv1 of VGG-16 contracts only 27 values per output pixel (3x3 taps x 3 channels), so as an
// implicit GEMM it is pure data movement: the im2col GEMM path (pack_im2col -> 418 MB patch
// matrix in HBM -> GEMM -> 822 MB output; wgrad GEMM re-reading both) spent ~1 ms per step
// on ~66 GFLOP (profiles/r01).  Here the patch rows are built in shared memory straight from
// the fp32 NHWC image (77 MB at b=128) by four producer warps and fed to tcgen05:
//
//   conv_first_fwd_kernel    A = patches [128 px][32] (K-major, SW64; column 27 = 1.0 carries
//                            the bias), B = filters [64][32] resident; D (TMEM, 2 buffers) ->
//                            ReLU -> bf16 -> shared staging (SW128) -> one TMA store per tile
//                            (coalesced 16 KB writes instead of per-thread 128 B rows).
//   conv_first_wgrad_kernel  dW[co][k] += sum_px dY[px][co] * patch[px][k]: A = patch^T
//                            (MN-major view of the same SW64 rows; M = 32 real rows of 128),
//                            B = dY tile (TMA, MN-major SW128); one TMEM accumulator per CTA
//                            over all its tiles, reduced into dW once at the end.
//
// Tiles are 8 rows x 16 columns of output pixels (h % 8 == 0, w % 16 == 0); stride 1,
// 3x3, pad 1, 3 input channels, 64 output channels.  Rounding matches pack_im2col + GEMM:
// image values and the bias column go through bf16 RN, accumulation in fp32 (oracle:
// oracle/step.py _front_forward, first-conv bias rounding).
#include <algorithm>
#include <cstring>
#include "conv.cuh"
#include "ptx.cuh"

namespace ralpb {

namespace {

constexpr int kTH = 8, kTW = 16;         // output tile (rows x cols) = 128 pixels
constexpr int kStages = 4;
#ifndef RALPB_FIRST_GROUPS
#define RALPB_FIRST_GROUPS 3
#endif
constexpr int kGroups = RALPB_FIRST_GROUPS;   // producer warpgroups (tiles alternate between them)
constexpr int kProd = 4 * kGroups;            // producer warps
#ifndef RALPB_FIRST_OUTBUFS
#define RALPB_FIRST_OUTBUFS 4
#endif
constexpr int kOutBufs = RALPB_FIRST_OUTBUFS;   // forward output staging buffers (16 KB each)
#ifndef RALPB_FIRST_EPI
#define RALPB_FIRST_EPI 2
#endif
constexpr int kEpi = RALPB_FIRST_EPI;            // forward epilogue warpgroups (tiles alternate)
constexpr int kFwdWarps = kProd + 4 * kEpi + 1;  // producers, epilogue warpgroups, MMA warp
constexpr int kMmaWarp = kProd + 4 * kEpi;
constexpr int kAccs = 2 * kEpi;                  // 64-column TMEM accumulators
constexpr int kTmemCols = kAccs * 64 <= 128 ? 128 : kAccs * 64 <= 256 ? 256 : 512;
static_assert(kAccs * 64 <= 512, "TMEM holds 512 columns");
static_assert(kOutBufs % kEpi == 0, "staging buffers split evenly over the epilogue warpgroups");

struct FirstConvParams {
  CUtensorMap tmY;        // fwd: output (store); wgrad: dY (load); [n][hp][wp][64] box {64,16,8,1}
  const float* img;       // [n][h][w][cin] fp32
  const __nv_bfloat16* wf;  // [64][32] bf16 (column 27 = bias)
  float* dw;              // wgrad: [64][32] fp32, accumulated
  int n, h, w, cin, pad_out;
  int tiles_w, tiles_h, total;
};

// Patch row of output pixel (y, x): k = (r*3+s)*cin + ch, column 9*cin = 1 (bias), then 0,
// stored as one 64-byte K-major SW64 row (16-byte chunk c lands at c ^ ((row >> 1) & 3)).
__device__ __forceinline__ void build_patch_row(const FirstConvParams& p, int img, int y, int x, uint8_t* tile,
                                                int row) {
  float v[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = 0.f;
  const float* base = p.img + (static_cast<long long>(img) * p.h) * p.w * p.cin;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int yy = y + r - 1;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int xx = x + s - 1;
      const bool in = yy >= 0 && yy < p.h && xx >= 0 && xx < p.w;
      const float* src = base + (static_cast<long long>(yy) * p.w + xx) * p.cin;
#pragma unroll
      for (int ch = 0; ch < 3; ++ch)
        if (in) v[(r * 3 + s) * 3 + ch] = __ldg(src + ch);
    }
  }
  v[27] = 1.f;
  uint32_t w32[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) w32[j] = pack_bf16(v[2 * j], v[2 * j + 1]);
  uint8_t* dst = tile + row * 64;
  const int sw = (row >> 1) & 3;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    *reinterpret_cast<uint4*>(dst + ((c ^ sw) << 4)) = make_uint4(w32[4 * c], w32[4 * c + 1], w32[4 * c + 2], w32[4 * c + 3]);
}

// Producer warpgroup g builds the patch tiles of local tiles j = g, g + kGroups, ... (thread =
// pixel, 27 gathers each); several groups keep more image loads in flight.
__device__ __forceinline__ void produce_tiles(const FirstConvParams& p, uint8_t* sP, uint64_t* full, uint64_t* empty) {
  const int g = threadIdx.x >> 7, m = threadIdx.x & 127;
  for (int j = g;; j += kGroups) {
    const int t = static_cast<int>(blockIdx.x) + j * static_cast<int>(gridDim.x);
    if (t >= p.total) break;
    const int tw = t % p.tiles_w, th = (t / p.tiles_w) % p.tiles_h, img = t / (p.tiles_w * p.tiles_h);
    const int st = j % kStages;
    mbar_wait(&empty[st], ((j / kStages) & 1) ^ 1);
    build_patch_row(p, img, th * kTH + m / kTW, tw * kTW + m % kTW, sP + st * 8192, m);
    fence_proxy_async_smem();
    mbar_arrive(&full[st]);
  }
}

__device__ __forceinline__ void load_filters(const FirstConvParams& p, uint8_t* sB) {
  for (int t = threadIdx.x; t < 64 * 4; t += blockDim.x) {
    const int r = t >> 2, c = t & 3;
    const uint4 u = *reinterpret_cast<const uint4*>(p.wf + r * 32 + c * 8);
    *reinterpret_cast<uint4*>(sB + r * 64 + ((c ^ ((r >> 1) & 3)) << 4)) = u;
  }
}

__device__ __forceinline__ void tma_load_4d_cta(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1,
                                                int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void tile_coords(const FirstConvParams& p, int t, int& img, int& y0, int& x0) {
  const int tw = t % p.tiles_w;
  t /= p.tiles_w;
  const int th = t % p.tiles_h;
  img = t / p.tiles_h;
  y0 = th * kTH;
  x0 = tw * kTW;
}

// warps 0..kProd-1: patch producers (thread = pixel); then kEpi epilogue warpgroups (thread =
// pixel = TMEM lane; local tile j goes to warpgroup j % kEpi, accumulator j % kAccs); the last:
// TMEM allocation + MMA issue.  One epilogue warpgroup capped the kernel at ~1150 cycles per
// 16 KB tile (TMEM load -> bf16 -> staging -> TMA store latency chain).
__global__ void __launch_bounds__(32 * kFwdWarps, 1) conv_first_fwd_kernel(const __grid_constant__ FirstConvParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = smem;                           // 4 KB filters
  uint8_t* sA = smem + 4096;                    // kStages x 8 KB patches
  uint8_t* sOut = sA + kStages * 8192;          // kOutBufs x 16 KB output staging
  uint64_t* a_full = reinterpret_cast<uint64_t*>(sOut + kOutBufs * 16384);
  uint64_t* a_empty = a_full + kStages;
  uint64_t* tfull = a_empty + kStages;
  uint64_t* tempty = tfull + kAccs;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + kAccs);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  pdl_wait_and_release();   // the filters are written by the previous step's update
  load_filters(p, sB);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) { mbar_init(&a_full[i], 128); mbar_init(&a_empty[i], 1); }
    for (int i = 0; i < kAccs; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 128); }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < kProd) {
    produce_tiles(p, sA, a_full, a_empty);
  } else if (warp == kMmaWarp) {
    const uint32_t idesc = umma_idesc_bf16(128, 64, false, false);
    const uint64_t b0 = umma_smem_desc(smem_u32(sB), 16, 512, 64);
    const uint64_t a0 = umma_smem_desc(smem_u32(sA), 16, 512, 64);
    int st = 0, acc = 0;
    uint32_t ph = 0, acc_ph = 0;
    for (int t = blockIdx.x; t < p.total; t += gridDim.x) {
      mbar_wait(&tempty[acc], acc_ph ^ 1);
      mbar_wait(&a_full[st], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint64_t ad = desc_add(a0, st * 8192);
        umma_bf16(tmem_base + acc * 64, ad, b0, idesc, 0u);
        umma_bf16(tmem_base + acc * 64, desc_add(ad, 32), desc_add(b0, 32), idesc, 1u);
        umma_commit(&a_empty[st]);
        umma_commit(&tfull[acc]);
      }
      __syncwarp();
      if (++st == kStages) { st = 0; ph ^= 1; }
      if (++acc == kAccs) { acc = 0; acc_ph ^= 1; }
    }
  } else {
    const int ewg = (warp - kProd) >> 2;
    const int q = warp & 3;
    const int m = q * 32 + lane;
    int acc = ewg, ob = 0;
    uint32_t acc_ph = 0;
    uint8_t* sOutW = sOut + ewg * (kOutBufs / kEpi) * 16384;   // this warpgroup's staging buffers
    for (int t = blockIdx.x + ewg * static_cast<int>(gridDim.x); t < p.total; t += kEpi * gridDim.x) {
      int img, y0, x0;
      tile_coords(p, t, img, y0, x0);
      mbar_wait(&tfull[acc], acc_ph);
      tc_fence_after();
      uint32_t rr[64];
      const uint32_t tb = tmem_base + acc * 64 + (static_cast<uint32_t>(q * 32) << 16);
      tmem_ld32(tb, *reinterpret_cast<uint32_t(*)[32]>(rr));
      tmem_ld32(tb + 32, *reinterpret_cast<uint32_t(*)[32]>(rr + 32));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      // the staging buffer written kOutBufs/kEpi tiles ago must have been read by its TMA store
      if (m == 0) bulk_wait_read<kOutBufs / kEpi - 1>();
      named_bar_sync(1 + ewg, 128);
      uint8_t* row = sOutW + ob * 16384 + m * 128;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint4 u;
        u.x = pack_bf16(fmaxf(__uint_as_float(rr[8 * c + 0]), 0.f), fmaxf(__uint_as_float(rr[8 * c + 1]), 0.f));
        u.y = pack_bf16(fmaxf(__uint_as_float(rr[8 * c + 2]), 0.f), fmaxf(__uint_as_float(rr[8 * c + 3]), 0.f));
        u.z = pack_bf16(fmaxf(__uint_as_float(rr[8 * c + 4]), 0.f), fmaxf(__uint_as_float(rr[8 * c + 5]), 0.f));
        u.w = pack_bf16(fmaxf(__uint_as_float(rr[8 * c + 6]), 0.f), fmaxf(__uint_as_float(rr[8 * c + 7]), 0.f));
        *reinterpret_cast<uint4*>(row + ((c ^ (m & 7)) << 4)) = u;
      }
      fence_proxy_async_smem();
      named_bar_sync(1 + ewg, 128);
      if (m == 0) {
        tma_store_4d(&p.tmY, sOutW + ob * 16384, 0, x0 + p.pad_out, y0 + p.pad_out, img);
        bulk_commit();
      }
      if (++ob == kOutBufs / kEpi) ob = 0;
      acc += kEpi;
      if (acc >= kAccs) { acc -= kAccs; acc_ph ^= 1; }
    }
    if (m == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

// warps 0-3: patch producers; warp 4: dY TMA; warp 5: TMEM + MMA.  Warp 0 reduces the
// accumulator into dW at the end (TMEM lanes 0-31 = patch columns).
__global__ void __launch_bounds__(32 * (kProd + 2), 1) conv_first_wgrad_kernel(const __grid_constant__ FirstConvParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sY = smem;                           // kStages x 16 KB dY tiles
  uint8_t* sP = sY + kStages * 16384;           // kStages x 8 KB patches
  uint64_t* full = reinterpret_cast<uint64_t*>(sP + kStages * 8192);
  uint64_t* empty = full + kStages;
  uint64_t* done = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tma_prefetch(&p.tmY);
    for (int i = 0; i < kStages; ++i) { mbar_init(&full[i], 129); mbar_init(&empty[i], 1); }  // 128 producers + TMA
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == kProd + 1) tmem_alloc(tmem_slot, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait_and_release();

  if (warp < kProd) {
    produce_tiles(p, sP, full, empty);
  } else if (warp == kProd) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < p.total; t += gridDim.x) {
        int img, y0, x0;
        tile_coords(p, t, img, y0, x0);
        mbar_wait(&empty[st], ph ^ 1);
        mbar_expect_tx(&full[st], 16384);
        tma_load_4d_cta(sY + st * 16384, &p.tmY, &full[st], 0, x0 + p.pad_out, y0 + p.pad_out, img);
        if (++st == kStages) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp == kProd + 1) {
    // A = patch^T: MN-major SW64 (M atoms of 32 columns; only atom 0 is real -- LBO = 0 makes
    // the other three alias it, their rows of D are ignored), K = pixels (8-row groups 512 B).
    const uint32_t idesc = umma_idesc_bf16(128, 64, true, true);
    const uint64_t a0 = umma_smem_desc(smem_u32(sP), 0, 512, 64);
    const uint64_t y0d = umma_smem_desc(smem_u32(sY), 8192, 1024, 128);
    int st = 0;
    uint32_t ph = 0;
    bool first = true;
    for (int t = blockIdx.x; t < p.total; t += gridDim.x) {
      mbar_wait(&full[st], ph);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          umma_bf16(tmem_base, desc_add(a0, st * 8192 + ks * 1024), desc_add(y0d, st * 16384 + ks * 2048), idesc,
                    (first && ks == 0) ? 0u : 1u);
        umma_commit(&empty[st]);
      }
      __syncwarp();
      first = false;
      if (++st == kStages) { st = 0; ph ^= 1; }
    }
    if (elect_one()) umma_commit(done);
    __syncwarp();
  }
  if (warp == 0 && blockIdx.x < p.total) {
    mbar_wait(done, 0);
    tc_fence_after();
    uint32_t rr[64];
    tmem_ld32(tmem_base, *reinterpret_cast<uint32_t(*)[32]>(rr));
    tmem_ld32(tmem_base + 32, *reinterpret_cast<uint32_t(*)[32]>(rr + 32));
    tmem_wait_ld();
    const int k = lane;  // patch column (27 = bias)
    if (k <= 27) {
#pragma unroll
      for (int co = 0; co < 64; ++co) red_add_f32(p.dw + co * 32 + k, __uint_as_float(rr[co]));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kProd + 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 64);
  }
}

}  // namespace

bool conv_first_ok(int h, int w, int cin, int cout, int k, int stride, int pad) {
  return k == 3 && stride == 1 && pad == 1 && cin == 3 && cout == 64 && h % kTH == 0 && w % kTW == 0;
}

static bool first_params(FirstConvParams* p, const float* img, int n, int h, int w, int cin, void* y_pad, int pad_out,
                         std::string* why) {
  std::memset(p, 0, sizeof(*p));
  p->img = img;
  p->n = n; p->h = h; p->w = w; p->cin = cin; p->pad_out = pad_out;
  p->tiles_w = w / kTW;
  p->tiles_h = h / kTH;
  p->total = n * p->tiles_w * p->tiles_h;
  return encode_act(&p->tmY, y_pad, 64, w + 2 * pad_out, h + 2 * pad_out, n, 64, kTW, kTH, 128, why);
}

cudaError_t conv_first_fwd(const float* img, int n, int h, int w, int cin, const void* wf, void* y_pad, int pad_out,
                           cudaStream_t s, std::string* why) {
  FirstConvParams p;
  if (!first_params(&p, img, n, h, w, cin, y_pad, pad_out, why)) return cudaErrorInvalidValue;
  p.wf = static_cast<const __nv_bfloat16*>(wf);
  const int smem = 1024 + 4096 + kStages * 8192 + kOutBufs * 16384 + 256;
  const int grid = std::min(p.total, num_sms());
  cudaFuncSetAttribute(conv_first_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  launch_timed([&] { static_cast<void>(launch_pdl(conv_first_fwd_kernel, dim3(grid), dim3(32 * kFwdWarps), smem, s, 1, p)); }, s, KIND_FIRST_FWD,
               2.0 * n * h * w * 27.0 * 64.0, static_cast<double>(n) * h * w * (cin * 4.0 + 64 * 2.0));
  return cudaGetLastError();
}

cudaError_t conv_first_wgrad(const float* img, int n, int h, int w, int cin, const void* dy_pad, int pad_out,
                             float* dw, cudaStream_t s, std::string* why) {
  FirstConvParams p;
  if (!first_params(&p, img, n, h, w, cin, const_cast<void*>(dy_pad), pad_out, why)) return cudaErrorInvalidValue;
  p.dw = dw;
  const int smem = 1024 + kStages * (16384 + 8192) + 256;
  const int grid = std::min(p.total, num_sms());
  cudaFuncSetAttribute(conv_first_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  launch_timed([&] { static_cast<void>(launch_pdl(conv_first_wgrad_kernel, dim3(grid), dim3(32 * (kProd + 2)), smem, s, 1, p)); }, s, KIND_FIRST_WGRAD,
               2.0 * n * h * w * 27.0 * 64.0, static_cast<double>(n) * h * w * (cin * 4.0 + 64 * 2.0));
  return cudaGetLastError();
}

}  // namespace ralpb
