// Row-streamed 3x3 convolution for 64 -> 64 channels (VGG conv1_2 forward and its
// backward-data), tcgen05 with a sliding TMEM accumulator window.
//
// With only 64 output channels the slab kernel's UMMAs are M=128 x N=64: every MMA reads a
// 4 KB A tile for 2 KB of filters and 32 cycles of math, so the tensor pipe is fed at ~60 %
// and the layer ran at ~0.75 PFLOP/s (profiles/r01: sm__pipe_tensor_cycles_active 35 %,
// tc pipe 59 %).  Here an M-tile is one image row segment of 128 pixels, and the three
// vertical taps (kr = 0, 1, 2) of a horizontal tap kc are issued as ONE UMMA with
// N = 192 = [W(0,kc) | W(1,kc) | W(2,kc)]: input row j feeds output rows j, j-1, j-2 at
// once, and their accumulators sit in adjacent 64-column TMEM slots because output row G
// (a per-CTA running row counter) lives in slot 7 - (G mod 8) -- descending, so the three
// rows of one input row are ascending columns.  Where the window wraps (slot 7 -> 0) the
// UMMA splits in two (N = 64 + 128 or 128 + 64).  An accumulator collects its three
// contributions from three different UMMAs, so no single UMMA can clear it: the epilogue
// zeroes a slot (tcgen05.st) after draining it and every UMMA accumulates.
//
//   warp 0      TMA: the 9 filter tiles once (72 KB resident), then one 130-pixel input row
//               per stage (box {64 ch, 130 px, 1, 1}, SW128; tap kc is the same row seen
//               kc pixels further -- a row-granular descriptor start)
//   warp 1      UMMA issue (one elected lane), commits "row G done" after input row G + 2
//   warps 4-11  two epilogue warpgroups, each draining pairs of output rows (2i, 2i+1):
//               bias + ReLU or ReLU-mask, bf16, TMA store (box {32 ch, 128 px}), optional
//               fused 2x2/2 max pool (horizontal pairs are lanes l, l^1; the vertical pair
//               is the row pair) and optional per-channel column sums (bias gradient).
//
// Work unit = (image, strip of output rows, 128-column block); the last column block of a
// row is shifted left to end at the image edge (224 = 128 + 96: 32 columns are computed
// twice, identical values; column sums count them once).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include "conv.cuh"
#include "gemm_host.cuh"
#include "ptx.cuh"

namespace ralpb {

namespace {

constexpr int kRowPx = 128;                 // pixels per M tile (one row segment)
constexpr int kRowIn = kRowPx + 2;          // input pixels per row stage (3 horizontal taps)
constexpr int kRowStage = 17408;            // 130 x 128 B, 1 KB aligned
constexpr int kTapBytes = 64 * 128;         // one filter tap: 64 out x 64 in bf16
constexpr int kRowThreads = 384;
// CTA-pair filter layout (per horizontal tap kc, 40 KB): every UMMA shape the issue loop
// uses -- N = 192 (kr 0-2), 128 (kr 0-1 or 1-2), 64 (one kr) -- has its own region at the
// same offset in both CTAs, holding the half of its N filter rows that CTA supplies.
constexpr int kPairKcBytes = 40960;
__host__ __device__ constexpr int pair_region(int lo, int cnt) {
  return cnt == 3 ? 0 : cnt == 2 ? (lo == 0 ? 12288 : 20480) : 28672 + lo * 4096;
}

struct alignas(64) RowConvParams {
  CUtensorMap tmX;    // padded input [n][hp][wp][64], box {64, 130, 1, 1}, SW128
  CUtensorMap tmW;    // filters [64][9 * 64], box {64, 64}, SW128
  CUtensorMap tmY;    // output interior view, box {32, 128, 1, 1}, SW64
  int n, h, w, hp, wp;
  int rows;           // output rows per strip (even)
  int n_strips, n_cb, total;
  const float* bias;
  int relu;
  const __nv_bfloat16* mask;   // padded [n][hp][wp][64] (backward-data ReLU mask)
  float* colsum;               // optional += per-channel sum of the stored values
  __nv_bfloat16* pool_out;     // optional fused 2x2/2 max pool, [n][h/2+2pp][w/2+2pp][64]
  int pool_pad;
};

__device__ __forceinline__ void tmem_st32_zero(uint32_t taddr) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(0u)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ int row_slot(int g) { return 7 - (g & 7); }

struct RowUnit {
  int img, r0, rows, x0, cb;
};

// single CTA: unit = (image, strip, column block); CTA pair: unit = (image, strip) and CTA r
// takes column block r (n_cb == 2)
template <bool PAIR>
__device__ __forceinline__ RowUnit row_unit(const RowConvParams& p, int u, uint32_t rank) {
  RowUnit r;
  r.cb = PAIR ? static_cast<int>(rank) : u % p.n_cb;
  const int t = PAIR ? u : u / p.n_cb;
  const int strip = t % p.n_strips;
  r.img = t / p.n_strips;
  r.r0 = strip * p.rows;
  r.rows = min(p.rows, p.h - r.r0);
  r.x0 = r.cb == p.n_cb - 1 ? p.w - kRowPx : r.cb * kRowPx;
  return r;
}

template <bool PAIR>
__global__ void __launch_bounds__(kRowThreads, 1) conv_row64_kernel(const __grid_constant__ RowConvParams p) {
  constexpr int kRowStages = PAIR ? 4 : 5;
  constexpr int NCTA = PAIR ? 2 : 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = smem;                              // single: 9 taps ordered (kc, kr); pair: 3 x 40 KB
  uint8_t* sA = sB + (PAIR ? 3 * kPairKcBytes : 9 * kTapBytes);   // kRowStages input rows
  uint8_t* sOut = sA + kRowStages * kRowStage;     // 2 warpgroups x 2 x 8 KB staging
  uint64_t* a_full = reinterpret_cast<uint64_t*>(sOut + 2 * 2 * 8192);
  uint64_t* a_empty = a_full + kRowStages;
  uint64_t* tfull = a_empty + kRowStages;          // per TMEM slot
  uint64_t* tempty = tfull + 8;
  uint64_t* bfull = tempty + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
  float* s_col = reinterpret_cast<float*>(tmem_slot + 4);   // [64]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const int u_first = PAIR ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int u_step = PAIR ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
  // barriers gating the issuer: own (single CTA) or CTA 0's (pair), as shared::cluster addresses
  auto lead = [&](uint64_t* bar) { return PAIR ? mapa_shared(smem_u32(bar), 0) : smem_u32(bar); };
  if (threadIdx.x < 64) s_col[threadIdx.x] = 0.f;
  if (threadIdx.x == 0) {
    tma_prefetch(&p.tmX);
    tma_prefetch(&p.tmW);
    tma_prefetch(&p.tmY);
    for (int i = 0; i < kRowStages; ++i) { mbar_init(&a_full[i], 1); mbar_init(&a_empty[i], 1); }
    for (int i = 0; i < 8; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 128 * NCTA); }
    mbar_init(bfull, 1);
    fence_barrier_init();
  }
  if constexpr (PAIR) {
    if (warp == 2) tmem_alloc_pair(tmem_slot, 512);
    tc_fence_before();
    cluster_sync();
  } else {
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (warp >= 4) {   // every slot starts at zero (UMMAs always accumulate)
    const int wg = (warp - 4) >> 2, q = warp & 3;
    const uint32_t lanes = static_cast<uint32_t>(q * 32) << 16;
    for (int c = wg * 256; c < wg * 256 + 256; c += 32) tmem_st32_zero(tmem_base + lanes + c);
    tmem_wait_st();
  }
  pdl_wait_and_release();
  // resident filters (each CTA its own copy / half), then one barrier over the CTA (pair:
  // the cluster -- CTA 0's UMMAs read CTA 1's filters and write CTA 1's zeroed TMEM)
  if (threadIdx.x == 0) {
    if constexpr (PAIR) {
      mbar_expect_tx(bfull, 3 * kPairKcBytes);
      auto chunk = [&](int kc, int off, int kr, int half) {
        tma_load_2d(sB + kc * kPairKcBytes + off, &p.tmW, bfull, (kr * 3 + kc) * 64, half * 32);
      };
      const int r = static_cast<int>(rank);
      for (int kc = 0; kc < 3; ++kc) {
        // N=192: rows [W0; W1lo] | [W1hi; W2]
        if (r == 0) { chunk(kc, 0, 0, 0); chunk(kc, 4096, 0, 1); chunk(kc, 8192, 1, 0); }
        else        { chunk(kc, 0, 1, 1); chunk(kc, 4096, 2, 0); chunk(kc, 8192, 2, 1); }
        // N=128 kr 0-1: W0 | W1; kr 1-2: W1 | W2
        chunk(kc, pair_region(0, 2), r, 0); chunk(kc, pair_region(0, 2) + 4096, r, 1);
        chunk(kc, pair_region(1, 2), 1 + r, 0); chunk(kc, pair_region(1, 2) + 4096, 1 + r, 1);
        // N=64: Wkr rows [32r, 32r + 32)
        for (int kr = 0; kr < 3; ++kr) chunk(kc, pair_region(kr, 1), kr, r);
      }
    } else {
      mbar_expect_tx(bfull, 9 * kTapBytes);
      for (int kc = 0; kc < 3; ++kc)
        for (int kr = 0; kr < 3; ++kr) {
          tma_load_2d(sB + (kc * 3 + kr) * kTapBytes, &p.tmW, bfull, (kr * 3 + kc) * 64, 0);
          tma_load_2d(sB + (kc * 3 + kr) * kTapBytes + 4096, &p.tmW, bfull, (kr * 3 + kc) * 64, 32);
        }
    }
  }
  mbar_wait(bfull, 0);
  tc_fence_before();
  if constexpr (PAIR) cluster_sync(); else __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    if (lane == 0) {
      int as = 0;
      uint32_t aph = 0;
      for (int u = u_first; u < p.total; u += u_step) {
        const RowUnit ru = row_unit<PAIR>(p, u, rank);
        for (int j = 0; j < ru.rows + 2; ++j) {   // padded input rows r0 .. r0 + rows + 1
          mbar_wait(&a_empty[as], aph ^ 1);
          if (rank == 0) mbar_expect_tx(&a_full[as], NCTA * kRowIn * 128);
          if constexpr (PAIR)
            tma_load_4d_pair(sA + as * kRowStage, &p.tmX, lead(&a_full[as]), 0, ru.x0, ru.r0 + j, ru.img);
          else
            tma_load_4d(sA + as * kRowStage, &p.tmX, &a_full[as], 0, ru.x0, ru.r0 + j, ru.img);
          if (++as == kRowStages) { as = 0; aph ^= 1; }
        }
      }
    }
  } else if (warp == 1 && rank == 0) {
    const uint64_t a0 = umma_smem_desc(smem_u32(sA), 16, 1024, 128);
    const uint64_t b0 = umma_smem_desc(smem_u32(sB), 16, 1024, 128);
    const uint32_t idesc0 = umma_idesc_bf16(128 * NCTA, 0, false, false);   // | (N >> 3) << 17 below
    int as = 0, G = 0;
    uint32_t aph = 0;
    for (int u = u_first; u < p.total; u += u_step) {
      const int R = row_unit<PAIR>(p, u, rank).rows;
      for (int j = 0; j < R + 2; ++j) {
        const int lo = max(0, j - R + 1), hi = min(2, j);
        if (j < R && G + j >= 8) {   // first write of output row j: its slot must be drained
          const int gj = G + j;
          mbar_wait(&tempty[row_slot(gj)], ((gj >> 3) - 1) & 1);
        }
        mbar_wait(&a_full[as], aph);
        tc_fence_after();
        const uint64_t ad = desc_add(a0, as * kRowStage);
        // at most two UMMAs per (kc, k-step): taps lo .. lo+c1-1 into slots s1.., the rest
        // (c2, after the window wraps) from slot 0; everything below is per input row, so the
        // 12 x (1|2) issues use compile-time descriptor offsets only (a descriptor computed per
        // MMA costs ~100 issue cycles; tools/exp_mma.cu)
        const int s1 = row_slot(G + j - lo);
        const int c1 = min(hi - lo + 1, 8 - s1), c2 = hi - lo + 1 - c1;
        const uint32_t d1 = tmem_base + s1 * 64, d2 = tmem_base;
        const uint32_t id1 = idesc0 | (static_cast<uint32_t>(8 * c1) << 17);
        const uint32_t id2 = idesc0 | (static_cast<uint32_t>(8 * (c2 > 0 ? c2 : 1)) << 17);
        constexpr int kKcBytes = PAIR ? kPairKcBytes : 3 * kTapBytes;
        const uint64_t bd1 = desc_add(b0, PAIR ? pair_region(lo, c1) : lo * kTapBytes);
        const uint64_t bd2 = desc_add(b0, PAIR ? pair_region(lo + c1, c2 > 0 ? c2 : 1) : (lo + c1) * kTapBytes);
        if (elect_one()) {
#pragma unroll
          for (int kc = 0; kc < 3; ++kc)
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              const uint64_t ada = desc_add(ad, kc * 128 + ks * 32);
              if constexpr (PAIR) {
                umma_bf16_pair(d1, ada, desc_add(bd1, kc * kKcBytes + ks * 32), id1, 1u);
                if (c2 > 0) umma_bf16_pair(d2, ada, desc_add(bd2, kc * kKcBytes + ks * 32), id2, 1u);
              } else {
                umma_bf16(d1, ada, desc_add(bd1, kc * kKcBytes + ks * 32), id1, 1u);
                if (c2 > 0) umma_bf16(d2, ada, desc_add(bd2, kc * kKcBytes + ks * 32), id2, 1u);
              }
            }
          if constexpr (PAIR) {
            umma_commit_pair(&a_empty[as], 0x3);
            if (j >= 2) umma_commit_pair(&tfull[row_slot(G + j - 2)], 0x3);
          } else {
            umma_commit(&a_empty[as]);
            if (j >= 2) umma_commit(&tfull[row_slot(G + j - 2)]);
          }
        }
        __syncwarp();
        if (++as == kRowStages) { as = 0; aph ^= 1; }
      }
      G += R;
    }
  } else if (warp >= 4) {
    const int wg = (warp - 4) >> 2;
    const int q = warp & 3;
    const int m = q * 32 + lane;                 // pixel of the row segment = TMEM lane
    const uint32_t lanes = static_cast<uint32_t>(q * 32) << 16;
    uint8_t* stage = sOut + wg * 2 * 8192;
    int ob = 0, G = 0;
    const bool pool = p.pool_out != nullptr;
    for (int u = u_first; u < p.total; u += u_step) {
      const RowUnit ru = row_unit<PAIR>(p, u, rank);
      const bool count_col = ru.x0 + m >= ru.cb * kRowPx;   // shifted last block: count once
      for (int o = 0; o < ru.rows; o += 2) {
        if (((G + o) >> 1 & 1) != wg) continue;
        uint32_t hm[2][16];                      // pool: horizontal maxima of the even row
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int gr = G + o + rr;
          const int s = row_slot(gr);
          const int yy = ru.r0 + o + rr;
          const long long prow = (static_cast<long long>(ru.img) * p.hp + yy + 1) * p.wp + ru.x0 + m + 1;
          uint4 mk[4];
          if (p.mask != nullptr) {
            const uint4* mp = reinterpret_cast<const uint4*>(p.mask + prow * 64);
#pragma unroll
            for (int j = 0; j < 4; ++j) mk[j] = __ldg(mp + j);
          }
          mbar_wait(&tfull[s], (gr >> 3) & 1);
          tc_fence_after();
#pragma unroll
          for (int ch = 0; ch < 2; ++ch) {
            const int c0 = ch * 32;
            uint32_t r[32];
            tmem_ld32(tmem_base + lanes + s * 64 + c0, r);
            uint4 mk_next[4];
            if (p.mask != nullptr && ch == 0) {
              const uint4* mp = reinterpret_cast<const uint4*>(p.mask + prow * 64 + 32);
#pragma unroll
              for (int j = 0; j < 4; ++j) mk_next[j] = __ldg(mp + j);
            }
            tmem_wait_ld();
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
            if (p.bias != nullptr) {
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) {
                const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias + c0) + j4);
                v[4 * j4] += b4.x; v[4 * j4 + 1] += b4.y; v[4 * j4 + 2] += b4.z; v[4 * j4 + 3] += b4.w;
              }
            }
            if (p.relu) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
            }
            if (p.mask != nullptr) {
#pragma unroll
              for (int j4 = 0; j4 < 4; ++j4) {
                const __nv_bfloat16* hb2 = reinterpret_cast<const __nv_bfloat16*>(&mk[j4]);
#pragma unroll
                for (int e = 0; e < 8; ++e)
                  if (!(__bfloat162float(hb2[e]) > 0.f)) v[j4 * 8 + e] = 0.f;
              }
              if (ch == 0) {
#pragma unroll
                for (int j = 0; j < 4; ++j) mk[j] = mk_next[j];
              }
            }
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(v[2 * j], v[2 * j + 1]);
            uint8_t* buf = stage + ob * 8192;
            if (m == 0) bulk_wait_read<1>();
            named_bar_sync(1 + wg, 128);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<uint4*>(buf + m * 64 + ((j ^ ((m >> 1) & 3)) << 4)) =
                  make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
            fence_proxy_async_smem();
            named_bar_sync(1 + wg, 128);
            if (m == 0) {
              tma_store_4d(&p.tmY, buf, c0, ru.x0, yy, ru.img);
              bulk_commit();
            }
            ob ^= 1;
            if (pool) {
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const uint32_t o1 = __shfl_xor_sync(0xffffffffu, pk[j], 1);
                const __nv_bfloat162 t = __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&pk[j]),
                                                 *reinterpret_cast<const __nv_bfloat162*>(&o1));
                if (rr == 0) {
                  hm[ch][j] = *reinterpret_cast<const uint32_t*>(&t);
                } else {
                  const __nv_bfloat162 mm = __hmax2(t, *reinterpret_cast<const __nv_bfloat162*>(&hm[ch][j]));
                  hm[ch][j] = *reinterpret_cast<const uint32_t*>(&mm);
                }
              }
              if (rr == 1 && (m & 1) == 0) {
                const int ph = (ru.r0 + o) >> 1, pw = (ru.x0 + m) >> 1;
                const long long orow = (static_cast<long long>(ru.img) * ((p.h >> 1) + 2 * p.pool_pad) + ph + p.pool_pad) *
                                           ((p.w >> 1) + 2 * p.pool_pad) + pw + p.pool_pad;
                uint4* po = reinterpret_cast<uint4*>(p.pool_out + orow * 64 + c0);
#pragma unroll
                for (int j = 0; j < 4; ++j) po[j] = make_uint4(hm[ch][4 * j], hm[ch][4 * j + 1], hm[ch][4 * j + 2], hm[ch][4 * j + 3]);
              }
            }
            if (p.colsum != nullptr) {
              float cs[32];
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const __nv_bfloat162 b2 = *reinterpret_cast<const __nv_bfloat162*>(&pk[j]);
                cs[2 * j] = count_col ? __low2float(b2) : 0.f;
                cs[2 * j + 1] = count_col ? __high2float(b2) : 0.f;
              }
#pragma unroll
              for (int off = 16; off >= 1; off >>= 1) {
                const bool up = lane & off;
#pragma unroll
                for (int j = 0; j < off; ++j) {
                  const float send = up ? cs[j] : cs[j + off];
                  const float keep = up ? cs[j + off] : cs[j];
                  cs[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                }
              }
              atomicAdd(&s_col[c0 + lane], cs[0]);
            }
          }
          // drained: clear the slot for the row that reuses it and hand it back
          tmem_st32_zero(tmem_base + lanes + s * 64);
          tmem_st32_zero(tmem_base + lanes + s * 64 + 32);
          tmem_wait_st();
          tc_fence_before();
          if constexpr (PAIR) mbar_arrive_cluster(lead(&tempty[s])); else mbar_arrive(&tempty[s]);
        }
      }
      G += ru.rows;
    }
    if (m == 0) bulk_wait_all();
  }
  tc_fence_before();
  if constexpr (PAIR) {
    cluster_sync();   // the peer's barriers / TMEM stay alive until the pair is done
    if (warp == 2) {
      tc_fence_after();
      tmem_dealloc_pair(tmem_base, 512);
    }
  } else {
    __syncthreads();
    if (warp == 2) {
      tc_fence_after();
      tmem_dealloc(tmem_base, 512);
    }
  }
  if (p.colsum != nullptr && threadIdx.x < 64) atomicAdd(p.colsum + threadIdx.x, s_col[threadIdx.x]);
}

}  // namespace

bool row64_ok(const ConvGeom& g, int c, int cout, const void* pool_idx) {
  static const bool on = [] {
    const char* e = getenv("RALPB_ROW64");
    return e == nullptr || e[0] != '0';
  }();
  return on && g.k == 3 && g.pad == 1 && c == 64 && cout == 64 && g.w >= kRowPx && g.h % 2 == 0 && g.w % 2 == 0 &&
         pool_idx == nullptr && g.q() < (1LL << 31);
}

cudaError_t conv_row64_fwd(const ConvGeom& g, const void* x_pad, const void* w, const float* bias, int relu,
                           const void* mask_pad, void* y_pad, float* colsum, void* pool_out, int pool_pad,
                           cudaStream_t s, std::string* why) {
  RowConvParams p;
  std::memset(&p, 0, sizeof(p));
  p.n = g.n; p.h = g.h; p.w = g.w; p.hp = g.hp(); p.wp = g.wp();
  p.n_cb = (g.w + kRowPx - 1) / kRowPx;
  // strip height: the fewest input-row loads per wave of the persistent grid (each strip
  // re-reads 2 halo rows); rows even for the row-pair epilogue
  const int sms = num_sms();
  long long best = -1;
  for (int ns = 1; ns <= g.h / 2; ++ns) {
    const int rows = ((g.h + ns - 1) / ns + 1) & ~1;
    const int strips = (g.h + rows - 1) / rows;
    const long long units = static_cast<long long>(g.n) * p.n_cb * strips;
    const long long waves = (units + sms - 1) / sms;
    const long long cost = waves * (rows + 2);
    if (best < 0 || cost < best) { best = cost; p.rows = rows; p.n_strips = strips; }
  }
  // CTA pairs (M = 256: the two column blocks of a row; RALPB_ROW64_PAIR=1) are implemented
  // and pass the parity tests, but measured 22 % slower than single CTAs on conv1_2
  // (0.574 vs 0.471 ms forward, tools/probe_conv.py --layer 1): off by default
  const char* pe = getenv("RALPB_ROW64_PAIR");
  const bool pair = p.n_cb == 2 && pe != nullptr && pe[0] == '1';
  p.total = g.n * (pair ? 1 : p.n_cb) * p.n_strips;
  p.bias = bias;
  p.relu = relu;
  p.mask = static_cast<const __nv_bfloat16*>(mask_pad);
  p.colsum = colsum;
  p.pool_out = static_cast<__nv_bfloat16*>(pool_out);
  p.pool_pad = pool_pad;
  if (!encode_act(&p.tmX, x_pad, 64, g.wp(), g.hp(), g.n, 64, kRowIn, 1, 128, why)) return cudaErrorInvalidValue;
  if (!encode_mat(&p.tmW, w, 64, 9 * 64, 64, 32, 128, why)) return cudaErrorInvalidValue;   // 32-row boxes
  if (!encode_interior_box(&p.tmY, y_pad, 64, g.w, g.h, g.wp(), g.hp(), g.n, 1, kRowPx, 1, why))
    return cudaErrorInvalidValue;
  const double flops = 2.0 * g.n * g.h * g.w * 9.0 * 64.0 * 64.0;
  if (pair) {
    const int smem = 1024 + 3 * kPairKcBytes + 4 * kRowStage + 2 * 2 * 8192 + 1024;
    const int grid = 2 * std::min(p.total, sms / 2);
    static_cast<void>(cudaFuncSetAttribute(conv_row64_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    launch_timed([&] {
      static_cast<void>(launch_pdl(conv_row64_kernel<true>, dim3(grid), dim3(kRowThreads), smem, s, 2, p));
    }, s, KIND_CONV_FWD_PAIR, flops, slab_fwd_bytes(g, 64, 64, mask_pad != nullptr, pool_out != nullptr, false));
  } else {
    const int smem = 1024 + 9 * kTapBytes + 5 * kRowStage + 2 * 2 * 8192 + 1024;
    const int grid = std::min(p.total, sms);
    static_cast<void>(cudaFuncSetAttribute(conv_row64_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    launch_timed([&] {
      static_cast<void>(launch_pdl(conv_row64_kernel<false>, dim3(grid), dim3(kRowThreads), smem, s, 1, p));
    }, s, KIND_CONV_FWD, flops, slab_fwd_bytes(g, 64, 64, mask_pad != nullptr, pool_out != nullptr, false));
  }
  return cudaGetLastError();
}

}  // namespace ralpb
