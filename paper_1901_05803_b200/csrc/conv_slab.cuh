// Slab-tiled implicit-GEMM convolution on tcgen05 (stride 1, k = 2p+1, padded NHWC).
//
// Output tiles are 2-D pixel blocks: one UMMA M-tile = 16 image rows x 8 columns
// (8-pixel groups are image-row segments).  For a channel block, ONE 3-D TMA box
// of (16*macc + k-1) x (8 + k-1) pixels ("halo slab") lands in shared memory with
// the 128B swizzle, and every tap (r, s) of the filter is the same slab seen
// through a shifted UMMA descriptor:
//     start = slab + ((16a + r) * SW + s) * row_bytes,   SBO = SW * row_bytes
// (SW = 8 + k - 1).  UMMA applies the swizzle from absolute shared-memory
// address bits, so row-granular starts and SBO = SW*row_bytes are legal
// (tools/exp_desc.cu).  This cuts operand traffic for the activation by ~k^2
// versus one TMA load per tap.
//
//   conv_slab_fwd_kernel   forward and backward-data (K-major A from the slab,
//                          K-major B = per-tap filter tiles), fused bias/ReLU or
//                          ReLU-mask epilogue, writes interior pixels only.
//   conv_slab_wgrad_kernel backward-filter: M = (tap, ci) pairs of taps read as two
//                          MN-major atoms of the same slab (LBO = tap distance),
//                          N = 64 output channels, K = pixels; one extra
//                          accumulator with an all-ones A yields the bias gradient
//                          (3x3).  5x5 filters: 13 tap pairs > 8 TMEM accumulators,
//                          so the taps split into two groups (part of the tile index;
//                          each group re-reads its pixel blocks) and db comes from dY's
//                          column sums.
#pragma once
#include "ptx.cuh"

namespace ralpb {

constexpr int kSlabMaxTaps = 25;
#ifndef RALPB_OUT_BUFS
#define RALPB_OUT_BUFS 2
#endif
constexpr int kOutBufs = RALPB_OUT_BUFS;   // 8 KB output staging boxes per epilogue warpgroup (3: -1 %, smem)
#ifndef RALPB_B_PRODUCERS
#define RALPB_B_PRODUCERS 2
#endif
constexpr int kBProducers = RALPB_B_PRODUCERS;   // warps issuing filter-tile TMA loads (3: warp 0 joins;
                                                  // measured +10 % on conv3_1 alone, -1 % per step)

struct alignas(64) SlabConvParams {
  CUtensorMap tmX;      // activation [N][Hp][Wp][C], box {kb, SW, SH, 1}
  CUtensorMap tmB;      // fwd: filters [Cout][taps*C] box {kb, BN}; wgrad: dY [N][Hp][Wp][Cout] box {64, 8, 16, 1}
  CUtensorMap tmY;      // fwd: output INTERIOR view {Cout, W, H, N} (padded strides), box {32, 8, 16, 1}, SW64
  int n, h, w, hp, wp, pad, k, taps;
  int c;                // contracted channels (fwd: input channels of the GEMM; wgrad: layer cin)
  int cout;             // output channels of the GEMM (fwd) / layer cout (wgrad)
  int kb, row_bytes;    // channels per k-block, bytes per slab row
  int sw, sh;           // slab width / height in pixels
  int macc;             // accumulators along M (16-row pixel blocks)
  int bn;
  int n_hb, n_wb, n_nt;
  int slab_stage, b_stage;   // aligned bytes per stage
  int slab_load, b_load;     // TMA bytes per stage
  int na, nb;                // ring depths (wgrad uses na only)
  int acc_bufs;
  uint32_t tmem_cols;
  uint32_t idesc;
  // fwd epilogue
  __nv_bfloat16* out;
  const float* bias;
  int relu;
  const __nv_bfloat16* mask;
  float* colsum;        // optional: += per-channel sum over pixels of the stored (bf16) output
  __nv_bfloat16* pool_out;  // optional fused 2x2/2 max pool of the stored output: [n][h/2+2pp][w/2+2pp][cout]
  int pool_pad;
  uint8_t* pool_idx;        // optional: per pooled element the window position of the first max
                            // (0..3 row-major), 255 when the max is not > 0 (ReLU: no gradient)
  // wgrad
  float* dw;
  float* db;
  int n_ci_blocks, n_co_blocks, n_splits, blocks_per_split, n_pix_blocks;
  int dbg;              // experiments: bit0 skip the epilogue, bit1 skip MMAs, bit2 skip pooled stores
  int wres;             // filters resident in smem: B stage t holds tap t, loaded once per CTA
};

// ------------------------------------------------------------------ forward / backward-data
// Template parameters fix the filter size, the k-steps per channel block and the M
// accumulators so that every UMMA descriptor in the issue loop is a base plus a
// compile-time offset (a descriptor computed at run time costs ~100+ cycles of issue
// latency per MMA; tools/exp_mma.cu).
//
// PAIR: a cluster of two CTAs issues cta_group::2 UMMAs (M = 2 x 128 pixel rows, N = bn):
// CTA r owns the pixel rows [h0 + r*16*MACC, +16*MACC) of the work item and HALF of the
// filter tile (bn/2 rows), so per MMA each SM reads its 4 KB of A and bn/2 x 32 B of B.
// Used for bn <= 128, where the single-CTA MMA is shared-memory-bound (64-channel filters:
// 6 KB per 32 cycles of math); every barrier that gates an MMA lives in CTA 0 (the issuer),
// whose producers expect both CTAs' bytes; MMA completions are multicast to both CTAs.
template <int K, int KSTEPS, int MACC, bool PAIR>
__global__ void __launch_bounds__(128 + 128 * (MACC >= 2 ? 2 : 1), 1)
    conv_slab_fwd_kernel(const __grid_constant__ SlabConvParams p) {
  constexpr int EWG = MACC >= 2 ? 2 : 1;
  constexpr int NCTA = PAIR ? 2 : 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + p.na * p.slab_stage;
  uint8_t* sOut = sB + p.nb * p.b_stage;         // EWG x 2 x 8 KB output staging (TMA store)
  uint64_t* a_full = reinterpret_cast<uint64_t*>(sOut + EWG * kOutBufs * 8192);
  uint64_t* a_empty = a_full + p.na;
  uint64_t* b_full = a_empty + p.na;
  uint64_t* b_empty = b_full + p.nb;
  uint64_t* tfull = b_empty + p.nb;
  uint64_t* tempty = tfull + 4;   // up to 4 TMEM accumulator buffers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);
  float* s_col = reinterpret_cast<float*>(tmem_slot + 4);  // [cout] when p.colsum

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (p.colsum != nullptr)
    for (int i = threadIdx.x; i < p.cout; i += blockDim.x) s_col[i] = 0.f;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.tmX);
    tma_prefetch(&p.tmB);
    for (int i = 0; i < p.na; ++i) { mbar_init(&a_full[i], 1); mbar_init(&a_empty[i], 1); }
    for (int i = 0; i < p.nb; ++i) { mbar_init(&b_full[i], 1); mbar_init(&b_empty[i], 1); }
    for (int i = 0; i < 4; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 128 * EWG * NCTA); }
    fence_barrier_init();
  }
  uint32_t rank = 0;
  if constexpr (PAIR) {
    rank = cluster_ctarank();
    if (warp == 2) tmem_alloc_pair(tmem_slot, p.tmem_cols);
    tc_fence_before();
    cluster_sync();
  } else {
    if (warp == 2) tmem_alloc(tmem_slot, p.tmem_cols);
    tc_fence_before();
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait_and_release();
  const int total = p.n * p.n_hb * p.n_wb * p.n_nt;
  const int cblks = p.c / p.kb;
  const int mrows = 16 * p.macc;
  const int w_first = PAIR ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int w_step = PAIR ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
  // barriers gating the issuer: own (single CTA) or CTA 0's (pair), as shared::cluster addresses
  auto lead = [&](uint64_t* bar) { return PAIR ? mapa_shared(smem_u32(bar), 0) : smem_u32(bar); };

  if (warp == 0 || warp == 2 || warp == 3) {
    // Producers: warp 0 streams the activation slabs, warps 2 and 3 take alternate filter
    // tiles (a TMA issue occupies its thread for hundreds of cycles; see tools/exp_tma.cu).
    if (lane == 0) {
      int as = 0, bs = 0;
      uint32_t aph = 0, bph = 0;
      int bseq = 0;
      const int bhalf = PAIR ? p.bn / 2 : p.bn;   // filter rows this CTA loads
      for (int wi = w_first; wi < total; wi += w_step) {
        int t = wi;
        const int nt = t % p.n_nt; t /= p.n_nt;
        const int wb = t % p.n_wb; t /= p.n_wb;
        const int hb = t % p.n_hb;
        const int img = t / p.n_hb;
        const int h0 = (hb * NCTA + static_cast<int>(rank)) * mrows, w0 = wb * 8;
        for (int cb = 0; cb < cblks; ++cb) {
          if (warp == 0) {
            mbar_wait(&a_empty[as], aph ^ 1);
            if (rank == 0) mbar_expect_tx(&a_full[as], NCTA * p.slab_load);
            if constexpr (PAIR)
              tma_load_4d_pair(sA + as * p.slab_stage, &p.tmX, lead(&a_full[as]), cb * p.kb, w0, h0, img);
            else
              tma_load_4d(sA + as * p.slab_stage, &p.tmX, &a_full[as], cb * p.kb, w0, h0, img);
            if (++as == p.na) { as = 0; aph ^= 1; }
            if (p.wres || kBProducers == 2) continue;   // warp 0 only streams slabs
          }
          if (p.wres) {  // whole filter bank once per CTA (single channel block, single N tile)
            if (wi == w_first)
              for (int tap = warp - 2; tap < p.taps; tap += 2) {
                if (rank == 0) mbar_expect_tx(&b_full[tap], NCTA * p.b_load);
                if constexpr (PAIR)
                  tma_load_2d_pair(sB + tap * p.b_stage, &p.tmB, lead(&b_full[tap]), tap * p.c, static_cast<int>(rank) * bhalf);
                else
                  tma_load_2d(sB + tap * p.b_stage, &p.tmB, &b_full[tap], tap * p.c, 0);
              }
            continue;
          }
          // filter tiles rotate over the producer warps (2, 3[, 0]): a TMA issue occupies its
          // thread for hundreds of cycles (tools/exp_tma.cu)
          const int pidx = warp == 0 ? 2 : warp - 2;
          for (int tap = 0; tap < p.taps; ++tap, ++bseq) {
            if (bseq % kBProducers == pidx) {
              mbar_wait(&b_empty[bs], bph ^ 1);
              if (rank == 0) mbar_expect_tx(&b_full[bs], NCTA * p.b_load);
              if constexpr (PAIR)
                tma_load_2d_pair(sB + bs * p.b_stage, &p.tmB, lead(&b_full[bs]), tap * p.c + cb * p.kb,
                                 nt * p.bn + static_cast<int>(rank) * bhalf);
              else
                tma_load_2d(sB + bs * p.b_stage, &p.tmB, &b_full[bs], tap * p.c + cb * p.kb, nt * p.bn);
            }
            if (++bs == p.nb) { bs = 0; bph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1 && rank == 0) {
    constexpr int SW = 8 + K - 1;       // slab width (pixels)
    constexpr int RB = KSTEPS * 32;     // slab row bytes
    constexpr int TAPS = K * K;
    int as = 0, bs = 0, acc = 0;
    uint32_t aph = 0, bph = 0, acc_ph = 0;
    const uint64_t a0 = umma_smem_desc(smem_u32(sA), 16, SW * RB, RB);
    const uint64_t b0 = umma_smem_desc(smem_u32(sB), 16, 8 * RB, RB);
    const bool issue = !(p.dbg & 2);
    auto commit = [&](uint64_t* bar) {
      if constexpr (PAIR) umma_commit_pair(bar, 0x3); else umma_commit(bar);
    };
    for (int wi = w_first; wi < total; wi += w_step) {
      mbar_wait(&tempty[acc], acc_ph ^ 1);
      tc_fence_after();
      const uint32_t d0 = tmem_base + acc * MACC * p.bn;
      for (int cb = 0; cb < cblks; ++cb) {
        mbar_wait(&a_full[as], aph);
        tc_fence_after();
        const uint64_t ad = desc_add(a0, as * p.slab_stage);
#pragma unroll
        for (int tap = 0; tap < TAPS; ++tap) {
          const int bst = p.wres ? tap : bs;
          mbar_wait(&b_full[bst], p.wres ? 0u : bph);
          tc_fence_after();
          const uint64_t bd = desc_add(b0, bst * p.b_stage);
          if (elect_one()) {
            if (issue) {
#pragma unroll
              for (int a = 0; a < MACC; ++a)
#pragma unroll
                for (int ks = 0; ks < KSTEPS; ++ks) {
                  const uint64_t ada = desc_add(ad, ((a * 16 + tap / K) * SW + tap % K) * RB + ks * 32);
                  const uint32_t accum = (cb > 0 || tap > 0 || ks > 0) ? 1u : 0u;
                  if constexpr (PAIR)
                    umma_bf16_pair(d0 + a * p.bn, ada, desc_add(bd, ks * 32), p.idesc, accum);
                  else
                    umma_bf16(d0 + a * p.bn, ada, desc_add(bd, ks * 32), p.idesc, accum);
                }
            }
            if (!p.wres) commit(&b_empty[bs]);
          }
          __syncwarp();
          if (!p.wres && ++bs == p.nb) { bs = 0; bph ^= 1; }
        }
        if (elect_one()) commit(&a_empty[as]);
        __syncwarp();
        if (++as == p.na) { as = 0; aph ^= 1; }
      }
      if (elect_one()) commit(&tfull[acc]);
      __syncwarp();
      if (++acc == p.acc_bufs) { acc = 0; acc_ph ^= 1; }
    }
  } else if (warp >= 4) {
    const int g = (warp - 4) >> 2;   // epilogue warpgroup
    const int q = warp & 3;          // TMEM lane quarter
    const int m = q * 32 + lane;
    int acc = 0, ob = 0;
    uint32_t acc_ph = 0;
    uint8_t* stage = sOut + g * kOutBufs * 8192;
    // ReLU-mask rows (backward-data) are fetched one 32-channel chunk ahead -- the first chunk
    // of a work item before its accumulator is waited on -- so the global-load latency hides
    // behind the MMAs / the previous chunk instead of stalling every chunk of the epilogue.
    const bool use_mask = p.mask != nullptr;
    uint4 mk[4];
    auto mask_fetch = [&](int img_, int hb_, int wb_, int nt_, int a_, int c_) {
      const int hh_ = (hb_ * NCTA + static_cast<int>(rank)) * mrows + a_ * 16 + (m >> 3);
      const int ww_ = wb_ * 8 + (m & 7);
      const int n0_ = nt_ * p.bn + c_;
      if (hh_ < p.h && ww_ < p.w && n0_ + 32 <= p.cout) {
        const uint4* mp = reinterpret_cast<const uint4*>(
            p.mask + ((static_cast<long long>(img_) * p.hp + hh_ + p.pad) * p.wp + ww_ + p.pad) * p.cout + n0_);
#pragma unroll
        for (int j = 0; j < 4; ++j) mk[j] = __ldg(mp + j);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) mk[j] = make_uint4(0u, 0u, 0u, 0u);
      }
    };
    for (int wi = w_first; wi < total; wi += w_step) {
      int t = wi;
      const int nt = t % p.n_nt; t /= p.n_nt;
      const int wb = t % p.n_wb; t /= p.n_wb;
      const int hb = t % p.n_hb;
      const int img = t / p.n_hb;
      if (use_mask) mask_fetch(img, hb, wb, nt, g, 0);
      mbar_wait(&tfull[acc], acc_ph);
      tc_fence_after();
      for (int a = g; a < p.macc; a += EWG) {
        const int h0 = (hb * NCTA + static_cast<int>(rank)) * mrows + a * 16;
        const int hh = h0 + (m >> 3);
        const int ww = wb * 8 + (m & 7);
        const bool valid = hh < p.h && ww < p.w;
        const long long orow = (static_cast<long long>(img) * p.hp + hh + p.pad) * p.wp + ww + p.pad;
        const uint32_t tb = tmem_base + (acc * p.macc + a) * p.bn + (static_cast<uint32_t>(q * 32) << 16);
        for (int c = 0; c < p.bn; c += 32) {
          uint4 cur[4];
          if (use_mask) {
#pragma unroll
            for (int j = 0; j < 4; ++j) cur[j] = mk[j];
            const int c2 = c + 32 < p.bn ? c + 32 : 0;
            const int a2 = c + 32 < p.bn ? a : a + EWG;
            if (a2 < p.macc) mask_fetch(img, hb, wb, nt, a2, c2);
          }
          uint32_t rr[32];
          tmem_ld32(tb + c, rr);
          tmem_wait_ld();
          const int n0 = nt * p.bn + c;
          if (n0 >= p.cout || (p.dbg & 1)) continue;   // warp-uniform
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[j]);
          const bool full = n0 + 32 <= p.cout;
          if (p.bias != nullptr) {
            if (full) {
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) {
                const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias + n0) + j4);
                v[4 * j4] += b4.x; v[4 * j4 + 1] += b4.y; v[4 * j4 + 2] += b4.z; v[4 * j4 + 3] += b4.w;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += n0 + j < p.cout ? __ldg(p.bias + n0 + j) : 0.f;
            }
          }
          if (p.relu) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
          }
          if (p.mask != nullptr && valid) {
            const __nv_bfloat16* mp = p.mask + orow * p.cout + n0;
            if (full) {
#pragma unroll
              for (int j4 = 0; j4 < 4; ++j4) {
                const uint4 u = cur[j4];
                const __nv_bfloat16* hb2 = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
                for (int e = 0; e < 8; ++e)
                  if (!(__bfloat162float(hb2[e]) > 0.f)) v[j4 * 8 + e] = 0.f;
              }
            } else {
              _Pragma("unroll") for (int j = 0; j < 32; ++j) if (n0 + j < p.cout)
                if (!(__bfloat162float(mp[j]) > 0.f)) v[j] = 0.f;
            }
          }
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(v[2 * j], v[2 * j + 1]);
          // stage this pixel's 32 channels (one 64-byte SW64 row: chunk j at j ^ ((m >> 1) & 3))
          // and write the 16x8-pixel x 32-channel block with one TMA store; the interior-view
          // tensor map clips rows/columns outside the image, so borders are never written
          // one barrier per box: before it, thread 0 also waits until every earlier store has
          // read its staging buffer, so the other buffer is free for the next box
          uint8_t* buf = stage + ob * 8192;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint4*>(buf + m * 64 + ((j ^ ((m >> 1) & 3)) << 4)) =
                make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          fence_proxy_async_smem();
          if (m == 0) bulk_wait_read<kOutBufs - 2>();
          named_bar_sync(1 + g, 128);
          if (m == 0) {
            tma_store_4d(&p.tmY, buf, n0, wb * 8, h0, img);
            bulk_commit();
          }
          if (++ob == kOutBufs) ob = 0;
          if (p.pool_out != nullptr) {
            // fused 2x2/2 max pool: a warp holds 4 image rows x 8 columns, so the window of an
            // (even row, even column) pixel is lanes {l, l^1, l^8, l^9}
            uint32_t mx[16];
            uint32_t ix[16];  // argmax per channel pair: position in the low byte of each 16-bit half
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const uint32_t o1 = __shfl_xor_sync(0xffffffffu, pk[j], 1);
              const uint32_t o8 = __shfl_xor_sync(0xffffffffu, pk[j], 8);
              const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&pk[j]);
              const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&o1);
              const __nv_bfloat162 c2 = *reinterpret_cast<const __nv_bfloat162*>(&o8);
              if (p.pool_idx != nullptr) {
                const uint32_t o9 = __shfl_xor_sync(0xffffffffu, pk[j], 9);
                const __nv_bfloat162 d = *reinterpret_cast<const __nv_bfloat162*>(&o9);
                const __nv_bfloat162 mm = __hmax2(__hmax2(a, b), __hmax2(c2, d));
                mx[j] = *reinterpret_cast<const uint32_t*>(&mm);
                // window positions (row-major): 0 = self, 1 = lane^1, 2 = lane^8, 3 = lane^9; first
                // max wins; 255 when the max is not > 0.  16-bit-lane masks, no conversions.
                const uint32_t ma = __heq2_mask(a, mm), mb = __heq2_mask(b, mm), mc = __heq2_mask(c2, mm);
                const uint32_t gt = __hgt2_mask(mm, __float2bfloat162_rn(0.f));
                const uint32_t B = mb & ~ma, C = mc & ~ma & ~mb, D = ~(ma | mb | mc);
                ix[j] = ((B & 0x00010001u) | (C & 0x00020002u) | (D & 0x00030003u) | (~gt & 0x00FF00FFu));
              } else {
                __nv_bfloat162 t = __hmax2(a, b);
                uint32_t tw = *reinterpret_cast<const uint32_t*>(&t);
                const uint32_t o = __shfl_xor_sync(0xffffffffu, tw, 8);
                t = __hmax2(t, *reinterpret_cast<const __nv_bfloat162*>(&o));
                mx[j] = *reinterpret_cast<const uint32_t*>(&t);
                (void)c2;
              }
            }
            if ((m & 9) == 0 && valid && p.pool_idx != nullptr) {
              const long long irow = (static_cast<long long>(img) * (p.h >> 1) + (hh >> 1)) * (p.w >> 1) + (ww >> 1);
              uint4* ip = reinterpret_cast<uint4*>(p.pool_idx + irow * p.cout + n0);
              uint32_t by[8];   // bytes of channels 4q..4q+3
#pragma unroll
              for (int q4 = 0; q4 < 8; ++q4) by[q4] = __byte_perm(ix[2 * q4], ix[2 * q4 + 1], 0x6420);
              ip[0] = make_uint4(by[0], by[1], by[2], by[3]);
              ip[1] = make_uint4(by[4], by[5], by[6], by[7]);
            }
            if ((m & 9) == 0 && valid && !(p.dbg & 4)) {
              const int ph = hh >> 1, pw = ww >> 1;
              const long long prow = (static_cast<long long>(img) * ((p.h >> 1) + 2 * p.pool_pad) + ph + p.pool_pad) *
                                         ((p.w >> 1) + 2 * p.pool_pad) + pw + p.pool_pad;
              __nv_bfloat16* po = p.pool_out + prow * p.cout + n0;
#pragma unroll
              for (int j = 0; j < 4; ++j)
                *reinterpret_cast<uint4*>(po + 8 * j) = make_uint4(mx[4 * j], mx[4 * j + 1], mx[4 * j + 2], mx[4 * j + 3]);
            }
          }
          if (p.colsum != nullptr) {
            // sum of the stored bf16 values over this warp's 32 pixels: transpose-reduce so
            // that lane l ends with channel n0 + l (31 shuffles), then one shared atomic
            float r[32];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const __nv_bfloat162 b2 = *reinterpret_cast<const __nv_bfloat162*>(&pk[j]);
              r[2 * j] = valid ? __low2float(b2) : 0.f;
              r[2 * j + 1] = valid ? __high2float(b2) : 0.f;
            }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {
              const bool up = lane & off;
#pragma unroll
              for (int j = 0; j < off; ++j) {
                const float send = up ? r[j] : r[j + off];
                const float keep = up ? r[j + off] : r[j];
                r[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
              }
            }
            if (n0 + lane < p.cout) atomicAdd(&s_col[n0 + lane], r[0]);
          }
        }
      }
      tc_fence_before();
      if constexpr (PAIR) mbar_arrive_cluster(lead(&tempty[acc])); else mbar_arrive(&tempty[acc]);
      if (++acc == p.acc_bufs) { acc = 0; acc_ph ^= 1; }
    }
    if (m == 0) bulk_wait_all();
  }
  tc_fence_before();
  if constexpr (PAIR) {
    cluster_sync();
    if (warp == 2) {
      tc_fence_after();
      tmem_dealloc_pair(tmem_base, p.tmem_cols);
    }
  } else {
    __syncthreads();
    if (warp == 2) {
      tc_fence_after();
      tmem_dealloc(tmem_base, p.tmem_cols);
    }
  }
  if (p.colsum != nullptr)
    for (int i = threadIdx.x; i < p.cout; i += blockDim.x) atomicAdd(p.colsum + i, s_col[i]);
}

// ------------------------------------------------------------------ backward-filter
// Stage = one pixel block of BH image rows x 8 columns (BH = 14 divides every VGG feature-map
// height, so blocks never straddle the image edge there): X halo slab (64 ci) + dY tile
// (64 co).  Accumulator a (0..4) holds taps (2a, 2a+1) x 64 ci; accumulator 5 holds the bias
// gradient (ones x dY) when this CTA owns ci-block 0.  Work is split stream-K style: the
// (tile, pixel-block) units are divided evenly over the persistent CTAs, and every
// contiguous run of one tile is flushed with fp32 reductions.
template <int BH, int K>
__global__ void __launch_bounds__(256, 1) conv_slab_wgrad_kernel(const __grid_constant__ SlabConvParams p) {
  constexpr int SW = 8 + K - 1;     // slab width (pixels)
  constexpr int TAPS = K * K;
  // tap-pair accumulators per pass: 3x3 -> 5 (+ the bias accumulator); 5x5 -> 8 (512 TMEM
  // columns), so the 13 tap pairs take two passes ("tap groups", part of the tile index)
  constexpr int NACC = K == 3 ? 5 : 8;
  constexpr int KSTEPS = BH / 2;    // 16-pixel K-steps per block (two 8-pixel rows each)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sOnes = smem;                           // 4 KB of bf16 ones (MN-major 2 atoms x 16 rows)
  uint8_t* sStage = smem + 4096;
  const int stage_bytes = p.slab_stage + p.b_stage;
  uint64_t* full = reinterpret_cast<uint64_t*>(sStage + p.na * stage_bytes);
  uint64_t* empty = full + p.na;
  uint64_t* tfull = empty + p.na;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4096 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sOnes)[i] = 0x3F803F80u;  // bf16 1.0 pairs
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.tmX);
    tma_prefetch(&p.tmB);
    for (int i = 0; i < p.na; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(&tfull[0], 1);
    mbar_init(&tempty[0], 128);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait_and_release();
  const int PB = p.n_pix_blocks;
  const int ngrp = p.n_splits;   // tap groups (1 for 3x3)
  const long long units = static_cast<long long>(p.n_ci_blocks) * p.n_co_blocks * ngrp * PB;
  const long long u_begin = units * blockIdx.x / gridDim.x;
  const long long u_end = units * (blockIdx.x + 1) / gridDim.x;
  const int pb_per_img = p.n_hb * p.n_wb;

  if (warp == 0) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (long long u = u_begin; u < u_end;) {
        const int tile = static_cast<int>(u / PB);
        const int pb0 = static_cast<int>(u - static_cast<long long>(tile) * PB);
        const int pb1 = static_cast<int>(u_end - u < PB - pb0 ? pb0 + (u_end - u) : PB);
        const int nb = (tile / ngrp) % p.n_co_blocks, cb = tile / ngrp / p.n_co_blocks;
        for (int pb = pb0; pb < pb1; ++pb) {
          const int img = pb / pb_per_img;
          const int rem = pb - img * pb_per_img;
          const int h0 = (rem / p.n_wb) * BH, w0 = (rem % p.n_wb) * 8;
          mbar_wait(&empty[st], ph ^ 1);
          mbar_expect_tx(&full[st], p.slab_load + p.b_load);
          uint8_t* base = sStage + st * stage_bytes;
          tma_load_4d(base, &p.tmX, &full[st], cb * 64, w0, h0, img);
          tma_load_4d(base + p.slab_stage, &p.tmB, &full[st], nb * 64, w0 + p.pad, h0 + p.pad, img);
          if (++st == p.na) { st = 0; ph ^= 1; }
        }
        u += pb1 - pb0;
      }
    }
  } else if (warp == 1) {
    int st = 0;
    uint32_t ph = 0, acc_ph = 0;
    const uint64_t ones_d = umma_smem_desc(smem_u32(sOnes), 2048, 1024, 128);
    const uint64_t x0 = umma_smem_desc(smem_u32(sStage), 0, SW * 128, 128);   // LBO set per tap pair
    const uint64_t y0 = umma_smem_desc(smem_u32(sStage) + p.slab_stage, 8192, 1024, 128);
    for (long long u = u_begin; u < u_end;) {
      const int tile = static_cast<int>(u / PB);
      const int pb0 = static_cast<int>(u - static_cast<long long>(tile) * PB);
      const int pb1 = static_cast<int>(u_end - u < PB - pb0 ? pb0 + (u_end - u) : PB);
      const bool with_bias = K == 3 && tile / p.n_co_blocks == 0 && p.db != nullptr;
      const int tbase = (tile % ngrp) * 2 * NACC;   // first tap of this tap group
      mbar_wait(&tempty[0], acc_ph ^ 1);
      tc_fence_after();
      for (int pb = pb0; pb < pb1; ++pb) {
        mbar_wait(&full[st], ph);
        tc_fence_after();
        const uint32_t soff = st * stage_bytes;
        if (elect_one()) {
#pragma unroll
          for (int a = 0; a < NACC; ++a) {
            const int t0 = tbase + 2 * a;
            if (t0 >= TAPS) break;
            const int t1 = t0 + 1 < TAPS ? t0 + 1 : t0;
            const int o0 = (t0 / K) * SW + t0 % K, o1 = (t1 / K) * SW + t1 % K;
            // LBO (bits 16..29, >>4) = distance between the two taps' atoms inside the slab
            const uint64_t xa = desc_add(x0, soff + o0 * 128) | (static_cast<uint64_t>(((o1 - o0) * 128) >> 4) << 16);
#pragma unroll
            for (int ks = 0; ks < KSTEPS; ++ks)
              umma_bf16(tmem_base + a * 64, desc_add(xa, 2 * ks * SW * 128), desc_add(y0, soff + ks * 2048), p.idesc,
                        (pb > pb0 || ks > 0) ? 1u : 0u);
          }
          if (with_bias) {
#pragma unroll
            for (int ks = 0; ks < KSTEPS; ++ks)
              umma_bf16(tmem_base + NACC * 64, ones_d, desc_add(y0, soff + ks * 2048), p.idesc,
                        (pb > pb0 || ks > 0) ? 1u : 0u);
          }
          umma_commit(&empty[st]);
        }
        __syncwarp();
        if (++st == p.na) { st = 0; ph ^= 1; }
      }
      if (elect_one()) umma_commit(&tfull[0]);
      __syncwarp();
      acc_ph ^= 1;
      u += pb1 - pb0;
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int m = q * 32 + lane;
    uint32_t acc_ph = 0;
    const long long wstride = static_cast<long long>(p.taps) * p.c;  // dW[co][tap][ci]
    for (long long u = u_begin; u < u_end;) {
      const int tile = static_cast<int>(u / PB);
      const int pb0 = static_cast<int>(u - static_cast<long long>(tile) * PB);
      const int pb1 = static_cast<int>(u_end - u < PB - pb0 ? pb0 + (u_end - u) : PB);
      const int nb = (tile / ngrp) % p.n_co_blocks, cb = tile / ngrp / p.n_co_blocks;
      const bool with_bias = K == 3 && cb == 0 && p.db != nullptr;
      const int tbase = (tile % ngrp) * 2 * NACC;
      mbar_wait(&tfull[0], acc_ph);
      tc_fence_after();
      for (int a = 0; a <= NACC; ++a) {
        if (a == NACC && !with_bias) break;
        if (a < NACC && tbase + 2 * a >= TAPS) break;
        const uint32_t tb = tmem_base + a * 64 + (static_cast<uint32_t>(q * 32) << 16);
        for (int c = 0; c < 64; c += 32) {
          uint32_t rr[32];
          tmem_ld32(tb + c, rr);
          tmem_wait_ld();
          const int co0 = nb * 64 + c;
          if (a < NACC) {
            const int tap = tbase + 2 * a + (m >> 6);
            if (tap < TAPS) {
              float* dst = p.dw + static_cast<long long>(co0) * wstride + static_cast<long long>(tap) * p.c + cb * 64 + (m & 63);
#pragma unroll
              for (int j = 0; j < 32; ++j) red_add_f32(dst + j * wstride, __uint_as_float(rr[j]));
            }
          } else if (m == 0) {
#pragma unroll
            for (int j = 0; j < 32; ++j) red_add_f32(p.db + co0 + j, __uint_as_float(rr[j]));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[0]);
      acc_ph ^= 1;
      u += pb1 - pb0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

// ------------------------------------------------------------------ backward-filter, CTA pairs
// The single-CTA kernel above issues N=64 UMMAs whose A+B shared-memory reads (6 KB per
// 128x64x16 MMA) exceed the tensor core's math time: it is smem-bound at ~55 cycles/MMA
// (profiles/r01: the smem->tensor-core pipe at 84-86 %).  Here two CTAs of a cluster issue
// cta_group::2 UMMAs of M = 256 (2 x (tap pair, 64 ci)) x N = 128 output channels: each SM
// reads its 4 KB of A plus its 2 KB half of B per MMA (48 cycles) against 64 cycles of math,
// so the pair is tensor-bound.  TMEM per SM is 128 lanes x N per accumulator, so the 9 taps
// are covered by three accumulators: CTA 1's slab is CTA 0's shifted down two rows, and
//   MMA 0: base tap (0,0), atom distance 1 px  -> CTA0 taps (0,0),(0,1)  CTA1 (2,0),(2,1)
//   MMA 1: base tap (0,2), atom distance 1 row -> CTA0 taps (0,2),(1,2)  CTA1 (2,2), -
//   MMA 2: base tap (1,0), atom distance 1 px  -> CTA0 taps (1,0),(1,1)  CTA1  -  , -
// (3 of 12 slots unused: 75 % of the pair's MMA work is useful, vs 4.5/6 x smem-bound for the
// single-CTA kernel).  The bias gradient is not formed here (the dY producers sum it).
template <int BH>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    conv_slab_wgrad_pair_kernel(const __grid_constant__ SlabConvParams p) {
  constexpr int SW = 10;
  constexpr int KSTEPS = BH / 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sStage = smem;
  const int stage_bytes = p.slab_stage + p.b_stage;
  uint64_t* full = reinterpret_cast<uint64_t*>(sStage + p.na * stage_bytes);
  uint64_t* empty = full + p.na;
  uint64_t* tfull = empty + p.na;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.tmX);
    tma_prefetch(&p.tmB);
    for (int i = 0; i < p.na; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(&tfull[0], 1);
    mbar_init(&tempty[0], 256);   // both CTAs' epilogue threads release the accumulators
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, p.tmem_cols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait_and_release();
  const int PB = p.n_pix_blocks;
  const long long units = static_cast<long long>(p.n_ci_blocks) * p.n_co_blocks * PB;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const long long u_begin = units * cid / ncl;
  const long long u_end = units * (cid + 1) / ncl;
  const int pb_per_img = p.n_hb * p.n_wb;

  if (warp == 0) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (long long u = u_begin; u < u_end;) {
        const int tile = static_cast<int>(u / PB);
        const int pb0 = static_cast<int>(u - static_cast<long long>(tile) * PB);
        const int pb1 = static_cast<int>(u_end - u < PB - pb0 ? pb0 + (u_end - u) : PB);
        const int nb = tile % p.n_co_blocks, cb = tile / p.n_co_blocks;
        for (int pb = pb0; pb < pb1; ++pb) {
          const int img = pb / pb_per_img;
          const int rem = pb - img * pb_per_img;
          const int h0 = (rem / p.n_wb) * BH, w0 = (rem % p.n_wb) * 8;
          mbar_wait(&empty[st], ph ^ 1);
          if (rank == 0) mbar_expect_tx(&full[st], 2 * (p.slab_load + p.b_load));
          const uint32_t bar0 = mapa_shared(smem_u32(&full[st]), 0);
          uint8_t* base = sStage + st * stage_bytes;
          tma_load_4d_pair(base, &p.tmX, bar0, cb * 64, w0, h0 + 2 * static_cast<int>(rank), img);
          tma_load_4d_pair(base + p.slab_stage, &p.tmB, bar0, nb * 128 + 64 * static_cast<int>(rank), w0 + p.pad,
                           h0 + p.pad, img);
          if (++st == p.na) { st = 0; ph ^= 1; }
        }
        u += pb1 - pb0;
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      int st = 0;
      uint32_t ph = 0, acc_ph = 0;
      const uint64_t x0 = umma_smem_desc(smem_u32(sStage), 0, SW * 128, 128);
      const uint64_t y0 = umma_smem_desc(smem_u32(sStage) + p.slab_stage, 8192, 1024, 128);
      for (long long u = u_begin; u < u_end;) {
        const int tile = static_cast<int>(u / PB);
        const int pb0 = static_cast<int>(u - static_cast<long long>(tile) * PB);
        const int pb1 = static_cast<int>(u_end - u < PB - pb0 ? pb0 + (u_end - u) : PB);
        mbar_wait(&tempty[0], acc_ph ^ 1);
        tc_fence_after();
        for (int pb = pb0; pb < pb1; ++pb) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          const uint32_t soff = st * stage_bytes;
          if (elect_one()) {
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              const int o0 = j == 0 ? 0 : j == 1 ? 2 : SW;        // base tap offset (pixels)
              const int lbo = j == 1 ? SW * 128 : 128;             // second atom's distance
              const uint64_t xa = desc_add(x0, soff + o0 * 128) | (static_cast<uint64_t>(lbo >> 4) << 16);
#pragma unroll
              for (int ks = 0; ks < KSTEPS; ++ks)
                umma_bf16_pair(tmem_base + j * 128, desc_add(xa, 2 * ks * SW * 128), desc_add(y0, soff + ks * 2048),
                               p.idesc, (pb > pb0 || ks > 0) ? 1u : 0u);
            }
            umma_commit_pair(&empty[st], 0x3);
          }
          __syncwarp();
          if (++st == p.na) { st = 0; ph ^= 1; }
        }
        if (elect_one()) umma_commit_pair(&tfull[0], 0x3);
        __syncwarp();
        acc_ph ^= 1;
        u += pb1 - pb0;
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int m = q * 32 + lane;
    uint32_t acc_ph = 0;
    const long long wstride = static_cast<long long>(p.taps) * p.c;  // dW[co][tap][ci]
    const uint32_t tempty0 = mapa_shared(smem_u32(&tempty[0]), 0);
    // taps held by (accumulator j, row half m>>6) of this CTA; -1 = unused slot
    const int half = m >> 6;
    int tap_of[3];
    if (rank == 0) {
      tap_of[0] = half ? 1 : 0;
      tap_of[1] = half ? 5 : 2;
      tap_of[2] = half ? 4 : 3;
    } else {
      tap_of[0] = half ? 7 : 6;
      tap_of[1] = half ? -1 : 8;
      tap_of[2] = -1;
    }
    for (long long u = u_begin; u < u_end;) {
      const int tile = static_cast<int>(u / PB);
      const int pb0 = static_cast<int>(u - static_cast<long long>(tile) * PB);
      const int pb1 = static_cast<int>(u_end - u < PB - pb0 ? pb0 + (u_end - u) : PB);
      const int nb = tile % p.n_co_blocks, cb = tile / p.n_co_blocks;
      mbar_wait(&tfull[0], acc_ph);
      tc_fence_after();
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        if (rank == 1 && j == 2) break;  // warp-uniform: CTA 1's third accumulator is unused
        const int tap = tap_of[j];
        const uint32_t tb = tmem_base + j * 128 + (static_cast<uint32_t>(q * 32) << 16);
        for (int c = 0; c < 128; c += 32) {
          uint32_t rr[32];
          tmem_ld32(tb + c, rr);
          tmem_wait_ld();
          if (tap >= 0) {
            const int co0 = nb * 128 + c;
            float* dst = p.dw + static_cast<long long>(co0) * wstride + static_cast<long long>(tap) * p.c + cb * 64 + (m & 63);
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) red_add_f32(dst + jj * wstride, __uint_as_float(rr[jj]));
          }
        }
      }
      tc_fence_before();
      mbar_arrive_cluster(tempty0);
      acc_ph ^= 1;
      u += pb1 - pb0;
    }
  }
  tc_fence_before();
  cluster_sync();   // the peer's shared memory / barriers stay alive until the pair is done
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, p.tmem_cols);
  }
}

}  // namespace ralpb
