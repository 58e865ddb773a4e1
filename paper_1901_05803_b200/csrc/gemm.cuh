// Kernel body of the tcgen05 GEMM engine (included by gemm_host.cu only).
#pragma once
#include "gemm_types.cuh"

namespace ralpb {

__device__ __forceinline__ bool is_border_row(const GemmParams& p, int m) {
  int r = m % p.img_rows;
  int ph = r / p.wp;
  int pw = r - ph * p.wp;
  return ph < p.pad || ph >= p.h + p.pad || pw < p.pad || pw >= p.w + p.pad;
}

// Issue the TMA loads of one operand for one k-block.
__device__ __forceinline__ void load_operand(const CUtensorMap* tm, int mode, uint8_t* dst,
                                             uint64_t* bar, int tile0, int rows, int kblk,
                                             int kb, int swz, const GemmParams& p, bool is_a) {
  if (mode == LD_K) {
    tma_load_2d(dst, tm, bar, kblk * kb, tile0);
  } else if (mode == LD_K_CONV) {
    int tap = kblk / p.cblks;
    int cb = kblk - tap * p.cblks;
    tma_load_2d(dst, tm, bar, cb * kb, tile0 + p.tap_off[tap]);
  } else {
    const int atom = swz / 2;              // MN elements per swizzle atom
    const int natoms = rows / atom;
    const int atom_bytes = 64 * swz;       // 64 K-rows per block
    const int k0 = kblk * 64;
    for (int j = 0; j < natoms; ++j) {
      int mn = tile0 + j * atom;
      if (mode == LD_MN) {
        tma_load_2d(dst + j * atom_bytes, tm, bar, mn, k0);
      } else {  // LD_MN_CONV
        int tap = mn / p.a_cin;
        int ci = mn - tap * p.a_cin;
        if (tap >= p.taps) { tap = p.taps - 1; }  // rows beyond M: any valid data, never stored
        tma_load_2d(dst + j * atom_bytes, tm, bar, ci, k0 + p.tap_off[tap]);
      }
    }
  }
  (void)is_a;
}

__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int mode, int swz, int kstep) {
  if (mode == LD_K || mode == LD_K_CONV) {
    // K-major: 8-row groups of swz-byte rows; K advances 16 elements = 32 bytes inside the atom.
    return umma_smem_desc(base + kstep * 32, 16, 8 * swz, swz);
  }
  // MN-major: atoms of (swz/2 elements x 64 rows); K advances 16 rows.
  return umma_smem_desc(base + kstep * 16 * swz, 64 * swz, 8 * swz, swz);
}

__global__ void __launch_bounds__(kThreads, 1) gemm_sm100_kernel(const __grid_constant__ GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stages = p.stages;
  uint8_t* sA = smem;
  uint8_t* sB = smem + stages * kAStage;
  uint8_t* sC = sB + stages * p.b_stage_bytes;   // tma_epi: 16 KB output staging per epilogue warpgroup
  uint64_t* full = reinterpret_cast<uint64_t*>(sC + (p.tma_epi ? 2 * 16384 : 0));
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int bn = p.block_n;
  const uint32_t tmem_cols = bn * 2 <= 32 ? 32 : (bn * 2 <= 64 ? 64 : (bn * 2 <= 128 ? 128 : (bn * 2 <= 256 ? 256 : 512)));

  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.tmA);
    tma_prefetch(&p.tmB);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 32 * kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, tmem_cols);
  pdl_wait_and_release();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int total = p.n_mt * p.n_nt * p.n_ks;

  if (warp == 0 || warp == 3 || (warp == 2 && p.producers == 3)) {
    // Producer warps take k-blocks round-robin: a TMA issue keeps its thread busy for
    // hundreds of cycles (tools/exp_tma.cu), so issuing from two threads doubles the rate.  The
    // MN-major modes issue one box per swizzle atom (up to 4 + 4 per k-block): there the
    // TMEM-allocator warp joins as a third producer (backward-filter GEMMs 20-33 % faster at narrow
    // channels; issuing the atoms lane-parallel from one warp measured slower).
    const int np = p.producers;
    const int pid = warp == 0 ? 0 : (warp == 3 ? 1 : 2);
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int seq = 0;
      for (int w = blockIdx.x; w < total; w += gridDim.x) {
        int nt = w % p.n_nt;
        int t = w / p.n_nt;
        int mt = t % p.n_mt;
        int ks = t / p.n_mt;
        int kb0 = ks * p.kblocks_per_split;
        int kb1 = min(kb0 + p.kblocks_per_split, p.kblocks_total);
        for (int kk = kb0; kk < kb1; ++kk, ++seq) {
          if (seq % np != pid) {
            if (++stage == stages) { stage = 0; phase ^= 1; }
            continue;
          }
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], p.a_bytes + p.b_bytes);
          load_operand(&p.tmA, p.a_mode, sA + stage * kAStage, &full[stage], mt * kBM, kBM, kk,
                       p.kb, p.a_swz, p, true);
          load_operand(&p.tmB, p.b_mode, sB + stage * p.b_stage_bytes, &full[stage], nt * bn, bn,
                       kk, p.kb, p.b_swz, p, false);
          if (++stage == stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // Whole warp runs the loop (warp-uniform state in uniform registers), one elected lane
    // issues; descriptors are stage bases plus a per-k-step increment (no per-MMA rebuild).
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const bool a_k = p.a_mode == LD_K || p.a_mode == LD_K_CONV;
    const bool b_k = p.b_mode == LD_K || p.b_mode == LD_K_CONV;
    const int ksteps = a_k ? p.kb / 16 : 4;
    const uint64_t a0 = operand_desc(smem_u32(sA), p.a_mode, p.a_swz, 0);
    const uint64_t b0 = operand_desc(smem_u32(sB), p.b_mode, p.b_swz, 0);
    const uint32_t a_step = a_k ? 32u : 16u * p.a_swz;
    const uint32_t b_step = b_k ? 32u : 16u * p.b_swz;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      int t = w / p.n_nt;
      int ks = t / p.n_mt;
      int kb0 = ks * p.kblocks_per_split;
      int kb1 = min(kb0 + p.kblocks_per_split, p.kblocks_total);
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * bn;
      for (int kk = kb0; kk < kb1; ++kk) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint64_t ad = desc_add(a0, stage * kAStage);
        const uint64_t bd = desc_add(b0, stage * p.b_stage_bytes);
        if (elect_one()) {
          for (int s = 0; s < ksteps; ++s)
            umma_bf16(d_tmem, desc_add(ad, s * a_step), desc_add(bd, s * b_step), p.idesc,
                      (kk > kb0 || s > 0) ? 1u : 0u);
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= 4) {
    // Two epilogue warpgroups drain each accumulator: group g takes the 32-column chunks
    // c = 32 * (2j + g), with its own staging (bf16: two 8 KB boxes; fp32: one 16 KB box), named
    // barrier and TMA-issuing thread -- the narrow-K GEMMs (1x1 convolutions, K = 64..512) are
    // epilogue-bound, one warpgroup storing 128 x 256 bf16 per tile took ~3.8 us.
    const int g = (warp - 4) >> 2;
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;
    const int lead = 128 + 128 * g;
    const bool two_bufs = p.epi == EPI_BF16;
    uint8_t* sCg = sC + g * 16384;
    int acc = 0, ks_out = 0;
    uint32_t acc_phase = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      int nt = w % p.n_nt;
      int t = w / p.n_nt;
      int mt = t % p.n_mt;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int m = mt * kBM + row;
      const bool row_ok = m < p.M;
      const bool zero_row = row_ok && p.border && is_border_row(p, m);
      const uint32_t t_base = tmem_base + acc * bn + (static_cast<uint32_t>(q * 32) << 16);
      for (int c = 32 * g; c < bn; c += 64) {
        uint32_t r[32];
        tmem_ld32(t_base + c, r);
        tmem_wait_ld();
        const int n0 = nt * bn + c;
        if (n0 >= p.N) continue;           // warp-uniform
        if (!row_ok && !p.tma_epi) continue;
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        const bool full_chunk = n0 + 32 <= p.N;
        if (p.bias != nullptr) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] += (full_chunk || n0 + j < p.N) ? __ldg(p.bias + n0 + j) : 0.f;
        }
        if (p.relu) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
        }
        if (p.mask != nullptr && row_ok) {   // (rows >= M: never stored, and past the mask's end)
          const __nv_bfloat16* mp = p.mask + static_cast<long long>(m) * p.mask_s + n0;
          if (full_chunk) {
#pragma unroll
            for (int j4 = 0; j4 < 4; ++j4) {
              uint4 u = *reinterpret_cast<const uint4*>(mp + j4 * 8);
              const __nv_bfloat16* hb = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (!(__bfloat162float(hb[e]) > 0.f)) v[j4 * 8 + e] = 0.f;
            }
          } else {
            _Pragma("unroll") for (int j = 0; j < 32; ++j) if (n0 + j < p.N)
              if (!(__bfloat162float(mp[j]) > 0.f)) v[j] = 0.f;
          }
        }
        if (p.residual != nullptr && row_ok) {   // out += residual (a gradient summed into this one)
          const __nv_bfloat16* rp = p.residual + static_cast<long long>(m) * p.res_s + n0;
          if (full_chunk) {
#pragma unroll
            for (int j4 = 0; j4 < 4; ++j4) {
              uint4 u = *reinterpret_cast<const uint4*>(rp + j4 * 8);
              const __nv_bfloat16* hb = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
              for (int e = 0; e < 8; ++e) v[j4 * 8 + e] += __bfloat162float(hb[e]);
            }
          } else {
            _Pragma("unroll") for (int j = 0; j < 32; ++j) if (n0 + j < p.N) v[j] += __bfloat162float(rp[j]);
          }
        }
        if (zero_row) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.f;
        }
        if (p.tma_epi) {
          // stage this row's 32 values (fp32: 128-byte SW128 row; bf16: 64-byte SW64 row) and
          // write the 128 x 32 block with one TMA store / reduce-add (rows >= M and columns >= N
          // are clipped by the tensor map)
          uint8_t* buf = sCg + (two_bufs ? ((ks_out & 1) << 13) : 0);
          if (threadIdx.x == lead) {
            if (two_bufs) bulk_wait_read<1>();
            else bulk_wait_read<0>();
          }
          named_bar_sync(1 + g, 128);
          if (p.epi == EPI_BF16) {
            uint8_t* rp = buf + row * 64;
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<uint4*>(rp + ((j ^ ((row >> 1) & 3)) << 4)) =
                  make_uint4(pack_bf16(v[8 * j], v[8 * j + 1]), pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                             pack_bf16(v[8 * j + 4], v[8 * j + 5]), pack_bf16(v[8 * j + 6], v[8 * j + 7]));
          } else {
            uint8_t* rp = buf + row * 128;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<float4*>(rp + ((j ^ (row & 7)) << 4)) =
                  make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          }
          fence_proxy_async_smem();
          named_bar_sync(1 + g, 128);
          if (threadIdx.x == lead) {
            if (p.tma_epi == 2) tma_reduce_add_2d(&p.tmC, buf, n0, mt * kBM);
            else tma_store_2d(&p.tmC, buf, n0, mt * kBM);
            bulk_commit();
          }
          ++ks_out;
          continue;
        }
        if (p.epi == EPI_BF16) {
          __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + m * p.s_m + n0 * p.s_n;
          if (full_chunk && p.s_n == 1) {
#pragma unroll
            for (int j4 = 0; j4 < 4; ++j4) {
              uint4 u;
              u.x = pack_bf16(v[j4 * 8 + 0], v[j4 * 8 + 1]);
              u.y = pack_bf16(v[j4 * 8 + 2], v[j4 * 8 + 3]);
              u.z = pack_bf16(v[j4 * 8 + 4], v[j4 * 8 + 5]);
              u.w = pack_bf16(v[j4 * 8 + 6], v[j4 * 8 + 7]);
              *reinterpret_cast<uint4*>(o + j4 * 8) = u;
            }
          } else {
            _Pragma("unroll") for (int j = 0; j < 32; ++j) if (n0 + j < p.N) o[j * p.s_n] = __float2bfloat16_rn(v[j]);
          }
        } else if (p.epi == EPI_F32) {
          float* o = reinterpret_cast<float*>(p.out) + m * p.s_m + n0 * p.s_n;
          if (full_chunk && p.s_n == 1) {
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4)
              *reinterpret_cast<float4*>(o + j4 * 4) =
                  make_float4(v[j4 * 4], v[j4 * 4 + 1], v[j4 * 4 + 2], v[j4 * 4 + 3]);
          } else {
            _Pragma("unroll") for (int j = 0; j < 32; ++j) if (n0 + j < p.N) o[j * p.s_n] = v[j];
          }
        } else if (p.epi == EPI_SGD) {
          const long long base = m * p.s_m + n0 * p.s_n;
          float* pp = reinterpret_cast<float*>(p.out) + base;
          float* vv = p.sgd_mom + base;
          __nv_bfloat16* bb = p.sgd_bf16 + base;
          if (full_chunk && p.s_n == 1) {
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4) {
              float4 pv = *reinterpret_cast<float4*>(pp + j4 * 4);
              float4 mv = *reinterpret_cast<float4*>(vv + j4 * 4);
              mv.x = p.sgd_mu * mv.x + v[j4 * 4 + 0]; pv.x -= p.sgd_lr * mv.x;
              mv.y = p.sgd_mu * mv.y + v[j4 * 4 + 1]; pv.y -= p.sgd_lr * mv.y;
              mv.z = p.sgd_mu * mv.z + v[j4 * 4 + 2]; pv.z -= p.sgd_lr * mv.z;
              mv.w = p.sgd_mu * mv.w + v[j4 * 4 + 3]; pv.w -= p.sgd_lr * mv.w;
              *reinterpret_cast<float4*>(pp + j4 * 4) = pv;
              *reinterpret_cast<float4*>(vv + j4 * 4) = mv;
              uint2 b2;
              b2.x = pack_bf16(pv.x, pv.y);
              b2.y = pack_bf16(pv.z, pv.w);
              *reinterpret_cast<uint2*>(bb + j4 * 4) = b2;
            }
          } else {
            _Pragma("unroll") for (int j = 0; j < 32; ++j) if (n0 + j < p.N) {
              const long long o = j * p.s_n;
              const float mv = p.sgd_mu * vv[o] + v[j];
              vv[o] = mv;
              pp[o] -= p.sgd_lr * mv;
              bb[o] = __float2bfloat16_rn(pp[o]);
            }
          }
        } else {  // EPI_F32_ATOMIC
          float* o = reinterpret_cast<float*>(p.out) + m * p.s_m + n0 * p.s_n;
          _Pragma("unroll") for (int j = 0; j < 32; ++j) if (n0 + j < p.N) red_add_f32(o + j * p.s_n, v[j]);
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (p.tma_epi && threadIdx.x == lead) bulk_wait_all();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, tmem_cols);
  }
}

}  // namespace ralpb
