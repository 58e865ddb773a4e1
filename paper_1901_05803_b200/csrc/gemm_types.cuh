// Warp-specialised, persistent tcgen05 GEMM engine used by every dense
// contraction of the layer-placed step (conv fwd / dgrad / wgrad as implicit
// GEMMs over the padded-NHWC activation layout, FC fwd / dgrad / wgrad on the
// PS-owner GPU).
//
//   D[m, n] = sum_k A[m, k] * B[n, k]       (bf16 operands, fp32 in TMEM)
//
// Roles (384 threads): warp 0 (and 3) = TMA producers, warp 1 = MMA issuer,
// warp 2 = TMEM allocator, warps 4..11 = two epilogue warpgroups (one TMEM lane = one row).
// Accumulators are double-buffered in TMEM so the epilogue of tile i overlaps
// the main loop of tile i+1.
//
// Operand "modes" describe how a K-block of an operand tile is fetched by TMA:
//   LD_K       K-major 2-D matrix [rows][K]; box {kb, rows}
//   LD_K_CONV  K-major, rows shifted by a per-tap offset: implicit-GEMM conv
//              over the padded-flattened NHWC layout (k-block -> (tap, cblk))
//   LD_MN      MN-major 2-D matrix [K][cols]; box {atom, 64} per MN atom
//   LD_MN_CONV MN-major, M index = (tap, ci), rows shifted by the tap offset
//              (the activation operand of conv wgrad)
#pragma once
#include "ptx.cuh"

namespace ralpb {

enum LoadMode : int { LD_K = 0, LD_K_CONV = 1, LD_MN = 2, LD_MN_CONV = 3 };
// EPI_SGD: the accumulator is a parameter gradient g; the epilogue applies SGD-momentum in
// place (v = mu*v + g; p -= lr*v on out = p, sgd_mom = v) and refreshes the bf16 copy, so
// the gradient never round-trips through HBM.
enum EpiMode : int { EPI_BF16 = 0, EPI_F32 = 1, EPI_F32_ATOMIC = 2, EPI_SGD = 3 };

constexpr int kBM = 128;
constexpr int kMaxTaps = 32;
constexpr int kAStage = 128 * 128;  // 16 KB: 128 rows x 128 B (or 2 MN atoms x 64 rows)
constexpr int kEpiWarps = 8;                     // two epilogue warpgroups (warps 4..11)
constexpr int kThreads = 128 + 32 * kEpiWarps;   // + producer, MMA, TMEM-allocator warps

struct alignas(64) GemmParams {
  CUtensorMap tmA;
  CUtensorMap tmB;
  CUtensorMap tmC;          // tma_epi: output [M][N] (row stride s_m), box {32, 128}
  int tma_epi;              // 0: per-thread stores; 1: TMA store (EPI_F32 / EPI_BF16); 2: TMA reduce-add (EPI_F32_ATOMIC)
  int M, N;                 // output extent (rows of A, rows of B)
  int n_mt, n_nt, n_ks;     // tile grid (m tiles, n tiles, k splits)
  int kblocks_total;        // k-blocks over the whole K
  int kblocks_per_split;
  int block_n;              // BN (32..256)
  int kb;                   // K elements per k-block (K-major); MN-major blocks are 64 rows
  int stages;
  int producers;            // TMA-issuing warps (2, or 3 for MN-major operands)
  int b_stage_bytes;
  uint32_t idesc;
  int a_mode, b_mode;
  int a_swz, b_swz;         // swizzle row bytes (32/64/128)
  int a_bytes, b_bytes;     // TMA bytes per stage
  // implicit-conv geometry
  int cblks;                // k-blocks per tap (LD_K_CONV)
  int a_cin;                // channels per tap (LD_MN_CONV)
  int taps;
  int tap_off[kMaxTaps];    // row offset per tap in the padded-flattened layout
  // epilogue
  int epi;
  int relu;
  void* out;
  long long s_m, s_n;       // element strides of out
  const float* bias;        // per-n bias (or nullptr)
  float* sgd_mom;           // EPI_SGD: momentum (same layout as out)
  __nv_bfloat16* sgd_bf16;  // EPI_SGD: bf16 copy of the updated parameters (same layout)
  float sgd_lr, sgd_mu;
  const __nv_bfloat16* mask;  // relu-backward mask source (mask[m*mask_s + n] > 0), or nullptr
  long long mask_s;
  const __nv_bfloat16* residual;  // EPI_BF16: out = acc + residual[m*res_s + n] (may alias out), or nullptr
  long long res_s;
  int border;               // zero rows that are padding positions of the padded layout
  int img_rows, wp, pad, h, w;
};

}  // namespace ralpb
