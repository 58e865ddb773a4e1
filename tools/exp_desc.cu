// Experiment: can a UMMA shared-memory descriptor start at an arbitrary 128-byte row
// inside a 128B-swizzled tile (row shifts not multiple of 8), and can SBO be a
// non-multiple of 1024?  Answers decide whether implicit-GEMM conv taps can reuse one
// TMA-loaded slab via shifted descriptors.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o exp_desc tools/exp_desc.cu -I paper_1901_05803_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <cudaTypedefs.h>
#include <vector>
#include "ptx.cuh"

using namespace ralpb;

// A: [rows=512][64] bf16 K-major, loaded into smem as 4 boxes of 128 rows (SW128), contiguous.
// B: [64][64] bf16 K-major (identity in the first 16 columns).
// One MMA M=128 N=64 K=16: D[m][n] = sum_k Aview[m][k] * B[n][k].
__global__ void exp_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           int shift_rows, int sbo, int base_off, int a_mn, float* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                 // 64 KB
  uint8_t* sB = smem + 65536;         // 8 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536 + 8192);
  uint64_t* mbar = bar + 1;
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(mbar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(slot, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    mbar_expect_tx(bar, 65536 + 8192);
    for (int i = 0; i < 4; ++i) tma_load_2d(sA + i * 16384, &tmA, bar, 0, i * 128);
    tma_load_2d(sB, &tmB, bar, 0, 0);
    mbar_wait(bar, 0);
    tc_fence_after();
    uint32_t a_addr = smem_u32(sA) + shift_rows * 128;
    uint64_t ad = umma_smem_desc(a_addr, a_mn ? 64 * 128 : 16, sbo, 128);
    ad |= static_cast<uint64_t>(base_off & 7) << 49;
    uint64_t bd = umma_smem_desc(smem_u32(sB), 16, 1024, 128);
    uint32_t idesc = umma_idesc_bf16(128, 64, a_mn != 0, false);
    umma_bf16(tmem, ad, bd, idesc, 0);
    umma_commit(mbar);
    mbar_wait(mbar, 0);
  }
  __syncthreads();
  tc_fence_after();
  if (warp < 4) {
    uint32_t r[32];
    for (int c = 0; c < 64; c += 32) {
      tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, r);
      tmem_wait_ld();
      for (int j = 0; j < 32; ++j) out[(warp * 32 + threadIdx.x % 32) * 64 + c + j] = __uint_as_float(r[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 64);
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

static void make_map(CUtensorMap* tm, void* ptr, int rows, int cols, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  enc()(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

int main() {
  const int R = 512, C = 64;
  std::vector<__nv_bfloat16> hA(R * C), hB(64 * 64);
  // A[r][c] = r + c/64 (exact in bf16 for r < 256), unique per row; small ints
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) hA[r * C + c] = __float2bfloat16((float)((r % 256) + (c == 0 ? 0 : 0)) + (c < 16 ? c * 0 : 0));
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) hA[r * C + c] = __float2bfloat16((float)(r % 200) + (float)(c % 16) * 256.0f);
  for (int n = 0; n < 64; ++n)
    for (int k = 0; k < 64; ++k) hB[n * 64 + k] = __float2bfloat16(n == k && n < 16 ? 1.f : 0.f);
  void *dA, *dB;
  float* dO;
  cudaMalloc(&dA, R * C * 2);
  cudaMalloc(&dB, 64 * 64 * 2);
  cudaMalloc(&dO, 128 * 64 * 4);
  cudaMemcpy(dA, hA.data(), R * C * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), 64 * 64 * 2, cudaMemcpyHostToDevice);
  CUtensorMap tA, tB;
  make_map(&tA, dA, R, C, 128);
  make_map(&tB, dB, 64, 64, 64);
  cudaFuncSetAttribute(exp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  std::vector<float> o(128 * 64);
  struct Case { int shift, sbo, base; const char* what; };
  // K-major: expected D[m][n] (n<16) = A[rowof(m)][n] where rowof(m) = shift + (m/8)*(sbo/128) + m%8
  Case cases[] = {{0, 1024, 0, "k-major baseline"},  {1, 1024, 0, "shift 1, base 0"},  {1, 1024, 1, "shift 1, base 1"},
                  {3, 1024, 0, "shift 3, base 0"},   {3, 1024, 3, "shift 3, base 3"},  {8, 1024, 0, "shift 8, base 0"},
                  {9, 1024, 0, "shift 9, base 0"},   {9, 1024, 1, "shift 9, base 1"},  {0, 1280, 0, "sbo 1280"},
                  {2, 1280, 0, "shift 2 sbo 1280"},  {2, 1280, 2, "shift 2 sbo 1280 base 2"},
                  {5, 1152, 0, "shift 5 sbo 1152"}};
  for (auto& cs : cases) {
    cudaMemset(dO, 0, 128 * 64 * 4);
    exp_kernel<<<1, 128, 100 * 1024>>>(tA, tB, cs.shift, cs.sbo, cs.base, 0, dO);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: CUDA error %s\n", cs.what, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(o.data(), dO, 128 * 64 * 4, cudaMemcpyDeviceToHost);
    int bad = 0, first_bad = -1;
    for (int m = 0; m < 128; ++m) {
      int row = cs.shift + (m / 8) * (cs.sbo / 128) + m % 8;
      for (int n = 0; n < 16; ++n) {
        float want = __bfloat162float(hA[row * C + n]);
        if (o[m * 64 + n] != want) { if (first_bad < 0) first_bad = m; ++bad; }
      }
    }
    printf("%-28s : %s (%d mismatches, first bad row %d; D[0][0..2]=%g %g %g, D[9][0]=%g)\n", cs.what,
           bad ? "WRONG" : "ok", bad, first_bad, o[0], o[1], o[2], o[9 * 64]);
  }
  return 0;
}
