// Experiment: tcgen05.mma (kind::f16, cta_group::1, SS operands) issue-to-issue throughput
// per SM for N = 64/128/256, K-major vs MN-major operands and non-canonical SBOs, with all
// 148 SMs busy.  No TMA: operands are whatever sits in shared memory.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tools/bin/exp_mma tools/exp_mma.cu -I paper_1901_05803_b200/csrc
#include <cstdio>
#include "ptx.cuh"

using namespace ralpb;

struct Cfg { int n; int a_mn; int b_mn; int a_sbo; int reps; int per_commit; int a_off; int rot; };

__global__ void __launch_bounds__(128, 1) mma_kernel(Cfg c, unsigned long long* cycles) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 160 * 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 64 * 1024);
    const uint32_t idesc = umma_idesc_bf16(128, c.n, c.a_mn, c.b_mn);
    const uint64_t ad = c.a_mn ? umma_smem_desc(a + c.a_off, 8192, 1024, 128) : umma_smem_desc(a + c.a_off, 16, c.a_sbo, 128);
    const uint64_t bd = c.b_mn ? umma_smem_desc(b, 8192, 1024, 128) : umma_smem_desc(b, 16, 1024, 128);
    uint32_t ph = 0;
    const unsigned long long t0 = clock64();
    for (int r = 0; r < c.reps; r += c.per_commit) {
      if (c.rot == 2) {
        // unrolled taps with compile-time descriptor offsets
        for (int k = 0; k < c.per_commit; k += 9) {
#pragma unroll
          for (int t = 0; t < 9; ++t) umma_bf16(tmem, ad + (((t / 3) * 10 + (t % 3)) * 128 >> 4), bd, idesc, 1u);
        }
      } else {
        for (int k = 0; k < c.per_commit; ++k) {
          // rot: cycle the A start through 9 tap shifts of a 10-wide slab (as the conv kernels do)
          const uint64_t a2 = c.rot ? ad + ((((k % 9) / 3) * 10 + (k % 3)) * 128 >> 4) : ad;
          umma_bf16(tmem, a2, bd, idesc, 1u);
        }
      }
      umma_commit(bar);
      mbar_wait(bar, ph);
      ph ^= 1;
    }
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 256); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  Cfg cases[] = {{64, 0, 0, 1280, 4608, 72, 0, 1}, {64, 0, 0, 1280, 4608, 72, 0, 2}, {128, 0, 0, 1280, 4608, 72, 0, 2},
                 {256, 0, 0, 1280, 4608, 72, 0, 2}, {256, 0, 0, 1024, 4608, 72, 0, 0}};
  for (auto& c : cases) {
    mma_kernel<<<148, 128, 170 * 1024>>>(c, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mma_kernel<<<148, 128, 170 * 1024>>>(c, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    double flops = 2.0 * 128 * c.n * 16 * c.reps * 148;
    printf("N=%3d A %s B %s SBO %4d off %4d rot %d commit/%2d: %6.1f cyc/mma (floor %3d)  %7.1f TF/s%s\n", c.n, c.a_mn ? "MN" : "K ",
           c.b_mn ? "MN" : "K ", c.a_sbo, c.a_off, c.rot, c.per_commit, double(cyc) / c.reps, 128 * c.n / 256, flops / (ms * 1e-3) / 1e12,
           cudaGetLastError() == cudaSuccess ? "" : " ERR");
  }
  return 0;
}
