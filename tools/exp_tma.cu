// Experiment: per-SM TMA streaming throughput for the box shapes the step uses.
// 148 persistent CTAs; warp 0 lane 0 issues TMA loads into an S-stage ring, warp 1 lane 0
// waits for each stage and releases it immediately (no MMA).  Reports GB/s chip-wide.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tools/bin/exp_tma tools/exp_tma.cu -I paper_1901_05803_b200/csrc
#include <cstdio>
#include <cudaTypedefs.h>
#include "ptx.cuh"

using namespace ralpb;

__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
               ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}

struct Cfg {
  int mode;            // 0 = 2-D box, 1 = 4-D box
  int stages, stage_bytes, load_bytes, boxes_per_stage;
  int iters;           // stages per CTA
  int producers;       // producer warps (stage st is issued by warp st % producers)
  int prefetch;
  int rows, cols;      // 2-D tensor
  int box_rows;
  int n, hp, wp, c, bw, bh;  // 4-D tensor
};

__global__ void __launch_bounds__(192, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, Cfg cfg) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + cfg.stages * cfg.stage_bytes);
  uint64_t* empty = full + cfg.stages;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < cfg.stages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  // prefetch field reused: 0 = producers are warps 1..P (lane 0 each), 1 = producers are lanes 0..P-1 of warp 1
  const bool is_prod = cfg.prefetch ? (warp == 1 && lane < cfg.producers) : (warp >= 1 && warp <= cfg.producers && lane == 0);
  if (is_prod) {
    const int me = cfg.prefetch ? lane : warp - 1;
    int st = 0; uint32_t ph = 0;
    unsigned seed = blockIdx.x * 7919u + 17u + me * 31u;
    for (int it = 0; it < cfg.iters; ++it) {
      const bool mine = (st % cfg.producers) == me;
      if (!mine) { if (++st == cfg.stages) { st = 0; ph ^= 1; } continue; }
      mbar_wait(&empty[st], ph ^ 1);
      mbar_expect_tx(&full[st], cfg.load_bytes);
      for (int b = 0; b < cfg.boxes_per_stage; ++b) {
        seed = seed * 1664525u + 1013904223u;
        uint8_t* dst = smem + st * cfg.stage_bytes + b * (cfg.load_bytes / cfg.boxes_per_stage);
        if (cfg.mode == 0) {
          int row = (seed >> 8) % (cfg.rows / cfg.box_rows) * cfg.box_rows;
          tma_load_2d(dst, &tm, &full[st], 0, row);
        } else {
          int img = (seed >> 8) % cfg.n;
          int h0 = (seed >> 4) % (cfg.hp - cfg.bh);
          int w0 = ((seed >> 12) % ((cfg.wp - cfg.bw) / 8)) * 8;
          tma4(dst, &tm, &full[st], 0, w0, h0, img);
        }
      }
      if (++st == cfg.stages) { st = 0; ph ^= 1; }
    }
  } else if (warp == 0 && lane == 0) {
    int st = 0; uint32_t ph = 0;
    for (int it = 0; it < cfg.iters; ++it) {
      mbar_wait(&full[st], ph);
      mbar_arrive(&empty[st]);
      if (++st == cfg.stages) { st = 0; ph ^= 1; }
    }
  }
  __syncthreads();
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

static float run(const CUtensorMap& tm, Cfg cfg, double* gbs) {
  int smem = cfg.stages * cfg.stage_bytes + 2048;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  stream_kernel<<<148, 192, smem>>>(tm, cfg);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  stream_kernel<<<148, 192, smem>>>(tm, cfg);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  *gbs = 148.0 * cfg.iters * cfg.load_bytes / (ms * 1e-3) / 1e9;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return ms;
}

int main() {
  const long long rows = 8LL << 20;
  void* big;
  cudaMalloc(&big, rows * 128);
  cudaMemset(big, 1, rows * 128);
  for (int small = 1; small >= 1; --small) {
    long long r = small ? 4096 : rows;
    for (int box_rows : {64, 128, 256}) {
      for (int producers : {1, 2, 4, 8}) {
        for (int pf : {0, 1}) {
          CUtensorMap tm;
          cuuint64_t dims[2] = {64, (cuuint64_t)r};
          cuuint64_t strides[1] = {128};
          cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
          cuuint32_t es[2] = {1, 1};
          enc()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, big, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          Cfg cfg{};
          cfg.mode = 0; cfg.stages = 8; cfg.stage_bytes = box_rows * 128; cfg.load_bytes = box_rows * 128;
          if (cfg.stages * cfg.stage_bytes > 200 * 1024) cfg.stages = 4;
          cfg.boxes_per_stage = 1; cfg.rows = (int)r; cfg.box_rows = box_rows;
          cfg.iters = 4000 * 128 / box_rows; cfg.producers = producers; cfg.prefetch = pf;
          double gbs;
          float ms = run(tm, cfg, &gbs);
          printf("%s 2D box %3d rows, %d stages, %d producer %s: %8.1f GB/s (%.3f ms)\n", small ? "L2 " : "HBM",
                 box_rows, cfg.stages, producers, pf ? "lanes" : "warps", gbs, ms);
        }
      }
    }
  }
  return 0;
}
