// Host-side planning for the tcgen05 GEMM engine: tensor-map encoding, tile /
// split-K choice and the persistent launch.  Internal C++ API (no torch types).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <string>
#include <utility>
#include "gemm_types.cuh"

namespace ralpb {

struct Operand2D {
  const void* ptr = nullptr;  // bf16, row-major [rows][cols] with leading dimension ld (elements)
  long long rows = 0, cols = 0, ld = 0;
};

struct GemmDesc {
  int M = 0, N = 0;
  long long K = 0;            // reduction extent: elements (K-major) or rows (MN-major)
  int a_mode = LD_K, b_mode = LD_K;
  Operand2D a, b;
  int kb = 64;                // K elements per k-block for K-major operands (16/32/64)
  int block_n = 0;            // 0 = choose
  int k_splits = 1;           // 0 = choose (split-K; only valid with EPI_F32_ATOMIC)
  // implicit conv
  int taps = 1;
  int tap_off[kMaxTaps] = {0};
  int cblks = 1;
  int a_cin = 0;
  // epilogue
  int epi = EPI_BF16;
  int relu = 0;
  void* out = nullptr;
  long long s_m = 0, s_n = 1;
  const float* bias = nullptr;
  float* sgd_mom = nullptr;
  __nv_bfloat16* sgd_bf16 = nullptr;
  float sgd_lr = 0.f, sgd_mu = 0.f;
  const void* mask = nullptr;
  long long mask_s = 0;
  const void* residual = nullptr;   // EPI_BF16: += residual[m*res_s + n] before the store (may alias out)
  long long res_s = 0;
  int border = 0;
  int img_rows = 1, wp = 1, pad = 0, h = 0, w = 0;
};

// Returns cudaSuccess or an error; on a planning error returns cudaErrorInvalidValue and
// fills *why.
cudaError_t gemm_launch(const GemmDesc& d, cudaStream_t stream, std::string* why);

int num_sms();

// Optional per-launch timing of the GEMM engine (CUDA events on the launch stream).
// Tensor-core kernel families, as reported per timed launch (ralpb_launch_rec.kind).
enum LaunchKind {
  KIND_CONV_FWD = 0,      // conv_slab_fwd_kernel, single CTA (forward and backward-data)
  KIND_CONV_FWD_PAIR = 1, // conv_slab_fwd_kernel, CTA pairs
  KIND_WGRAD_PAIR = 2,    // conv_slab_wgrad_pair_kernel
  KIND_WGRAD = 3,         // conv_slab_wgrad_kernel
  KIND_FIRST_FWD = 4,     // conv_first_fwd_kernel
  KIND_FIRST_WGRAD = 5,   // conv_first_wgrad_kernel
  KIND_GEMM = 6,          // gemm_sm100_kernel
  KIND_PUSH = 7,          // push_kernel (cut gather / act-grad scatter); "flops" = bytes moved
  KIND_SHARD_UPDATE = 8,  // shard_update_kernel (sharded-PS RS + SGD + AG); "flops" = NVLink bytes per direction
  KIND_POOL_BWD = 9,      // maxpool_bwd* (HBM-bound; "flops" = 0)
  KIND_SGD = 10,          // sgd_momentum* (HBM-bound)
};

struct GemmTimer {
  cudaEvent_t* ev = nullptr;  // 2*cap events
  int cap = 0;
  int n = 0;
  int* kind = nullptr;        // [cap]
  double* flops = nullptr;    // [cap] algorithmic FLOPs of the launch
  double* bytes = nullptr;    // [cap] algorithmic DRAM (or NVLink) bytes of the launch
  cudaStream_t* stream = nullptr;   // [cap] the launching stream
};
void set_gemm_timer(GemmTimer* t);  // thread-local; nullptr disables
GemmTimer* current_gemm_timer();

// Launch `f` (a kernel launch on stream s) bracketed by the timer's events, if armed.
template <class F>
void launch_timed(F&& f, cudaStream_t s, int kind = KIND_GEMM, double flops = 0.0, double bytes = 0.0) {
  GemmTimer* tm = current_gemm_timer();
  const bool timed = tm != nullptr && tm->n < tm->cap;
  if (timed) {
    cudaEventRecord(tm->ev[2 * tm->n], s);
    tm->kind[tm->n] = kind;
    tm->flops[tm->n] = flops;
    tm->bytes[tm->n] = bytes;
    if (tm->stream != nullptr) tm->stream[tm->n] = s;
  }
  f();
  if (timed) cudaEventRecord(tm->ev[2 * tm->n++ + 1], s);
}

// Launch with programmatic dependent launch (and an optional cluster); RALPB_PDL=0 disables the
// early launch.  The kernel must call pdl_wait_and_release() before any global memory access.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int cluster_x,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[na].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  ++na;
  if (cluster_x > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster_x;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace ralpb
