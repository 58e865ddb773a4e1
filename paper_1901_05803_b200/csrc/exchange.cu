#include <algorithm>
#include <cstdlib>
#include "exchange.cuh"
#include "gemm_host.cuh"

namespace ralpb {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Last CTA to finish sets the flags.
__device__ __forceinline__ void finish_and_signal(const PeerSignal& sig, const uint32_t* value,
                                                  uint32_t* counter) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t prev = atomicAdd(counter, 1u);
    if (prev == gridDim.x * gridDim.y - 1) {
      __threadfence_system();
      for (int i = 0; i < sig.n; ++i)
        if (sig.flag[i] != nullptr) st_release_sys(sig.flag[i], *value);
      *counter = 0;  // re-arm (only this CTA touches it now)
    }
  }
}

__global__ void push_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, long long n16,
                            PeerSignal sig, const uint32_t* value, uint32_t* counter) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  // 4 independent 16-byte loads in flight per thread
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n16; i += stride) dst[i] = src[i];
  finish_and_signal(sig, value, counter);
}

static int push_ctas_per_sm() {  // RALPB_PUSH_CTAS_PER_SM (A/B knob; default 2)
  const char* e = getenv("RALPB_PUSH_CTAS_PER_SM");
  const int v = e != nullptr ? atoi(e) : 2;
  return v >= 1 && v <= 16 ? v : 2;
}

cudaError_t push_and_signal(void* dst, const void* src, long long n16, const PeerSignal& sig,
                            const uint32_t* value, uint32_t* counter, cudaStream_t s) {
  const char* legacy = getenv("RALPB_PUSH_LEGACY");
  if (legacy == nullptr || legacy[0] != '1') {
    PeerScatter sc{};
    sc.dst[0] = dst;
    sc.src[0] = src;
    sc.n = 1;
    return scatter_and_signal(sc, n16, sig, value, counter, s);
  }
  int grid = static_cast<int>(std::max<long long>(1, std::min<long long>((n16 + 511) / 512, num_sms() * 2)));
  launch_timed([&] {
    push_kernel<<<grid, 512, 0, s>>>(reinterpret_cast<uint4*>(dst), reinterpret_cast<const uint4*>(src), n16, sig,
                                     value, counter);
  }, s, KIND_PUSH, 16.0 * n16, 16.0 * n16);
  return cudaGetLastError();
}

// One launch for several destinations: blockIdx.y picks the (dst, src) pair, so the copies to
// all peers are in flight together instead of one launch (and one drain) per peer.  Each
// destination row has its own last-CTA counter (counter[blockIdx.y]) and releases its own flag
// (sig.flag[blockIdx.y] when sig.n == gridDim.y) as soon as ITS bytes are visible, so a worker
// never waits for the copies to the other peers.
__global__ void scatter_kernel(PeerScatter sc, long long n16, PeerSignal sig, const uint32_t* value,
                               uint32_t* counter) {
  uint4* __restrict__ dst = reinterpret_cast<uint4*>(sc.dst[blockIdx.y]);
  const uint4* __restrict__ src = reinterpret_cast<const uint4*>(sc.src[blockIdx.y]);
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  uint4 t[3];
#pragma unroll
  for (int k = 0; k < 3; ++k)
    if (i + k * stride < n16) t[k] = src[i + k * stride];
#pragma unroll
  for (int k = 0; k < 3; ++k)
    if (i + k * stride < n16) dst[i + k * stride] = t[k];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t* row_counter = counter + blockIdx.y;
    if (atomicAdd(row_counter, 1u) == gridDim.x - 1) {
      __threadfence_system();
      if (sig.n == static_cast<int>(gridDim.y)) {
        if (sig.flag[blockIdx.y] != nullptr) st_release_sys(sig.flag[blockIdx.y], *value);
      } else {
        for (int f = 0; f < sig.n; ++f)
          if (sig.flag[f] != nullptr) st_release_sys(sig.flag[f], *value);
      }
      *row_counter = 0;  // re-arm (only this CTA touches it now)
    }
  }
}

cudaError_t scatter_and_signal(const PeerScatter& sc, long long n16, const PeerSignal& sig, const uint32_t* value,
                               uint32_t* counter, cudaStream_t s) {
  if (sc.n < 1 || sc.n > kMaxRanks) return cudaErrorInvalidValue;
  const long long want = std::max<long long>(1, (static_cast<long long>(push_ctas_per_sm()) * num_sms() + sc.n - 1) / sc.n);
  const int gx = static_cast<int>(std::max<long long>(1, std::min<long long>((n16 + 511) / 512, want)));
  launch_timed([&] {
    scatter_kernel<<<dim3(gx, sc.n), 512, 0, s>>>(sc, n16, sig, value, counter);
  }, s, KIND_PUSH, 16.0 * n16 * sc.n, 16.0 * n16 * sc.n);
  return cudaGetLastError();
}

__global__ void signal_kernel(PeerSignal sig, const uint32_t* value) {
  __threadfence_system();
  if (threadIdx.x < sig.n && sig.flag[threadIdx.x] != nullptr) st_release_sys(sig.flag[threadIdx.x], *value);
}

__global__ void bump_kernel(uint32_t* counter) {
  const uint32_t v = *counter + 1;
  *counter = v;
  counter[-1] = v - 1;  // the previous step's value (flags "done with step t-1")
}

cudaError_t bump_counter(uint32_t* counter, cudaStream_t s) {
  bump_kernel<<<1, 1, 0, s>>>(counter);
  return cudaGetLastError();
}

cudaError_t signal_only(const PeerSignal& sig, const uint32_t* value, cudaStream_t s) {
  signal_kernel<<<1, 32, 0, s>>>(sig, value);
  return cudaGetLastError();
}

__global__ void wait_kernel(const uint32_t* flags, int n, const uint32_t* value) {
  const uint32_t target = *value;
  if (threadIdx.x < n) {
    while (ld_acquire_sys(flags + threadIdx.x) < target) {
      __nanosleep(64);
    }
  }
  __syncthreads();
  __threadfence_system();
}

cudaError_t wait_flags(const uint32_t* flags, int n, const uint32_t* value, cudaStream_t s) {
  wait_kernel<<<1, 32, 0, s>>>(flags, n, value);
  return cudaGetLastError();
}

__device__ __forceinline__ void shard_range(const ShardUpdate& u, long long b4, long long e4) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = b4 + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < e4; i += stride) {
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = 0; r < u.nranks; ++r) {
      float4 x = reinterpret_cast<const float4*>(u.grads[r])[i];
      g.x += x.x; g.y += x.y; g.z += x.z; g.w += x.w;
    }
    float4 v = reinterpret_cast<float4*>(u.momentum)[i];
    float4 p = reinterpret_cast<const float4*>(u.params[u.self])[i];
    v.x = u.mu * v.x + u.gscale * g.x; p.x -= u.lr * v.x;
    v.y = u.mu * v.y + u.gscale * g.y; p.y -= u.lr * v.y;
    v.z = u.mu * v.z + u.gscale * g.z; p.z -= u.lr * v.z;
    v.w = u.mu * v.w + u.gscale * g.w; p.w -= u.lr * v.w;
    reinterpret_cast<float4*>(u.momentum)[i] = v;
    for (int r = 0; r < u.nranks; ++r) reinterpret_cast<float4*>(u.params[r])[i] = p;
  }
}

__global__ void shard_update_kernel(ShardUpdate u, PeerSignal done, const uint32_t* value, uint32_t* counter) {
  if (u.nr > 0) {
    for (int k = 0; k < u.nr; ++k) shard_range(u, u.rb[k] / 4, u.re[k] / 4);
  } else {
    shard_range(u, u.begin / 4, u.end / 4);
  }
  finish_and_signal(done, value, counter);
}

cudaError_t shard_update(const ShardUpdate& u, const PeerSignal& done, const uint32_t* value,
                         uint32_t* counter, cudaStream_t s) {
  long long n = u.end - u.begin;
  if (u.nr > 0) {
    n = 0;
    for (int k = 0; k < u.nr; ++k) n += u.re[k] - u.rb[k];
  }
  const long long n4 = n / 4;
  int grid = static_cast<int>(std::max<long long>(1, std::min<long long>((n4 + 255) / 256, num_sms() * 4)));
  // NVLink bytes of this rank PER DIRECTION: (W-1) peer shard reads of the gradient come in, the
  // same number of bytes of updated parameters go out (both directions run concurrently, so the
  // per-direction figure is what compares with the per-direction link peak)
  const double peer_bytes = (u.nranks - 1) * static_cast<double>(n) * sizeof(float);
  launch_timed([&] { shard_update_kernel<<<grid, 256, 0, s>>>(u, done, value, counter); }, s, KIND_SHARD_UPDATE,
               peer_bytes, peer_bytes);
  return cudaGetLastError();
}

}  // namespace ralpb
