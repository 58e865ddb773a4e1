// HBM-bound kernels of the bottleneck-block model (resnet.cuh).  Eight channels per thread
// (16-byte loads / stores).  The per-pixel kernels give every thread ONE fixed channel group for
// its whole life (per-channel constants -- statistics, folded scale / shift -- live in registers,
// loaded once) and walk pixels with a grid stride; pixel -> address is a multiply for unpadded
// tensors and two 32-bit divisions for padded ones (every tensor here has < 2^31 pixels).
// Reductions: registers, then shared memory, then one global atomic per channel per block.
#include <algorithm>
#include "gemm_host.cuh"
#include "resnet.cuh"

namespace ralpb {

namespace {

using bf16 = __nv_bfloat16;

int grid_for(long long work, int threads) {
  const long long blocks = (work + threads - 1) / threads;
  const long long cap = static_cast<long long>(num_sms()) * 8;
  return static_cast<int>(std::max<long long>(1, std::min(blocks, cap)));
}

// element offset of pixel p (= (img*h + y)*w + x over the interior grid) in a tensor with border pad
__device__ __forceinline__ long long toff(int p, int hw, int h, int w, int pad, int c) {
  if (pad == 0) return static_cast<long long>(p) * c;
  const int img = p / hw;
  const int r = p - img * hw;
  const int y = r / w, x = r - y * w;
  return (static_cast<long long>(img * (h + 2 * pad) + y + pad) * (w + 2 * pad) + x + pad) * c;
}

// pixel stride (elements) of a tensor: its own channel count unless it is a channel slice
template <class T>
__device__ __forceinline__ int ld_of(const T& t, int c) { return t.ld ? t.ld : c; }

__device__ __forceinline__ void load8(const bf16* p, float* v) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const bf16* b = reinterpret_cast<const bf16*>(&u);
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = __bfloat162float(b[j]);
}
__device__ __forceinline__ uint4 ld16(const bf16* p) { return *reinterpret_cast<const uint4*>(p); }
__device__ __forceinline__ float elem(const uint4& u, int j) {   // j: compile-time after unrolling
  const uint32_t w = j < 2 ? u.x : j < 4 ? u.y : j < 6 ? u.z : u.w;
  return __uint_as_float((j & 1) ? (w & 0xffff0000u) : (w << 16));
}
__device__ __forceinline__ void store8(bf16* p, const float* v) {
  uint4 u;
  bf16* b = reinterpret_cast<bf16*>(&u);
#pragma unroll
  for (int j = 0; j < 8; ++j) b[j] = __float2bfloat16_rn(v[j]);
  *reinterpret_cast<uint4*>(p) = u;
}

// Thread geometry of the per-pixel kernels: blockDim.x = lanes * groups (groups = c/8 <= 256),
// thread = (pixel lane, channel group g).
struct Lane {
  int g, lane, lanes;
  __device__ __forceinline__ explicit Lane(int c) {
    const int groups = c >> 3;
    lanes = blockDim.x / groups;
    g = threadIdx.x % groups;
    lane = threadIdx.x / groups;
  }
  __device__ __forceinline__ bool active() const { return lane < lanes; }
  __device__ __forceinline__ int first() const { return blockIdx.x * lanes + lane; }
  __device__ __forceinline__ int stride() const { return gridDim.x * lanes; }
};

// ------------------------------------------------------------------ batch norm statistics
constexpr int kU = 4;   // pixels in flight per thread in the reductions

// The reduction's last block (a ticket after every block's flush) turns the sums into the result
// and zeroes the accumulators for the next reduction: no memset, no separate finishing launch.
__device__ __forceinline__ unsigned* bn_ticket(float* work) { return reinterpret_cast<unsigned*>(work + 4 * 2048); }
__device__ __forceinline__ bool bn_last_block(float* work) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(bn_ticket(work), 1u) == gridDim.x - 1;
  __syncthreads();
  if (last) __threadfence();
  return last;
}

__global__ void __launch_bounds__(256) bn_stats_kernel(Act4 x, int pixels, int h, int w, int c, float* __restrict__ sums,
                                                       float inv_m, float eps, float* __restrict__ mean,
                                                       float* __restrict__ rstd) {
  extern __shared__ float sh[];  // [2][c]
  const Lane L(c);
  for (int i = threadIdx.x; i < 2 * c; i += blockDim.x) sh[i] = 0.f;
  __syncthreads();
  float s[8] = {0.f}, q[8] = {0.f};
  if (L.active()) {
    const int hw = h * w, st = L.stride();
    for (int p0 = L.first(); p0 < pixels; p0 += kU * st) {
      uint4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int p = p0 + u * st;
        v[u] = p < pixels ? ld16(x.p + toff(p, hw, h, w, x.pad, ld_of(x, c)) + L.g * 8) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float e = elem(v[u], j);
          s[j] += e;
          q[j] += e * e;
        }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      atomicAdd(&sh[L.g * 8 + j], s[j]);
      atomicAdd(&sh[c + L.g * 8 + j], q[j]);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * c; i += blockDim.x) atomicAdd(sums + i, sh[i]);
  if (!bn_last_block(sums)) return;
  for (int i = threadIdx.x; i < c; i += blockDim.x) {
    const float m = __ldcg(sums + i) * inv_m;
    const float var = fmaxf(__ldcg(sums + c + i) * inv_m - m * m, 0.f);
    mean[i] = m;
    rstd[i] = rsqrtf(var + eps);
    sums[i] = 0.f;
    sums[c + i] = 0.f;
  }
  if (threadIdx.x == 0) *bn_ticket(sums) = 0u;
}

// ------------------------------------------------------------------ apply
// y = act(x * sc + sh [+ r or r * rsc + rsh]), sc = rstd * gamma, sh = beta - mean * sc
__global__ void __launch_bounds__(256, 3) bn_apply_kernel(BnApply a, int pixels) {
  const Lane L(a.c);
  if (!L.active()) return;
  float sc[8], sf[8], rsc[8], rsf[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int ch = L.g * 8 + j;
    sc[j] = a.rstd[ch] * a.gamma[ch];
    sf[j] = a.beta[ch] - a.mean[ch] * sc[j];
    rsc[j] = 1.f;
    rsf[j] = 0.f;
    if (a.res_kind == 2) {
      rsc[j] = a.r_rstd[ch] * a.r_gamma[ch];
      rsf[j] = a.r_beta[ch] - a.r_mean[ch] * rsc[j];
    }
  }
  const int hw = a.h * a.w, st = L.stride();
  for (int p0 = L.first(); p0 < pixels; p0 += 2 * st) {
    uint4 v[2], r[2] = {};
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int p = p0 + u * st;
      if (p < pixels) {
        v[u] = ld16(a.x.p + toff(p, hw, a.h, a.w, a.x.pad, ld_of(a.x, a.c)) + L.g * 8);
        if (a.res_kind != 0) r[u] = ld16(a.r.p + toff(p, hw, a.h, a.w, a.r.pad, ld_of(a.r, a.c)) + L.g * 8);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int p = p0 + u * st;
      if (p >= pixels) break;
      float o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        o[j] = fmaf(elem(v[u], j), sc[j], sf[j]);
        if (a.res_kind != 0) o[j] += fmaf(elem(r[u], j), rsc[j], rsf[j]);
        if (a.relu) o[j] = fmaxf(o[j], 0.f);
      }
      store8(a.y.p + toff(p, hw, a.h, a.w, a.y.pad, ld_of(a.y, a.c)) + L.g * 8, o);
      if (a.mask_out != nullptr) {   // bits of the STORED (bf16) values
        uint32_t bits = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) bits |= (__bfloat162float(__float2bfloat16_rn(o[j])) > 0.f ? 1u : 0u) << j;
        a.mask_out[static_cast<long long>(p) * (a.c >> 3) + L.g] = static_cast<uint8_t>(bits);
      }
    }
  }
}

// ------------------------------------------------------------------ backward
// sums: [0, c) sum dz;  [c, 2c) sum dz * (x - mean)   (times rstd in bn_bwd_params / apply)
// The last block scales sum dz (x - mean) by rstd (-> sum dz * xhat), adds dbeta / dgamma, and
// leaves the finished pair at sums + 2 * 2048 for the apply pass.
template <bool BITS>   // BITS: the ReLU mask from mask_in bits (else from y)
__global__ void __launch_bounds__(256, 3) bn_bwd_reduce_kernel(BnBackward b, int pixels, float* __restrict__ sums) {
  extern __shared__ float sh[];  // [2][c]
  const int c = b.c;
  const Lane L(c);
  for (int i = threadIdx.x; i < 2 * c; i += blockDim.x) sh[i] = 0.f;
  __syncthreads();
  float sd[8] = {0.f}, sx[8] = {0.f}, mu[8];
  if (L.active()) {
#pragma unroll
    for (int j = 0; j < 8; ++j) mu[j] = b.mean[L.g * 8 + j];
    const int hw = b.h * b.w, st = L.stride();
    constexpr int U = BITS ? 4 : 2;
    for (int p0 = L.first(); p0 < pixels; p0 += U * st) {
      const uint4 z = make_uint4(0, 0, 0, 0), one = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
      uint4 dy[U], xv[U], y[BITS ? 1 : U];
      uint32_t mb[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int p = p0 + u * st;
        const bool in = p < pixels;
        dy[u] = in ? ld16(b.dy.p + toff(p, hw, b.h, b.w, b.dy.pad, ld_of(b.dy, c)) + L.g * 8) : z;
        xv[u] = in ? ld16(b.x.p + toff(p, hw, b.h, b.w, b.x.pad, ld_of(b.x, c)) + L.g * 8) : z;
        if constexpr (BITS) {
          mb[u] = in && b.relu_mask ? b.mask_in[static_cast<long long>(p) * (c >> 3) + L.g] : 0xFFu;
        } else {
          y[u] = in && b.relu_mask ? ld16(b.y.p + toff(p, hw, b.h, b.w, b.y.pad, ld_of(b.y, c)) + L.g * 8) : one;
          mb[u] = 0xFFu;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const bool live = BITS ? ((mb[u] >> j) & 1u) != 0 : elem(y[BITS ? 0 : u], j) > 0.f;
          const float d = live ? elem(dy[u], j) : 0.f;   // dy is 0 past the end
          sd[j] += d;
          sx[j] += d * (elem(xv[u], j) - mu[j]);
        }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      atomicAdd(&sh[L.g * 8 + j], sd[j]);
      atomicAdd(&sh[c + L.g * 8 + j], sx[j]);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * c; i += blockDim.x) atomicAdd(sums + i, sh[i]);
  if (!bn_last_block(sums)) return;
  float* fin = sums + 2 * 2048;
  for (int i = threadIdx.x; i < c; i += blockDim.x) {
    const float sd = __ldcg(sums + i);
    const float sx = __ldcg(sums + c + i) * b.rstd[i];   // -> sum dz * xhat
    fin[i] = sd;
    fin[c + i] = sx;
    b.dbeta[i] += sd;
    b.dgamma[i] += sx;
    sums[i] = 0.f;
    sums[c + i] = 0.f;
  }
  if (threadIdx.x == 0) *bn_ticket(sums) = 0u;
}

// dx = A * dz + (x - mean) * B + C,  A = gamma * rstd, B = -A * rstd * sum(dz xhat) / M,
// C = -A * sum(dz) / M
__global__ void __launch_bounds__(256) bn_bwd_apply_kernel(BnBackward b, int pixels, const float* __restrict__ sums,
                                                           float inv_m) {
  const int c = b.c;
  const Lane L(c);
  if (!L.active()) return;
  float A[8], B[8], C[8], mu[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int ch = L.g * 8 + j;
    const float r = b.rstd[ch];
    A[j] = b.gamma[ch] * r;
    B[j] = -A[j] * r * sums[c + ch] * inv_m;
    C[j] = -A[j] * sums[ch] * inv_m;
    mu[j] = b.mean[ch];
  }
  const int hw = b.h * b.w, st = L.stride();
  for (int p = L.first(); p < pixels; p += st) {
    float dy[8], xv[8], y[8], dx[8];
    load8(b.dy.p + toff(p, hw, b.h, b.w, b.dy.pad, ld_of(b.dy, c)) + L.g * 8, dy);
    load8(b.x.p + toff(p, hw, b.h, b.w, b.x.pad, ld_of(b.x, c)) + L.g * 8, xv);
    if (b.relu_mask && b.mask_in != nullptr) {
      const uint32_t bits = b.mask_in[static_cast<long long>(p) * (c >> 3) + L.g];
#pragma unroll
      for (int j = 0; j < 8; ++j) if (!((bits >> j) & 1u)) dy[j] = 0.f;
    } else if (b.relu_mask) {
      load8(b.y.p + toff(p, hw, b.h, b.w, b.y.pad, ld_of(b.y, c)) + L.g * 8, y);
#pragma unroll
      for (int j = 0; j < 8; ++j) if (!(y[j] > 0.f)) dy[j] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) dx[j] = fmaf(A[j], dy[j], fmaf(xv[j] - mu[j], B[j], C[j]));
    store8(b.dx.p + toff(p, hw, b.h, b.w, b.dx.pad, ld_of(b.dx, c)) + L.g * 8, dx);
    if (b.dz_out.p != nullptr) store8(b.dz_out.p + toff(p, hw, b.h, b.w, b.dz_out.pad, ld_of(b.dz_out, c)) + L.g * 8, dy);
  }
}

// ------------------------------------------------------------------ layouts
// thread = (patch row, tap, channel group); 32-bit index arithmetic
__global__ void im2col_bf16_kernel(Act4 x, int n, int h, int w, int c, int k, int st, int p, int ho, int wo,
                                   bf16* __restrict__ out) {
  const int groups = c >> 3;
  const int kk = k * k;
  const long long total = static_cast<long long>(n) * ho * wo * kk * groups;
  const int hp = h + 2 * x.pad, wp = w + 2 * x.pad;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % groups);
    const int t = static_cast<int>(i / groups);   // row * kk + tap < 2^31
    const int row = t / kk, tap = t - row * kk;
    const int img = row / (ho * wo);
    const int rr = row - img * ho * wo;
    const int oy = rr / wo, ox = rr - oy * wo;
    const int ty = tap / k;
    const int iy = oy * st + ty - p + x.pad, ix = ox * st + (tap - ty * k) - p + x.pad;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (iy >= 0 && iy < hp && ix >= 0 && ix < wp)
      v = *reinterpret_cast<const uint4*>(x.p + (static_cast<long long>(img * hp + iy) * wp + ix) * c + g * 8);
    *reinterpret_cast<uint4*>(out + static_cast<long long>(t) * c + g * 8) = v;
  }
}

__global__ void subsample_kernel(Act4 x, int n, int h, int w, int c, int st, bf16* __restrict__ out) {
  const int groups = c >> 3;
  const int ho = h / st, wo = w / st;
  const int total = n * ho * wo * groups;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int q = i / groups, g = i - q * groups;
    const int img = q / (ho * wo);
    const int r = q - img * ho * wo;
    const int oy = r / wo, ox = r - oy * wo;
    const long long src =
        (static_cast<long long>(img * (h + 2 * x.pad) + oy * st + x.pad) * (w + 2 * x.pad) + ox * st + x.pad) * c + g * 8;
    *reinterpret_cast<uint4*>(out + static_cast<long long>(q) * c + g * 8) = *reinterpret_cast<const uint4*>(x.p + src);
  }
}

__global__ void add_strided_kernel(const bf16* __restrict__ gsrc, int n, int ho, int wo, int c, int st, MutAct4 y) {
  const int groups = c >> 3;
  const int total = n * ho * wo * groups;
  const int h = ho * st, w = wo * st;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int q = i / groups, g = i - q * groups;
    const int img = q / (ho * wo);
    const int r = q - img * ho * wo;
    const int oy = r / wo, ox = r - oy * wo;
    bf16* dst = y.p + (static_cast<long long>(img * (h + 2 * y.pad) + oy * st + y.pad) * (w + 2 * y.pad) + ox * st + y.pad) * c +
                g * 8;
    float a[8], b[8];
    load8(dst, a);
    load8(gsrc + static_cast<long long>(q) * c + g * 8, b);
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] += b[j];
    store8(dst, a);
  }
}

__global__ void dilate_kernel(const bf16* __restrict__ dy, int n, int ho, int wo, int c, int st, MutAct4 out, int h,
                              int w) {
  const int groups = c >> 3;
  const int total = n * h * w * groups;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int p = i / groups, g = i - p * groups;
    const int img = p / (h * w);
    const int r = p - img * h * w;
    const int y = r / w, x = r - y * w;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (y % st == 0 && x % st == 0 && y / st < ho && x / st < wo)
      v = *reinterpret_cast<const uint4*>(dy + (static_cast<long long>(img * ho + y / st) * wo + x / st) * c + g * 8);
    *reinterpret_cast<uint4*>(out.p + (static_cast<long long>(img * (h + 2 * out.pad) + y + out.pad) * (w + 2 * out.pad) +
                                       x + out.pad) * c + g * 8) = v;
  }
}

__global__ void __launch_bounds__(256) add_act_kernel(Act4 a, Act4 b, MutAct4 y, int pixels, int h, int w, int c) {
  const Lane L(c);
  if (!L.active()) return;
  const int hw = h * w;
  for (int p = L.first(); p < pixels; p += L.stride()) {
    float u[8], v[8];
    load8(a.p + toff(p, hw, h, w, a.pad, ld_of(a, c)) + L.g * 8, u);
    load8(b.p + toff(p, hw, h, w, b.pad, ld_of(b, c)) + L.g * 8, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) u[j] += v[j];
    store8(y.p + toff(p, hw, h, w, y.pad, ld_of(y, c)) + L.g * 8, u);
  }
}

// ------------------------------------------------------------------ pools
// thread = (output pixel, 8 channels): k*k 16-byte loads, first max wins, padding never wins
template <int KC>   // KC > 0: compile-time KC x KC window (unrolled: the loads in flight together)
__global__ void maxpool_pad_fwd_kernel(Act4 x, int n, int h, int w, int c, int k_rt, int st, int p, MutAct4 y, int oh,
                                       int ow, uint8_t* __restrict__ idx) {
  const int k = KC > 0 ? KC : k_rt;
  const int groups = c >> 3;
  const int total = n * oh * ow * groups;
  const int hp = h + 2 * x.pad, wp = w + 2 * x.pad;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int q = i / groups, g = i - q * groups;
    const int img = q / (oh * ow);
    const int r = q - img * oh * ow;
    const int oy = r / ow, ox = r - oy * ow;
    float best[8];
    int arg[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { best[j] = 0.f; arg[j] = -1; }
#pragma unroll
    for (int ky = 0; ky < k; ++ky) {
      const int iy = oy * st + ky - p;
      if (iy < 0 || iy >= h) continue;
#pragma unroll
      for (int kx = 0; kx < k; ++kx) {
        const int ix = ox * st + kx - p;
        if (ix < 0 || ix >= w) continue;
        float v[8];
        load8(x.p + (static_cast<long long>(img * hp + iy + x.pad) * wp + ix + x.pad) * c + g * 8, v);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (arg[j] < 0 || v[j] > best[j]) { best[j] = v[j]; arg[j] = ky * k + kx; }
      }
    }
    store8(y.p + (static_cast<long long>(img * (oh + 2 * y.pad) + oy + y.pad) * (ow + 2 * y.pad) + ox + y.pad) * c + g * 8,
           best);
    uint2 ix8;
    uint8_t* b8 = reinterpret_cast<uint8_t*>(&ix8);
#pragma unroll
    for (int j = 0; j < 8; ++j) b8[j] = best[j] > 0.f ? static_cast<uint8_t>(arg[j]) : static_cast<uint8_t>(255);
    *reinterpret_cast<uint2*>(idx + static_cast<long long>(q) * c + g * 8) = ix8;
  }
}

// gather form: thread = (input pixel, 8 channels) sums dy over the windows whose argmax it is
// KC > 0: compile-time ceil(k / st) (windows covering one input per axis) -- the window
// loads are unrolled and issued together; KC == 0: runtime loops.
template <int KC>
__global__ void maxpool_pad_bwd_kernel(const uint8_t* __restrict__ idx, Act4 dy, int n, int h, int w, int c, int k,
                                       int st, int p, int oh, int ow, MutAct4 dx) {
  const int groups = c >> 3;
  const int total = n * h * w * groups;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int q = i / groups, g = i - q * groups;
    const int img = q / (h * w);
    const int r = q - img * h * w;
    const int y0 = r / w, x0 = r - y0 * w;
    // windows (oy, ox) covering (y0, x0): oy*st - p <= y0 <= oy*st - p + k - 1
    const int yy = y0 + p, xx = x0 + p;
    const int oy_lo = yy >= k ? (yy - k) / st + 1 : 0, oy_hi = min(oh - 1, yy / st);
    const int ox_lo = xx >= k ? (xx - k) / st + 1 : 0, ox_hi = min(ow - 1, xx / st);
    float acc[8] = {0.f};
    const long long dy_row = static_cast<long long>(ow + 2 * dy.pad);
    const __nv_bfloat16* dy_img = dy.p + (static_cast<long long>(img * (oh + 2 * dy.pad) + dy.pad) * dy_row + dy.pad) * c + g * 8;
    const uint8_t* idx_img = idx + static_cast<long long>(img * oh) * ow * c + g * 8;
    if constexpr (KC > 0) {
      uint2 ix8[KC][KC];
      float v[KC][KC][8];
#pragma unroll
      for (int a = 0; a < KC; ++a)
#pragma unroll
        for (int b = 0; b < KC; ++b) {
          const int oy = oy_hi - a, ox = ox_hi - b;
          ix8[a][b] = make_uint2(0xffffffffu, 0xffffffffu);
          if (oy >= oy_lo && ox >= ox_lo) {
            ix8[a][b] = *reinterpret_cast<const uint2*>(idx_img + static_cast<long long>(oy * ow + ox) * c);
            load8(dy_img + (oy * dy_row + ox) * c, v[a][b]);
          }
        }
#pragma unroll
      for (int a = 0; a < KC; ++a)
#pragma unroll
        for (int b = 0; b < KC; ++b) {
          const int pos = (yy - (oy_hi - a) * st) * k + (xx - (ox_hi - b) * st);
          const uint8_t* b8 = reinterpret_cast<const uint8_t*>(&ix8[a][b]);
#pragma unroll
          for (int j = 0; j < 8; ++j) if (b8[j] == pos) acc[j] += v[a][b][j];
        }
    } else {
      for (int oy = oy_lo; oy <= oy_hi; ++oy)
        for (int ox = ox_lo; ox <= ox_hi; ++ox) {
          const int pos = (yy - oy * st) * k + (xx - ox * st);
          const uint2 ix8 = *reinterpret_cast<const uint2*>(idx_img + static_cast<long long>(oy * ow + ox) * c);
          const uint8_t* b8 = reinterpret_cast<const uint8_t*>(&ix8);
          bool any = false;
#pragma unroll
          for (int j = 0; j < 8; ++j) any |= b8[j] == pos;
          if (!any) continue;
          float v[8];
          load8(dy_img + (oy * dy_row + ox) * c, v);
#pragma unroll
          for (int j = 0; j < 8; ++j) if (b8[j] == pos) acc[j] += v[j];
        }
    }
    store8(dx.p + (static_cast<long long>(img * (h + 2 * dx.pad) + y0 + dx.pad) * (w + 2 * dx.pad) + x0 + dx.pad) * c + g * 8,
           acc);
  }
}

__global__ void avgpool_fwd_kernel(Act4 x, int n, int h, int w, int c, bf16* __restrict__ y) {
  const long long total = static_cast<long long>(n) * c;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i % c);
    const long long img = i / c;
    float acc = 0.f;
    for (int yy = 0; yy < h; ++yy)
      for (int xx = 0; xx < w; ++xx)
        acc += __bfloat162float(
            x.p[((img * (h + 2 * x.pad) + yy + x.pad) * (w + 2 * x.pad) + xx + x.pad) * static_cast<long long>(c) + ch]);
    y[i] = __float2bfloat16_rn(acc / static_cast<float>(h * w));
  }
}

__global__ void avgpool_bwd_kernel(const bf16* __restrict__ dy, int n, int h, int w, int c, MutAct4 dx) {
  const int groups = c >> 3;
  const int total = n * h * w * groups;
  const float inv = 1.f / static_cast<float>(h * w);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int q = i / groups, g = i - q * groups;
    const int img = q / (h * w);
    const int r = q - img * h * w;
    const int yy = r / w, xx = r - yy * w;
    float v[8];
    load8(dy + static_cast<long long>(img) * c + g * 8, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] *= inv;
    store8(dx.p + (static_cast<long long>(img * (h + 2 * dx.pad) + yy + dx.pad) * (w + 2 * dx.pad) + xx + dx.pad) * c + g * 8,
           v);
  }
}

// blocks for the reductions: one wave of resident 256-thread blocks (each then walks its pixels
// with several loads in flight), never more blocks than pixel-lane groups
template <typename K>
int stats_grid(K kernel, size_t smem, long long pixels, int lanes) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, smem) != cudaSuccess || per_sm < 1) per_sm = 1;
  const long long want = static_cast<long long>(num_sms()) * per_sm;
  // >= 16 pixels per lane: every block flushes 2c global atomics, which dominate small tensors
  return static_cast<int>(std::max<long long>(1, std::min(want, (pixels + 16LL * lanes - 1) / (16LL * lanes))));
}
int pixel_grid(long long pixels, int lanes) {
  const long long want = static_cast<long long>(num_sms()) * 8;
  return static_cast<int>(std::max<long long>(1, std::min(want, (pixels + lanes - 1) / lanes)));
}
bool fits(long long elems) { return elems < (1LL << 31); }

}  // namespace

// image group g of a batch tensor (groups of n / groups consecutive images)
template <class T>
T group_slice(T a, long long img0, int h, int w, int c) {
  if (a.p != nullptr) a.p += img0 * (h + 2 * a.pad) * (w + 2 * a.pad) * static_cast<long long>(a.ld ? a.ld : c);
  return a;
}

cudaError_t bn_stats(Act4 x, int n, int h, int w, int c, float eps, float* work, float* mean, float* rstd,
                     cudaStream_t s, int groups, long long stat_stride) {
  if (groups > 1) {
    if (n % groups != 0) return cudaErrorInvalidValue;
    const int gn = n / groups;
    for (int g = 0; g < groups; ++g) {
      const cudaError_t e = bn_stats(group_slice(x, static_cast<long long>(g) * gn, h, w, c), gn, h, w, c, eps, work,
                                     mean + g * stat_stride, rstd + g * stat_stride, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  const long long pixels = static_cast<long long>(n) * h * w;
  if (c % 8 != 0 || c / 8 > 256 || !fits(pixels * c)) return cudaErrorInvalidValue;
  const int lanes = 256 / (c / 8);
  bn_stats_kernel<<<stats_grid(bn_stats_kernel, sizeof(float) * 2 * c, pixels, lanes), 256, sizeof(float) * 2 * c, s>>>(
      x, static_cast<int>(pixels), h, w, c, work, 1.f / static_cast<float>(pixels), eps, mean, rstd);
  return cudaGetLastError();
}

cudaError_t bn_apply(const BnApply& a, cudaStream_t s) {
  if (a.groups > 1) {
    if (a.n % a.groups != 0) return cudaErrorInvalidValue;
    const int gn = a.n / a.groups;
    for (int g = 0; g < a.groups; ++g) {
      BnApply q = a;
      const long long i0 = static_cast<long long>(g) * gn, o = g * a.stat_stride;
      q.groups = 1;
      q.n = gn;
      q.x = group_slice(a.x, i0, a.h, a.w, a.c);
      q.r = group_slice(a.r, i0, a.h, a.w, a.c);
      q.y = group_slice(a.y, i0, a.h, a.w, a.c);
      q.mean = a.mean + o; q.rstd = a.rstd + o;
      if (a.res_kind == 2) { q.r_mean = a.r_mean + o; q.r_rstd = a.r_rstd + o; }
      if (a.mask_out != nullptr) q.mask_out = a.mask_out + i0 * a.h * a.w * (a.c / 8);
      const cudaError_t e = bn_apply(q, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  const long long pixels = static_cast<long long>(a.n) * a.h * a.w;
  if (a.c % 8 != 0 || a.c / 8 > 256 || !fits(pixels * a.c)) return cudaErrorInvalidValue;
  const int lanes = 256 / (a.c / 8);
  bn_apply_kernel<<<pixel_grid(pixels, 2 * lanes), 256, 0, s>>>(a, static_cast<int>(pixels));
  return cudaGetLastError();
}

cudaError_t bn_backward(const BnBackward& b, float* work, cudaStream_t s) {
  if (b.groups > 1) {
    if (b.n % b.groups != 0) return cudaErrorInvalidValue;
    const int gn = b.n / b.groups;
    for (int g = 0; g < b.groups; ++g) {
      BnBackward q = b;
      const long long i0 = static_cast<long long>(g) * gn, o = g * b.stat_stride;
      q.groups = 1;
      q.n = gn;
      q.dy = group_slice(b.dy, i0, b.h, b.w, b.c);
      q.y = group_slice(b.y, i0, b.h, b.w, b.c);
      q.x = group_slice(b.x, i0, b.h, b.w, b.c);
      q.dx = group_slice(b.dx, i0, b.h, b.w, b.c);
      q.dz_out = group_slice(b.dz_out, i0, b.h, b.w, b.c);
      q.mean = b.mean + o; q.rstd = b.rstd + o;
      if (b.mask_in != nullptr) q.mask_in = b.mask_in + i0 * b.h * b.w * (b.c / 8);
      const cudaError_t e = bn_backward(q, work, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  const long long pixels = static_cast<long long>(b.n) * b.h * b.w;
  if (b.c % 8 != 0 || b.c / 8 > 256 || !fits(pixels * b.c)) return cudaErrorInvalidValue;
  const int lanes = 256 / (b.c / 8);
  if (b.mask_in != nullptr)
    bn_bwd_reduce_kernel<true><<<stats_grid(bn_bwd_reduce_kernel<true>, sizeof(float) * 2 * b.c, pixels, lanes), 256,
                                 sizeof(float) * 2 * b.c, s>>>(b, static_cast<int>(pixels), work);
  else
    bn_bwd_reduce_kernel<false><<<stats_grid(bn_bwd_reduce_kernel<false>, sizeof(float) * 2 * b.c, pixels, lanes), 256,
                                  sizeof(float) * 2 * b.c, s>>>(b, static_cast<int>(pixels), work);
  bn_bwd_apply_kernel<<<pixel_grid(pixels, lanes), 256, 0, s>>>(b, static_cast<int>(pixels), work + 2 * 2048,
                                                                1.f / static_cast<float>(pixels));
  return cudaGetLastError();
}

cudaError_t im2col_bf16(Act4 x, int n, int h, int w, int c, int k, int st, int p, int ho, int wo, __nv_bfloat16* out,
                        cudaStream_t s) {
  const long long total = static_cast<long long>(n) * ho * wo * k * k * (c / 8);
  if (c % 8 != 0 || !fits(static_cast<long long>(n) * ho * wo * k * k)) return cudaErrorInvalidValue;
  im2col_bf16_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, n, h, w, c, k, st, p, ho, wo, out);
  return cudaGetLastError();
}

cudaError_t subsample(Act4 x, int n, int h, int w, int c, int st, __nv_bfloat16* out, cudaStream_t s) {
  const long long total = static_cast<long long>(n) * (h / st) * (w / st) * (c / 8);
  if (c % 8 != 0 || !fits(total * 8)) return cudaErrorInvalidValue;
  subsample_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, n, h, w, c, st, out);
  return cudaGetLastError();
}

cudaError_t add_strided(const __nv_bfloat16* g, int n, int ho, int wo, int c, int st, MutAct4 y, cudaStream_t s) {
  const long long total = static_cast<long long>(n) * ho * wo * (c / 8);
  if (c % 8 != 0 || !fits(total * 8)) return cudaErrorInvalidValue;
  add_strided_kernel<<<grid_for(total, 256), 256, 0, s>>>(g, n, ho, wo, c, st, y);
  return cudaGetLastError();
}

cudaError_t dilate(const __nv_bfloat16* dy, int n, int ho, int wo, int c, int st, MutAct4 out, int h, int w,
                   cudaStream_t s) {
  const long long total = static_cast<long long>(n) * h * w * (c / 8);
  if (c % 8 != 0 || !fits(total * 8)) return cudaErrorInvalidValue;
  dilate_kernel<<<grid_for(total, 256), 256, 0, s>>>(dy, n, ho, wo, c, st, out, h, w);
  return cudaGetLastError();
}

cudaError_t add_act(Act4 a, Act4 b, MutAct4 y, int n, int h, int w, int c, cudaStream_t s) {
  const long long pixels = static_cast<long long>(n) * h * w;
  if (c % 8 != 0 || c / 8 > 256 || !fits(pixels * c)) return cudaErrorInvalidValue;
  const int lanes = 256 / (c / 8);
  add_act_kernel<<<pixel_grid(pixels, lanes), 256, 0, s>>>(a, b, y, static_cast<int>(pixels), h, w, c);
  return cudaGetLastError();
}

cudaError_t maxpool_pad_fwd(Act4 x, int n, int h, int w, int c, int k, int st, int p, MutAct4 y, int oh, int ow,
                            uint8_t* idx, cudaStream_t s) {
  const long long total = static_cast<long long>(n) * oh * ow * (c / 8);
  if (c % 8 != 0 || !fits(total * 8)) return cudaErrorInvalidValue;
  if (k == 3)
    maxpool_pad_fwd_kernel<3><<<grid_for(total, 256), 256, 0, s>>>(x, n, h, w, c, k, st, p, y, oh, ow, idx);
  else
    maxpool_pad_fwd_kernel<0><<<grid_for(total, 256), 256, 0, s>>>(x, n, h, w, c, k, st, p, y, oh, ow, idx);
  return cudaGetLastError();
}

cudaError_t maxpool_pad_bwd(const uint8_t* idx, Act4 dy, int n, int h, int w, int c, int k, int st, int p, int oh,
                            int ow, MutAct4 dx, cudaStream_t s) {
  const long long total = static_cast<long long>(n) * h * w * (c / 8);
  if (c % 8 != 0 || !fits(total * 8)) return cudaErrorInvalidValue;
  if (k == 3 && st == 2)
    maxpool_pad_bwd_kernel<2><<<grid_for(total, 256), 256, 0, s>>>(idx, dy, n, h, w, c, k, st, p, oh, ow, dx);
  else
    maxpool_pad_bwd_kernel<0><<<grid_for(total, 256), 256, 0, s>>>(idx, dy, n, h, w, c, k, st, p, oh, ow, dx);
  return cudaGetLastError();
}

cudaError_t avgpool_fwd(Act4 x, int n, int h, int w, int c, __nv_bfloat16* y, cudaStream_t s) {
  const long long total = static_cast<long long>(n) * c;
  avgpool_fwd_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, n, h, w, c, y);
  return cudaGetLastError();
}

cudaError_t avgpool_bwd(const __nv_bfloat16* dy, int n, int h, int w, int c, MutAct4 dx, cudaStream_t s) {
  const long long total = static_cast<long long>(n) * h * w * (c / 8);
  if (c % 8 != 0 || !fits(total * 8)) return cudaErrorInvalidValue;
  avgpool_bwd_kernel<<<grid_for(total, 256), 256, 0, s>>>(dy, n, h, w, c, dx);
  return cudaGetLastError();
}

}  // namespace ralpb
