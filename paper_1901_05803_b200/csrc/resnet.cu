// HBM-bound kernels of the bottleneck-block model (resnet.cuh).  Eight channels per thread
// (16-byte loads / stores); per-channel reductions in registers, then shared memory, then one
// global atomic per channel per block.
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

__device__ __forceinline__ long long px_off(long long pix, int h, int w, int pad, int c) {
  const long long img = pix / (static_cast<long long>(h) * w);
  const int r = static_cast<int>(pix - img * h * w);
  const int y = r / w, x = r - (r / w) * w;
  return ((img * (h + 2 * pad) + y + pad) * (w + 2 * pad) + x + pad) * static_cast<long long>(c);
}

__device__ __forceinline__ void load8(const bf16* p, float* v) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const bf16* b = reinterpret_cast<const bf16*>(&u);
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = __bfloat162float(b[j]);
}
__device__ __forceinline__ void store8(bf16* p, const float* v) {
  uint4 u;
  bf16* b = reinterpret_cast<bf16*>(&u);
#pragma unroll
  for (int j = 0; j < 8; ++j) b[j] = __float2bfloat16_rn(v[j]);
  *reinterpret_cast<uint4*>(p) = u;
}

// ------------------------------------------------------------------ batch norm statistics
// Block: 256 threads = (256 / groups) pixel lanes x groups channel groups (groups = c/8 <= 256).
__global__ void bn_stats_kernel(Act4 x, long long pixels, int h, int w, int c, float* __restrict__ sums) {
  extern __shared__ float sh[];  // [2][c]
  const int groups = c / 8;
  const int lanes = blockDim.x / groups;
  const int g = threadIdx.x % groups, lane = threadIdx.x / groups;
  for (int i = threadIdx.x; i < 2 * c; i += blockDim.x) sh[i] = 0.f;
  __syncthreads();
  float s[8] = {0.f}, q[8] = {0.f};
  if (lane < lanes) {
    for (long long p = static_cast<long long>(blockIdx.x) * lanes + lane; p < pixels;
         p += static_cast<long long>(gridDim.x) * lanes) {
      float v[8];
      load8(x.p + px_off(p, h, w, x.pad, c) + g * 8, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) { s[j] += v[j]; q[j] += v[j] * v[j]; }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      atomicAdd(&sh[g * 8 + j], s[j]);
      atomicAdd(&sh[c + g * 8 + j], q[j]);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * c; i += blockDim.x) atomicAdd(sums + i, sh[i]);
}

__global__ void bn_finish_kernel(const float* __restrict__ sums, int c, float inv_m, float eps, float* __restrict__ mean,
                                 float* __restrict__ rstd) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c) return;
  const float m = sums[i] * inv_m;
  const float var = fmaxf(sums[c + i] * inv_m - m * m, 0.f);
  mean[i] = m;
  rstd[i] = rsqrtf(var + eps);
}

// ------------------------------------------------------------------ apply
__global__ void bn_apply_kernel(BnApply a) {
  const int groups = a.c / 8;
  const long long total = static_cast<long long>(a.n) * a.h * a.w * groups;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % groups);
    const long long p = i / groups;
    float v[8];
    load8(a.x.p + px_off(p, a.h, a.w, a.x.pad, a.c) + g * 8, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int ch = g * 8 + j;
      v[j] = (v[j] - a.mean[ch]) * a.rstd[ch] * a.gamma[ch] + a.beta[ch];
    }
    if (a.res_kind != 0) {
      float r[8];
      load8(a.r.p + px_off(p, a.h, a.w, a.r.pad, a.c) + g * 8, r);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int ch = g * 8 + j;
        v[j] += a.res_kind == 2 ? (r[j] - a.r_mean[ch]) * a.r_rstd[ch] * a.r_gamma[ch] + a.r_beta[ch] : r[j];
      }
    }
    if (a.relu) {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = fmaxf(v[j], 0.f);
    }
    store8(a.y.p + px_off(p, a.h, a.w, a.y.pad, a.c) + g * 8, v);
  }
}

// ------------------------------------------------------------------ backward
__global__ void bn_bwd_reduce_kernel(BnBackward b, long long pixels, float* __restrict__ sums) {
  extern __shared__ float sh[];  // [2][c]: sum dz, sum dz * xhat
  const int c = b.c, groups = c / 8;
  const int lanes = blockDim.x / groups;
  const int g = threadIdx.x % groups, lane = threadIdx.x / groups;
  for (int i = threadIdx.x; i < 2 * c; i += blockDim.x) sh[i] = 0.f;
  __syncthreads();
  float sd[8] = {0.f}, sx[8] = {0.f};
  if (lane < lanes) {
    for (long long p = static_cast<long long>(blockIdx.x) * lanes + lane; p < pixels;
         p += static_cast<long long>(gridDim.x) * lanes) {
      float dy[8], xv[8];
      load8(b.dy.p + px_off(p, b.h, b.w, b.dy.pad, c) + g * 8, dy);
      load8(b.x.p + px_off(p, b.h, b.w, b.x.pad, c) + g * 8, xv);
      if (b.relu_mask) {
        float y[8];
        load8(b.y.p + px_off(p, b.h, b.w, b.y.pad, c) + g * 8, y);
#pragma unroll
        for (int j = 0; j < 8; ++j) if (!(y[j] > 0.f)) dy[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int ch = g * 8 + j;
        sd[j] += dy[j];
        sx[j] += dy[j] * (xv[j] - b.mean[ch]) * b.rstd[ch];
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      atomicAdd(&sh[g * 8 + j], sd[j]);
      atomicAdd(&sh[c + g * 8 + j], sx[j]);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * c; i += blockDim.x) atomicAdd(sums + i, sh[i]);
}

__global__ void bn_bwd_params_kernel(const float* __restrict__ sums, int c, float* __restrict__ dgamma,
                                     float* __restrict__ dbeta) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c) return;
  dbeta[i] += sums[i];
  dgamma[i] += sums[c + i];
}

__global__ void bn_bwd_apply_kernel(BnBackward b, const float* __restrict__ sums, float inv_m) {
  const int c = b.c, groups = c / 8;
  const long long total = static_cast<long long>(b.n) * b.h * b.w * groups;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % groups);
    const long long p = i / groups;
    float dy[8], xv[8], dx[8];
    load8(b.dy.p + px_off(p, b.h, b.w, b.dy.pad, c) + g * 8, dy);
    load8(b.x.p + px_off(p, b.h, b.w, b.x.pad, c) + g * 8, xv);
    if (b.relu_mask) {
      float y[8];
      load8(b.y.p + px_off(p, b.h, b.w, b.y.pad, c) + g * 8, y);
#pragma unroll
      for (int j = 0; j < 8; ++j) if (!(y[j] > 0.f)) dy[j] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int ch = g * 8 + j;
      const float xhat = (xv[j] - b.mean[ch]) * b.rstd[ch];
      dx[j] = b.gamma[ch] * b.rstd[ch] * (dy[j] - sums[ch] * inv_m - xhat * sums[c + ch] * inv_m);
    }
    store8(b.dx.p + px_off(p, b.h, b.w, b.dx.pad, c) + g * 8, dx);
    if (b.dz_out.p != nullptr) store8(b.dz_out.p + px_off(p, b.h, b.w, b.dz_out.pad, c) + g * 8, dy);
  }
}

// ------------------------------------------------------------------ layouts
__global__ void im2col_bf16_kernel(Act4 x, int n, int h, int w, int c, int k, int st, int p, int ho, int wo,
                                   bf16* __restrict__ out) {
  const int groups = c / 8;
  const int kk = k * k;
  const long long total = static_cast<long long>(n) * ho * wo * kk * groups;
  const int hp = h + 2 * x.pad, wp = w + 2 * x.pad;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % groups);
    long long t = i / groups;
    const int tap = static_cast<int>(t % kk);
    const long long row = t / kk;
    const int ox = static_cast<int>(row % wo);
    const long long r2 = row / wo;
    const int oy = static_cast<int>(r2 % ho);
    const long long img = r2 / ho;
    const int iy = oy * st + tap / k - p + x.pad, ix = ox * st + tap % k - p + x.pad;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (iy >= 0 && iy < hp && ix >= 0 && ix < wp)
      v = *reinterpret_cast<const uint4*>(x.p + ((img * hp + iy) * wp + ix) * c + g * 8);
    *reinterpret_cast<uint4*>(out + (row * kk + tap) * c + g * 8) = v;
  }
}

__global__ void subsample_kernel(Act4 x, int n, int h, int w, int c, int st, bf16* __restrict__ out) {
  const int groups = c / 8;
  const int ho = h / st, wo = w / st;
  const long long total = static_cast<long long>(n) * ho * wo * groups;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % groups);
    const long long q = i / groups;
    const int ox = static_cast<int>(q % wo);
    const long long r = q / wo;
    const int oy = static_cast<int>(r % ho);
    const long long img = r / ho;
    const long long src = ((img * (h + 2 * x.pad) + oy * st + x.pad) * (w + 2 * x.pad) + ox * st + x.pad) * c + g * 8;
    *reinterpret_cast<uint4*>(out + q * c + g * 8) = *reinterpret_cast<const uint4*>(x.p + src);
  }
}

__global__ void add_strided_kernel(const bf16* __restrict__ gsrc, int n, int ho, int wo, int c, int st, MutAct4 y) {
  const int groups = c / 8;
  const long long total = static_cast<long long>(n) * ho * wo * groups;
  const int h = ho * st, w = wo * st;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % groups);
    const long long q = i / groups;
    const int ox = static_cast<int>(q % wo);
    const long long r = q / wo;
    const int oy = static_cast<int>(r % ho);
    const long long img = r / ho;
    bf16* dst = y.p + ((img * (h + 2 * y.pad) + oy * st + y.pad) * (w + 2 * y.pad) + ox * st + y.pad) * c + g * 8;
    float a[8], b[8];
    load8(dst, a);
    load8(gsrc + q * c + g * 8, b);
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] += b[j];
    store8(dst, a);
  }
}

__global__ void dilate_kernel(const bf16* __restrict__ dy, int n, int ho, int wo, int c, int st, MutAct4 out, int h,
                              int w) {
  const int groups = c / 8;
  const long long total = static_cast<long long>(n) * h * w * groups;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % groups);
    const long long p = i / groups;
    const int x = static_cast<int>(p % w);
    const long long r = p / w;
    const int y = static_cast<int>(r % h);
    const long long img = r / h;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (y % st == 0 && x % st == 0 && y / st < ho && x / st < wo)
      v = *reinterpret_cast<const uint4*>(dy + ((img * ho + y / st) * wo + x / st) * c + g * 8);
    *reinterpret_cast<uint4*>(out.p + ((img * (h + 2 * out.pad) + y + out.pad) * (w + 2 * out.pad) + x + out.pad) * c +
                              g * 8) = v;
  }
}

__global__ void add_act_kernel(Act4 a, Act4 b, MutAct4 y, int n, int h, int w, int c) {
  const int groups = c / 8;
  const long long total = static_cast<long long>(n) * h * w * groups;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % groups);
    const long long p = i / groups;
    float u[8], v[8];
    load8(a.p + px_off(p, h, w, a.pad, c) + g * 8, u);
    load8(b.p + px_off(p, h, w, b.pad, c) + g * 8, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) u[j] += v[j];
    store8(y.p + px_off(p, h, w, y.pad, c) + g * 8, u);
  }
}

// ------------------------------------------------------------------ pools
__global__ void maxpool_pad_fwd_kernel(Act4 x, int n, int h, int w, int c, int k, int st, int p, MutAct4 y, int oh,
                                       int ow, uint8_t* __restrict__ idx) {
  const long long total = static_cast<long long>(n) * oh * ow * c;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i % c);
    const long long q = i / c;
    const int ox = static_cast<int>(q % ow);
    const long long r = q / ow;
    const int oy = static_cast<int>(r % oh);
    const long long img = r / oh;
    float best = 0.f;
    int arg = -1;
    for (int ky = 0; ky < k; ++ky)
      for (int kx = 0; kx < k; ++kx) {
        const int iy = oy * st + ky - p, ix = ox * st + kx - p;
        if (iy < 0 || iy >= h || ix < 0 || ix >= w) continue;   // padding never wins (-inf semantics)
        const float v = __bfloat162float(
            x.p[((img * (h + 2 * x.pad) + iy + x.pad) * (w + 2 * x.pad) + ix + x.pad) * static_cast<long long>(c) + ch]);
        if (arg < 0 || v > best) { best = v; arg = ky * k + kx; }
      }
    y.p[((img * (oh + 2 * y.pad) + oy + y.pad) * (ow + 2 * y.pad) + ox + y.pad) * static_cast<long long>(c) + ch] =
        __float2bfloat16_rn(best);
    idx[i] = best > 0.f ? static_cast<uint8_t>(arg) : static_cast<uint8_t>(255);
  }
}

__global__ void maxpool_pad_bwd_kernel(const uint8_t* __restrict__ idx, Act4 dy, int n, int h, int w, int c, int k,
                                       int st, int p, int oh, int ow, MutAct4 dx) {
  const long long total = static_cast<long long>(n) * h * w * c;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i % c);
    const long long q = i / c;
    const int x0 = static_cast<int>(q % w);
    const long long r = q / w;
    const int y0 = static_cast<int>(r % h);
    const long long img = r / h;
    // windows (oy, ox) covering (y0, x0): oy*st - p <= y0 <= oy*st - p + k - 1
    const int yy = y0 + p, xx = x0 + p;
    const int oy_lo = yy >= k ? (yy - k) / st + 1 : 0, oy_hi = min(oh - 1, yy / st);
    const int ox_lo = xx >= k ? (xx - k) / st + 1 : 0, ox_hi = min(ow - 1, xx / st);
    float acc = 0.f;
    for (int oy = oy_lo; oy <= oy_hi; ++oy)
      for (int ox = ox_lo; ox <= ox_hi; ++ox) {
        const int pos = (yy - oy * st) * k + (xx - ox * st);
        if (idx[((img * oh + oy) * ow + ox) * c + ch] != pos) continue;
        acc += __bfloat162float(
            dy.p[((img * (oh + 2 * dy.pad) + oy + dy.pad) * (ow + 2 * dy.pad) + ox + dy.pad) * static_cast<long long>(c) + ch]);
      }
    dx.p[((img * (h + 2 * dx.pad) + y0 + dx.pad) * (w + 2 * dx.pad) + x0 + dx.pad) * static_cast<long long>(c) + ch] =
        __float2bfloat16_rn(acc);
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
  const long long total = static_cast<long long>(n) * h * w * c;
  const float inv = 1.f / static_cast<float>(h * w);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i % c);
    const long long q = i / c;
    const long long img = q / (static_cast<long long>(h) * w);
    const int r = static_cast<int>(q - img * h * w);
    const int yy = r / w, xx = r - (r / w) * w;
    dx.p[((img * (h + 2 * dx.pad) + yy + dx.pad) * (w + 2 * dx.pad) + xx + dx.pad) * static_cast<long long>(c) + ch] =
        __float2bfloat16_rn(__bfloat162float(dy[img * c + ch]) * inv);
  }
}

int stats_grid(long long pixels, int lanes) {
  const long long want = static_cast<long long>(num_sms()) * 2;
  return static_cast<int>(std::max<long long>(1, std::min(want, (pixels + lanes - 1) / lanes)));
}

}  // namespace

cudaError_t bn_stats(Act4 x, int n, int h, int w, int c, float eps, float* work, float* mean, float* rstd,
                     cudaStream_t s) {
  if (c % 8 != 0 || c / 8 > 256) return cudaErrorInvalidValue;
  const long long pixels = static_cast<long long>(n) * h * w;
  cudaError_t e = cudaMemsetAsync(work, 0, sizeof(float) * 2 * c, s);
  if (e != cudaSuccess) return e;
  const int lanes = 256 / (c / 8);
  bn_stats_kernel<<<stats_grid(pixels, lanes), 256, sizeof(float) * 2 * c, s>>>(x, pixels, h, w, c, work);
  bn_finish_kernel<<<(c + 255) / 256, 256, 0, s>>>(work, c, 1.f / static_cast<float>(pixels), eps, mean, rstd);
  return cudaGetLastError();
}

cudaError_t bn_apply(const BnApply& a, cudaStream_t s) {
  if (a.c % 8 != 0) return cudaErrorInvalidValue;
  const long long total = static_cast<long long>(a.n) * a.h * a.w * (a.c / 8);
  bn_apply_kernel<<<grid_for(total, 256), 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t bn_backward(const BnBackward& b, float* work, cudaStream_t s) {
  if (b.c % 8 != 0 || b.c / 8 > 256) return cudaErrorInvalidValue;
  const long long pixels = static_cast<long long>(b.n) * b.h * b.w;
  cudaError_t e = cudaMemsetAsync(work, 0, sizeof(float) * 2 * b.c, s);
  if (e != cudaSuccess) return e;
  const int lanes = 256 / (b.c / 8);
  bn_bwd_reduce_kernel<<<stats_grid(pixels, lanes), 256, sizeof(float) * 2 * b.c, s>>>(b, pixels, work);
  bn_bwd_params_kernel<<<(b.c + 255) / 256, 256, 0, s>>>(work, b.c, b.dgamma, b.dbeta);
  const long long total = pixels * (b.c / 8);
  bn_bwd_apply_kernel<<<grid_for(total, 256), 256, 0, s>>>(b, work, 1.f / static_cast<float>(pixels));
  return cudaGetLastError();
}

cudaError_t im2col_bf16(Act4 x, int n, int h, int w, int c, int k, int st, int p, int ho, int wo, __nv_bfloat16* out,
                        cudaStream_t s) {
  if (c % 8 != 0) return cudaErrorInvalidValue;
  const long long total = static_cast<long long>(n) * ho * wo * k * k * (c / 8);
  im2col_bf16_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, n, h, w, c, k, st, p, ho, wo, out);
  return cudaGetLastError();
}

cudaError_t subsample(Act4 x, int n, int h, int w, int c, int st, __nv_bfloat16* out, cudaStream_t s) {
  if (c % 8 != 0) return cudaErrorInvalidValue;
  const long long total = static_cast<long long>(n) * (h / st) * (w / st) * (c / 8);
  subsample_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, n, h, w, c, st, out);
  return cudaGetLastError();
}

cudaError_t add_strided(const __nv_bfloat16* g, int n, int ho, int wo, int c, int st, MutAct4 y, cudaStream_t s) {
  if (c % 8 != 0) return cudaErrorInvalidValue;
  const long long total = static_cast<long long>(n) * ho * wo * (c / 8);
  add_strided_kernel<<<grid_for(total, 256), 256, 0, s>>>(g, n, ho, wo, c, st, y);
  return cudaGetLastError();
}

cudaError_t dilate(const __nv_bfloat16* dy, int n, int ho, int wo, int c, int st, MutAct4 out, int h, int w,
                   cudaStream_t s) {
  if (c % 8 != 0) return cudaErrorInvalidValue;
  const long long total = static_cast<long long>(n) * h * w * (c / 8);
  dilate_kernel<<<grid_for(total, 256), 256, 0, s>>>(dy, n, ho, wo, c, st, out, h, w);
  return cudaGetLastError();
}

cudaError_t add_act(Act4 a, Act4 b, MutAct4 y, int n, int h, int w, int c, cudaStream_t s) {
  if (c % 8 != 0) return cudaErrorInvalidValue;
  const long long total = static_cast<long long>(n) * h * w * (c / 8);
  add_act_kernel<<<grid_for(total, 256), 256, 0, s>>>(a, b, y, n, h, w, c);
  return cudaGetLastError();
}

cudaError_t maxpool_pad_fwd(Act4 x, int n, int h, int w, int c, int k, int st, int p, MutAct4 y, int oh, int ow,
                            uint8_t* idx, cudaStream_t s) {
  const long long total = static_cast<long long>(n) * oh * ow * c;
  maxpool_pad_fwd_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, n, h, w, c, k, st, p, y, oh, ow, idx);
  return cudaGetLastError();
}

cudaError_t maxpool_pad_bwd(const uint8_t* idx, Act4 dy, int n, int h, int w, int c, int k, int st, int p, int oh,
                            int ow, MutAct4 dx, cudaStream_t s) {
  const long long total = static_cast<long long>(n) * h * w * c;
  maxpool_pad_bwd_kernel<<<grid_for(total, 256), 256, 0, s>>>(idx, dy, n, h, w, c, k, st, p, oh, ow, dx);
  return cudaGetLastError();
}

cudaError_t avgpool_fwd(Act4 x, int n, int h, int w, int c, __nv_bfloat16* y, cudaStream_t s) {
  const long long total = static_cast<long long>(n) * c;
  avgpool_fwd_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, n, h, w, c, y);
  return cudaGetLastError();
}

cudaError_t avgpool_bwd(const __nv_bfloat16* dy, int n, int h, int w, int c, MutAct4 dx, cudaStream_t s) {
  const long long total = static_cast<long long>(n) * h * w * c;
  avgpool_bwd_kernel<<<grid_for(total, 256), 256, 0, s>>>(dy, n, h, w, c, dx);
  return cudaGetLastError();
}

}  // namespace ralpb
