// Branch groups executed (Inception-v3 / GoogLeNet modules; also any single
// convolution the slab kernels do not cover -- strided, unpadded or asymmetric windows).
//
// A module is a small DAG over its input x (graph.cuh ModNode): convolutions (kh x kw, stride,
// zero padding; batch norm + ReLU or bias + ReLU), max pools and average pools.  Output nodes are
// concatenated along channels: each writes its own channel slice of the module output directly
// (pixel stride = the module's channels), so the concatenation costs no copy, and its backward
// reads the slices of dy in place.  Semantics (the geometry behind the reference catalog's
// linearised inception-v3 / googlenet entries, pkg/tools/build_catalog.py:115-285):
//   conv     z = conv(x, W) (bf16);  y = relu(bn(z)) (training-mode batch statistics) or
//            y = relu(conv(x, W) + b)
//   maxpool  first maximum of the window, padding never wins
//   avgpool  mean over the in-image elements of the window (padding not counted)
// Contractions run on the tcgen05 GEMM engine: a 1x1 / stride-1 / unpadded convolution is one GEMM
// over the NHWC rows; a square 3x3 / 5x5 stride-1 'same' (or 'valid': cropped 'same') window with
// 32-aligned channels runs on the implicit-GEMM conv kernels (conv.cuh) over a padded copy of its
// input; every other window goes through an im2col patch matrix (forward, backward-filter) and a
// patch-gradient GEMM + col2im gather (backward-data, deterministic: no atomics).
// Gradients of a tensor read by several nodes are accumulated in bf16 (the first contribution
// stores, later ones add).
#include <algorithm>
#include <cstdlib>
#include "conv.cuh"
#include "elementwise.cuh"
#include "gemm_host.cuh"
#include "block.cuh"
#include "graph.cuh"
#include "resnet.cuh"

namespace ralpb {

namespace {

constexpr float kBnEps = 1e-5f;

#define RALPB_TRY(expr)                                   \
  do {                                                    \
    cudaError_t _e = (expr);                              \
    if (_e != cudaSuccess) {                              \
      if (why->empty()) *why = std::string(#expr);        \
      *why += std::string(": ") + cudaGetErrorString(_e); \
      return 1;                                           \
    }                                                     \
  } while (0)

int grid_for(long long work, int threads) {
  const long long blocks = (work + threads - 1) / threads;
  const long long cap = static_cast<long long>(num_sms()) * 8;
  return static_cast<int>(std::max<long long>(1, std::min(blocks, cap)));
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

// Decomposition of a flat (pixel, 8-channel group) index; pixel = (img*h + y)*w + x.
struct Pix {
  int g, p, img, y, x;
  __device__ __forceinline__ Pix(int i, int groups, int h, int w) {
    p = i / groups;
    g = i - p * groups;
    img = p / (h * w);
    const int r = p - img * h * w;
    y = r / w;
    x = r - y * w;
  }
};

// ------------------------------------------------------------------ layouts
// out [n*ho*wo][kh*kw*c]: column (r*kw + s)*c + ch = x[img][oy*st + r - ph][ox*st + s - pw][ch]
// (0 outside the image); x has pixel stride ldx.  One warp per patch row: the lanes walk the
// row's 16-byte chunks in order (tap-major), so every store instruction writes 512 contiguous
// bytes; the row's (img, oy, ox) is decomposed once, a chunk's tap comes from incremental
// (tap, group) counters and its (r - ph, s - pw) offsets from a per-block shared table.
constexpr int kMaxTapsGen = 64;
__global__ void __launch_bounds__(256) im2col_gen_kernel(const bf16* __restrict__ x, int ldx, int n, int h, int w, int c,
                                                         int kh, int kw, int st, int ph, int pw, int ho, int wo,
                                                         bf16* __restrict__ out) {
  __shared__ int2 toff[kMaxTapsGen];
  const int groups = c >> 3, taps = kh * kw, hw = ho * wo;
  for (int t = threadIdx.x; t < taps; t += blockDim.x) toff[t] = make_int2(t / kw - ph, t % kw - pw);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int rows = n * hw;
  const int chunks = taps * groups;
  const int q32 = 32 / groups, r32 = 32 % groups;   // advance of (tap, group) per 32 chunks
  const int t0 = lane / groups, g0 = lane % groups;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < rows; row += (gridDim.x * blockDim.x) >> 5) {
    const int img = row / hw;
    const int rr = row - img * hw;
    const int oy = rr / wo, ox = rr - oy * wo;
    const int y0 = oy * st, x0 = ox * st;
    const bf16* xi = x + static_cast<long long>(img) * h * w * ldx;
    uint4* orow = reinterpret_cast<uint4*>(out + static_cast<long long>(row) * chunks * 8);
    int tap = t0, g = g0;
    for (int j = lane; j < chunks; j += 32) {
      const int2 o = toff[tap];
      const int iy = y0 + o.x, ix = x0 + o.y;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (iy >= 0 && iy < h && ix >= 0 && ix < w)
        v = __ldg(reinterpret_cast<const uint4*>(xi + (static_cast<long long>(iy) * w + ix) * ldx) + g);
      orow[j] = v;
      tap += q32;
      g += r32;
      if (g >= groups) { g -= groups; ++tap; }
    }
  }
}

// dx[img][y][x][ch] (+)= sum over the taps (r, s) whose output position (oy, ox) reads (y, x) of
// dcol[(img*ho + oy)*wo + ox][(r*kw + s)*c + ch]  -- the adjoint of im2col_gen, gathered.
// Thread = (input pixel, up to kChunk 8-channel groups): one index decomposition per thread, the
// taps' window test per tap, then kChunk contiguous 16-byte loads per contributing tap.
constexpr int kChunk = 4;
template <bool S1>
__global__ void col2im_gen_kernel(const bf16* __restrict__ dcol, int n, int h, int w, int c, int kh, int kw, int st,
                                  int ph, int pw, int ho, int wo, bf16* __restrict__ dx, int ldx, int acc) {
  const int groups = c >> 3;
  const int chunks = (groups + kChunk - 1) / kChunk;
  const int total = n * h * w * chunks;
  const long long rowlen = static_cast<long long>(kh) * kw * c;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const Pix q(i, chunks, h, w);
    const int g0 = q.g * kChunk;
    const int ng = min(kChunk, groups - g0);
    float a[kChunk][8];
    bf16* dst = dx + static_cast<long long>(q.p) * ldx + g0 * 8;
#pragma unroll
    for (int u = 0; u < kChunk; ++u) {
      if (acc && u < ng) {
        load8(dst + u * 8, a[u]);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) a[u][j] = 0.f;
      }
    }
    for (int r = 0; r < kh; ++r) {
      int ty = q.y + ph - r;
      if (ty < 0) break;   // ty decreases with r
      if (!S1) {
        if (ty % st != 0) continue;
        ty /= st;
      }
      if (ty >= ho) continue;
      for (int s = 0; s < kw; ++s) {
        int tx = q.x + pw - s;
        if (tx < 0) break;
        if (!S1) {
          if (tx % st != 0) continue;
          tx /= st;
        }
        if (tx >= wo) continue;
        const bf16* src = dcol + (static_cast<long long>(q.img * ho + ty) * wo + tx) * rowlen + (r * kw + s) * c + g0 * 8;
#pragma unroll
        for (int u = 0; u < kChunk; ++u) {
          if (u < ng) {
            float v[8];
            load8(src + u * 8, v);
#pragma unroll
            for (int j = 0; j < 8; ++j) a[u][j] += v[j];
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kChunk; ++u)
      if (u < ng) store8(dst + u * 8, a[u]);
  }
}

// ------------------------------------------------------------------ pools
// thread = (output pixel, 8 channels); idx [n*ho*wo][c] (pixel stride c) = ky*kw + kx of the first
// max, 255 where the max is not > 0 (its producer's ReLU passes no gradient there)
template <int KC>   // KC > 0: a compile-time KC x KC window (unrolled: every load in flight at once)
__global__ void maxpool_gen_fwd_kernel(const bf16* __restrict__ x, int ldx, int n, int h, int w, int c, int kh_rt, int kw_rt,
                                       int st, int ph, int pw, int ho, int wo, bf16* __restrict__ y, int ldy,
                                       uint8_t* __restrict__ idx) {
  const int kh = KC > 0 ? KC : kh_rt, kw = KC > 0 ? KC : kw_rt;
  const int groups = c >> 3;
  const int total = n * ho * wo * groups;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const Pix q(i, groups, ho, wo);
    float best[8];
    int arg[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { best[j] = 0.f; arg[j] = -1; }
#pragma unroll
    for (int r = 0; r < kh; ++r) {
      const int iy = q.y * st + r - ph;
      if (iy < 0 || iy >= h) continue;
#pragma unroll
      for (int s = 0; s < kw; ++s) {
        const int ix = q.x * st + s - pw;
        if (ix < 0 || ix >= w) continue;
        float v[8];
        load8(x + (static_cast<long long>(q.img * h + iy) * w + ix) * ldx + q.g * 8, v);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (arg[j] < 0 || v[j] > best[j]) { best[j] = v[j]; arg[j] = r * kw + s; }
      }
    }
    store8(y + static_cast<long long>(q.p) * ldy + q.g * 8, best);
    uint2 ix8;
    uint8_t* b8 = reinterpret_cast<uint8_t*>(&ix8);
#pragma unroll
    for (int j = 0; j < 8; ++j) b8[j] = best[j] > 0.f ? static_cast<uint8_t>(arg[j]) : static_cast<uint8_t>(255);
    *reinterpret_cast<uint2*>(idx + static_cast<long long>(q.p) * c + q.g * 8) = ix8;
  }
}

// gather form: thread = (input pixel, 8 channels) sums dy over the windows whose argmax it is
template <bool S1, int KC = 0>   // KC > 0: compile-time KC x KC window (unrolled)
__global__ void maxpool_gen_bwd_kernel(const uint8_t* __restrict__ idx, const bf16* __restrict__ dy, int ldy, int n,
                                       int h, int w, int c, int kh_rt, int kw_rt, int st, int ph, int pw, int ho, int wo,
                                       bf16* __restrict__ dx, int ldx, int acc) {
  const int kh = KC > 0 ? KC : kh_rt, kw = KC > 0 ? KC : kw_rt;
  const int groups = c >> 3;
  const int total = n * h * w * groups;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const Pix q(i, groups, h, w);
    float a[8];
    bf16* dst = dx + static_cast<long long>(q.p) * ldx + q.g * 8;
    if (acc) {
      load8(dst, a);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = 0.f;
    }
#pragma unroll
    for (int r = 0; r < kh; ++r) {
      int oy = q.y + ph - r;
      if (oy < 0) break;   // decreases with r
      if (!S1) {
        if (oy % st != 0) continue;
        oy /= st;
      }
      if (oy >= ho) continue;
#pragma unroll
      for (int s = 0; s < kw; ++s) {
        int ox = q.x + pw - s;
        if (ox < 0) break;
        if (!S1) {
          if (ox % st != 0) continue;
          ox /= st;
        }
        if (ox >= wo) continue;
        const long long op = static_cast<long long>(q.img * ho + oy) * wo + ox;
        const uint2 ix8 = *reinterpret_cast<const uint2*>(idx + op * c + q.g * 8);
        const uint8_t* b8 = reinterpret_cast<const uint8_t*>(&ix8);
        const int pos = r * kw + s;
        bool any = false;
#pragma unroll
        for (int j = 0; j < 8; ++j) any |= b8[j] == pos;
        if (!any) continue;
        float v[8];
        load8(dy + op * ldy + q.g * 8, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) if (b8[j] == pos) a[j] += v[j];
      }
    }
    store8(dst, a);
  }
}

__device__ __forceinline__ int win_count(int o, int st, int p, int k, int extent) {
  const int lo = max(o * st - p, 0), hi = min(o * st - p + k, extent);
  return hi - lo;
}

// The 3x3 / stride-1 / pad-1 average pool of the Inception groups (the output grid is the input
// grid): a window's in-image count is (3 - [y at an edge]) x (3 - [x at an edge]), its inverse from a
// table -- no per-tap window arithmetic.  y (+)= / dx (+)= as the general kernels.
__constant__ float kInvCount[10] = {0.f, 1.f, 1.f / 2, 1.f / 3, 1.f / 4, 1.f / 5, 1.f / 6, 1.f / 7, 1.f / 8, 1.f / 9};
__device__ __forceinline__ int span3(int v, int n) { return 3 - (v == 0) - (v == n - 1); }

__global__ void avgpool3_fwd_kernel(const bf16* __restrict__ x, int ldx, int n, int h, int w, int c,
                                    bf16* __restrict__ y, int ldy) {
  const int groups = c >> 3;
  const int total = n * h * w * groups;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const Pix q(i, groups, h, w);
    float a[8] = {0.f};
    // fully unrolled, predicated window: all nine loads are in flight together
#pragma unroll
    for (int ry = -1; ry <= 1; ++ry)
#pragma unroll
      for (int rx = -1; rx <= 1; ++rx) {
        const int iy = q.y + ry, ix = q.x + rx;
        if (iy < 0 || iy >= h || ix < 0 || ix >= w) continue;
        float v[8];
        load8(x + (static_cast<long long>(q.img * h + iy) * w + ix) * ldx + q.g * 8, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] += v[j];
      }
    const float inv = kInvCount[span3(q.y, h) * span3(q.x, w)];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] *= inv;
    store8(y + static_cast<long long>(q.p) * ldy + q.g * 8, a);
  }
}

__global__ void avgpool3_bwd_kernel(const bf16* __restrict__ dy, int ldy, int n, int h, int w, int c,
                                    bf16* __restrict__ dx, int ldx, int acc) {
  const int groups = c >> 3;
  const int total = n * h * w * groups;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const Pix q(i, groups, h, w);
    float a[8];
    bf16* dst = dx + static_cast<long long>(q.p) * ldx + q.g * 8;
    if (acc) {
      load8(dst, a);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = 0.f;
    }
#pragma unroll
    for (int ry = -1; ry <= 1; ++ry)
#pragma unroll
      for (int rx = -1; rx <= 1; ++rx) {
        const int oy = q.y + ry, ox = q.x + rx;
        if (oy < 0 || oy >= h || ox < 0 || ox >= w) continue;
        const float inv = kInvCount[span3(oy, h) * span3(ox, w)];
        float v[8];
        load8(dy + (static_cast<long long>(q.img * h + oy) * w + ox) * ldy + q.g * 8, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] += v[j] * inv;
      }
    store8(dst, a);
  }
}

__global__ void avgpool_gen_fwd_kernel(const bf16* __restrict__ x, int ldx, int n, int h, int w, int c, int kh, int kw,
                                       int st, int ph, int pw, int ho, int wo, bf16* __restrict__ y, int ldy) {
  const int groups = c >> 3;
  const int total = n * ho * wo * groups;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const Pix q(i, groups, ho, wo);
    float a[8] = {0.f};
    for (int r = 0; r < kh; ++r) {
      const int iy = q.y * st + r - ph;
      if (iy < 0 || iy >= h) continue;
      for (int s = 0; s < kw; ++s) {
        const int ix = q.x * st + s - pw;
        if (ix < 0 || ix >= w) continue;
        float v[8];
        load8(x + (static_cast<long long>(q.img * h + iy) * w + ix) * ldx + q.g * 8, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] += v[j];
      }
    }
    const float inv = 1.f / static_cast<float>(win_count(q.y, st, ph, kh, h) * win_count(q.x, st, pw, kw, w));
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] *= inv;
    store8(y + static_cast<long long>(q.p) * ldy + q.g * 8, a);
  }
}

template <bool S1>
__global__ void avgpool_gen_bwd_kernel(const bf16* __restrict__ dy, int ldy, int n, int h, int w, int c, int kh, int kw,
                                       int st, int ph, int pw, int ho, int wo, bf16* __restrict__ dx, int ldx, int acc) {
  const int groups = c >> 3;
  const int total = n * h * w * groups;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const Pix q(i, groups, h, w);
    float a[8];
    bf16* dst = dx + static_cast<long long>(q.p) * ldx + q.g * 8;
    if (acc) {
      load8(dst, a);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = 0.f;
    }
    for (int r = 0; r < kh; ++r) {
      int oy = q.y + ph - r;
      if (oy < 0) break;   // decreases with r
      if (!S1) {
        if (oy % st != 0) continue;
        oy /= st;
      }
      if (oy >= ho) continue;
      for (int s = 0; s < kw; ++s) {
        int ox = q.x + pw - s;
        if (ox < 0) break;
        if (!S1) {
          if (ox % st != 0) continue;
          ox /= st;
        }
        if (ox >= wo) continue;
        const float inv = 1.f / static_cast<float>(win_count(oy, st, ph, kh, h) * win_count(ox, st, pw, kw, w));
        float v[8];
        load8(dy + (static_cast<long long>(q.img * ho + oy) * wo + ox) * ldy + q.g * 8, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] += v[j] * inv;
      }
    }
    store8(dst, a);
  }
}

// xp (interior of [n][h+2p][w+2p][c], borders untouched = zero) = x ([n][h][w], pixel stride ldx)
__global__ void pad_copy_kernel(const bf16* __restrict__ x, int ldx, int n, int h, int w, int c, int pad,
                                bf16* __restrict__ xp, int ldp) {
  const int groups = c >> 3;
  const int total = n * h * w * groups;
  const int hp = h + 2 * pad, wp = w + 2 * pad;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const Pix q(i, groups, h, w);
    *reinterpret_cast<uint4*>(xp + (static_cast<long long>(q.img * hp + q.y + pad) * wp + q.x + pad) * ldp + q.g * 8) =
        *reinterpret_cast<const uint4*>(x + static_cast<long long>(q.p) * ldx + q.g * 8);
  }
}

// dst ([n][h][w], pixel stride ldd) (+)= the interior of src ([n][h+2p][w+2p][c])
__global__ void unpad_kernel(const bf16* __restrict__ src, int lds, int n, int h, int w, int c, int pad,
                             bf16* __restrict__ dst, int ldd, int acc) {
  const int groups = c >> 3;
  const int total = n * h * w * groups;
  const int hp = h + 2 * pad, wp = w + 2 * pad;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const Pix q(i, groups, h, w);
    float a[8], v[8];
    load8(src + (static_cast<long long>(q.img * hp + q.y + pad) * wp + q.x + pad) * lds + q.g * 8, v);
    bf16* d = dst + static_cast<long long>(q.p) * ldd + q.g * 8;
    if (acc) {
      load8(d, a);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] += a[j];
    }
    store8(d, v);
  }
}

// dz = dy * relu'(y) over [n][h][w][c] (dy / y at pixel strides ldy / ldyv), stored bf16 at pixel
// stride ldz -- into the interior of a buffer padded by `pad` when pad > 0 (the implicit convs'
// layout) -- and, with db, the bias gradient db[c] += sum of the stored dz (block partial sums in
// shared memory, one global atomic per channel per block): the relu-grad, pad-copy and column-sum
// passes of a bias convolution in one.  blockDim must be a multiple of c / 8.
__global__ void relu_grad_colsum_kernel(const bf16* __restrict__ dy, int ldy, const bf16* __restrict__ y, int ldyv,
                                        int n, int h, int w, int c, bf16* __restrict__ dz, int ldz, int pad,
                                        float* __restrict__ db) {
  __shared__ float s_col[2048];
  const int groups = c >> 3;
  const int total = n * h * w * groups;
  float cs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const Pix q(i, groups, h, w);
    float d[8], v[8];
    load8(dy + static_cast<long long>(q.p) * ldy + q.g * 8, d);
    load8(y + static_cast<long long>(q.p) * ldyv + q.g * 8, v);
    uint4 u;
    bf16* b = reinterpret_cast<bf16*>(&u);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      b[j] = __float2bfloat16_rn(v[j] > 0.f ? d[j] : 0.f);
      cs[j] += __bfloat162float(b[j]);
    }
    const long long o = pad > 0 ? (static_cast<long long>(q.img * (h + 2 * pad) + q.y + pad) * (w + 2 * pad) + q.x + pad)
                                : static_cast<long long>(q.p);
    *reinterpret_cast<uint4*>(dz + o * ldz + q.g * 8) = u;
  }
  if (db == nullptr) return;
  for (int i = threadIdx.x; i < c; i += blockDim.x) s_col[i] = 0.f;
  __syncthreads();
  const int g = threadIdx.x % groups;
#pragma unroll
  for (int j = 0; j < 8; ++j) atomicAdd(&s_col[g * 8 + j], cs[j]);
  __syncthreads();
  for (int i = threadIdx.x; i < c; i += blockDim.x) atomicAdd(db + i, s_col[i]);
}

cudaError_t relu_grad_colsum(const bf16* dy, int ldy, const bf16* y, int ldyv, int n, int h, int w, int c, bf16* dz,
                             int ldz, int pad, float* db, cudaStream_t s) {
  const int groups = c / 8;
  if (c % 8 != 0 || groups > 256 || static_cast<long long>(n) * h * w * groups >= (1LL << 31)) return cudaErrorInvalidValue;
  const int threads = (256 / groups) * groups;
  const long long total = static_cast<long long>(n) * h * w * groups;
  const int grid = static_cast<int>(std::max<long long>(1, std::min((total + threads - 1) / threads,
                                                                   static_cast<long long>(num_sms()) * 4)));
  relu_grad_colsum_kernel<<<grid, threads, 0, s>>>(dy, ldy, y, ldyv, n, h, w, c, dz, ldz, pad, db);
  return cudaGetLastError();
}

// wp[r][cp] = w[r][c] for c < cin, 0 beyond (r = co * taps + t): filters over zero-extended channels
__global__ void filter_pad_kernel(const float* __restrict__ w, long long rows, int cin, int cpad, float* __restrict__ wp) {
  const long long total = rows * cpad;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / cpad;
    const int c = static_cast<int>(i - r * cpad);
    wp[i] = c < cin ? w[r * cin + c] : 0.f;
  }
}
// g[r][c] += gp[r][c] for c < cin: the padded filter gradient back onto the descriptor's filters
__global__ void filter_unpad_add_kernel(const float* __restrict__ gp, long long rows, int cin, int cpad, float* __restrict__ g) {
  const long long total = rows * cin;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / cin;
    const int c = static_cast<int>(i - r * cin);
    g[i] += gp[r * cpad + c];
  }
}

// ------------------------------------------------------------------ GEMM helpers
// out[rows][n] (pixel stride ldo) = a[rows][k] . w[n][k]^T, optional bias + ReLU epilogue
int gemm_fwd(Model* m, const bf16* a, long long rows, long long k, const bf16* w, int n, bf16* out, long long ldo,
             const float* bias, int relu, std::string* why) {
  GemmDesc d;
  d.M = static_cast<int>(rows); d.N = n; d.K = k;
  d.a = Operand2D{a, rows, k, k};
  d.b = Operand2D{w, n, k, k};
  d.epi = EPI_BF16; d.out = out; d.s_m = ldo;
  d.bias = bias; d.relu = relu;
  RALPB_TRY(gemm_launch(d, m->stream, why));
  ++m->launches;
  return 0;
}
// out[rows][k] = dz[rows][n] . w[n][k] (+ residual, e.g. out itself: accumulate in the epilogue)
int gemm_dgrad(Model* m, const bf16* dz, long long rows, int n, const bf16* w, long long k, bf16* out, std::string* why,
               const bf16* residual = nullptr) {
  GemmDesc d;
  d.M = static_cast<int>(rows); d.N = static_cast<int>(k); d.K = n;
  d.a_mode = LD_K; d.a = Operand2D{dz, rows, n, n};
  d.b_mode = LD_MN; d.b = Operand2D{w, n, k, k};
  d.epi = EPI_BF16; d.out = out; d.s_m = k;
  d.residual = residual; d.res_s = k;
  RALPB_TRY(gemm_launch(d, m->stream, why));
  ++m->launches;
  return 0;
}
// g[n][k] += dz[rows][n]^T . x[rows][k]
int gemm_wgrad(Model* m, const bf16* dz, long long rows, int n, const bf16* x, long long k, float* g, std::string* why) {
  GemmDesc d;
  d.M = n; d.N = static_cast<int>(k); d.K = rows;
  d.a_mode = LD_MN; d.a = Operand2D{dz, rows, n, n};
  d.b_mode = LD_MN; d.b = Operand2D{x, rows, k, k};
  d.k_splits = 0;
  d.epi = EPI_F32_ATOMIC; d.out = g; d.s_m = k; d.s_n = 1;
  RALPB_TRY(gemm_launch(d, m->stream, why));
  ++m->launches;
  return 0;
}

template <class T>
T* galloc(Model* m, size_t count, std::string* why) {
  void* p = nullptr;
  if (cudaMalloc(&p, std::max<size_t>(count * sizeof(T), 16)) != cudaSuccess) {
    *why = "cudaMalloc failed (" + std::to_string(count * sizeof(T)) + " bytes)";
    return nullptr;
  }
  m->owned.push_back(p);
  return static_cast<T*>(p);
}

long long al4(long long x) { return (x + 3) & ~3LL; }

// RALPB_MODULE_IMPLICIT=0: every non-1x1 window through im2col (the A/B baseline)
bool implicit_same() {
  static const bool on = [] {
    const char* e = getenv("RALPB_MODULE_IMPLICIT");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}
// channel alignment the implicit path requires (RALPB_MODULE_IMPLICIT_ALIGN, default 32): narrower
// K-blocks (16 channels) starve the implicit GEMM's pipeline
int implicit_align() {
  static const int a = [] {
    const char* e = getenv("RALPB_MODULE_IMPLICIT_ALIGN");
    return e != nullptr ? std::max(16, atoi(e)) : 32;
  }();
  return a;
}

// RALPB_MODULE_FUSE=0: sibling 1x1 convolutions run as separate GEMMs (the A/B baseline)
bool module_fuse() {
  static const bool on = [] {
    const char* e = getenv("RALPB_MODULE_FUSE");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

// input channels the implicit path takes: aligned, or (RALPB_MODULE_CPAD_MIN = c > 0) at least c
// 16-aligned channels, zero-extended to the alignment.  Off by default: measured on Inception-v3,
// its 80-channel 3x3 (73x73) lands on the flat implicit kernels, slower than im2col (28.6 vs 28.2 ms);
// 48 (adds the 35x35 groups' 48-channel 5x5s) 27.8 vs 27.9-28.2 ms -- within box noise.
bool implicit_cin(int c) {
  static const int lo = [] {
    const char* e = getenv("RALPB_MODULE_CPAD_MIN");
    return e != nullptr ? atoi(e) : 0;
  }();
  return c % implicit_align() == 0 || (lo > 0 && c % 16 == 0 && c >= lo);
}

template <class T>
T* galloc_zero(Model* m, size_t count, std::string* why) {
  T* p = galloc<T>(m, count, why);
  if (p != nullptr) cudaMemset(p, 0, std::max<size_t>(count * sizeof(T), 16));
  return p;
}

}  // namespace

int module_build(ModuleBufs& k, const ralpb_node_desc* nodes, int n_nodes, int n, int h, int w, int cin,
                 long long* off, std::vector<std::pair<long long, long long>>* runs, long long* count,
                 std::string* why) {
  if (nodes == nullptr || n_nodes <= 0) { *why = "module without nodes"; return 1; }
  k.n = n; k.h = h; k.w = w; k.cin = cin;
  k.nodes.assign(n_nodes, ModNode{});
  *count = 0;
  int ho = -1, wo = -1, cout = 0;
  for (int j = 0; j < n_nodes; ++j) {
    ModNode& q = k.nodes[j];
    q.d = nodes[j];
    const ralpb_node_desc& d = q.d;
    const std::string tag = "module node " + std::to_string(j) + ": ";
    if (d.input < -1 || d.input >= j) { *why = tag + "input must be an earlier node or -1"; return 1; }
    if (d.input >= 0 && k.nodes[d.input].d.output) { *why = tag + "reads an output node"; return 1; }
    if (d.kh < 1 || d.kw < 1 || d.stride < 1 || d.pad_h < 0 || d.pad_w < 0 || d.pad_h >= d.kh || d.pad_w >= d.kw) {
      *why = tag + "bad window";
      return 1;
    }
    if (d.input >= 0) {
      const ModNode& src = k.nodes[d.input];
      q.cin = src.d.op == RALPB_NODE_CONV ? src.d.cout : src.cin;
      q.h = src.ho; q.w = src.wo;
      k.nodes[d.input].consumers++;
    } else {
      q.cin = cin; q.h = h; q.w = w;
    }
    q.ho = (q.h + 2 * d.pad_h - d.kh) / d.stride + 1;
    q.wo = (q.w + 2 * d.pad_w - d.kw) / d.stride + 1;
    if (q.ho < 1 || q.wo < 1) { *why = tag + "window larger than its input"; return 1; }
    if (q.cin % 8 != 0) { *why = tag + "input channels must be a multiple of 8"; return 1; }
    if (d.kh * d.kw > 64) { *why = tag + "windows above 64 taps are not implemented"; return 1; }
    if (static_cast<long long>(n) * q.ho * q.wo * d.kh * d.kw * (q.cin / 8) >= (1LL << 31) ||
        static_cast<long long>(n) * q.h * q.w * q.cin >= (1LL << 31)) {
      *why = tag + "tensor too large for 32-bit indexing";
      return 1;
    }
    const int c_out = d.op == RALPB_NODE_CONV ? d.cout : q.cin;
    if (d.op == RALPB_NODE_CONV) {
      if (d.cout % 8 != 0 || d.cout < 8) { *why = tag + "conv output channels must be a multiple of 8"; return 1; }
      q.direct = d.kh == 1 && d.kw == 1 && d.stride == 1 && d.pad_h == 0 && d.pad_w == 0;
      // ... where the padded grid adds <= 35 % (the implicit kernels compute over it; measured: small
      // 7x7 / 14x14 windows are faster through im2col)
      // 'same' (pad (k-1)/2) or 'valid' (pad 0: the same convolution's outputs cropped by (k-1)/2)
      const int kp = (d.kh - 1) / 2;
      const bool valid = d.pad_h == 0 && d.pad_w == 0;
      q.same = implicit_same() && d.kh == d.kw && (d.kh == 3 || d.kh == 5) && d.stride == 1 && d.pad_h == d.pad_w &&
               (d.pad_h == kp || valid) && implicit_cin(q.cin) && d.cout % implicit_align() == 0 &&
               100LL * (q.h + 2 * kp) * (q.w + 2 * kp) <= 135LL * q.ho * q.wo;
      q.p = q.same ? kp : 0;
      q.cpad = q.same ? (q.cin + implicit_align() - 1) / implicit_align() * implicit_align() : q.cin;
      q.crop = q.same && valid ? kp : 0;
    } else if (d.op != RALPB_NODE_MAXPOOL && d.op != RALPB_NODE_AVGPOOL) {
      *why = tag + "unknown op";
      return 1;
    }
    if (d.output) {
      if (ho < 0) { ho = q.ho; wo = q.wo; }
      if (q.ho != ho || q.wo != wo) { *why = tag + "output nodes differ in spatial size"; return 1; }
      q.out_off = cout;
      cout += c_out;
    }
  }
  for (int j = 0; j < n_nodes; ++j) {
    const ModNode& q = k.nodes[j];
    if (!q.d.output && q.consumers == 0) { *why = "module node " + std::to_string(j) + ": output unused"; return 1; }
  }
  if (cout == 0) { *why = "module without output nodes"; return 1; }
  k.ho = ho; k.wo = wo; k.cout = cout;
  // sibling 1x1 groups: batch-normalised direct convs reading the same tensor
  k.sib.clear();
  if (module_fuse()) {
    for (int j = 0; j < n_nodes; ++j) {
      ModNode& q = k.nodes[j];
      if (q.d.op != RALPB_NODE_CONV || !q.direct || q.grp >= 0) continue;
      ModGroup g;
      for (int i = j; i < n_nodes; ++i) {
        ModNode& r = k.nodes[i];
        if (r.d.op == RALPB_NODE_CONV && r.direct && r.d.bn == q.d.bn && r.grp < 0 && r.d.input == q.d.input &&
            g.ncat + r.d.cout <= 2048)
          g.members.push_back(i), g.ncat += r.d.cout;
      }
      if (g.members.size() < 2) continue;
      for (int i : g.members) {
        k.nodes[i].grp = static_cast<int>(k.sib.size());
        k.nodes[i].grp_col = 0;
      }
      int col = 0;
      for (int i : g.members) k.nodes[i].grp_col = col, col += k.nodes[i].d.cout;
      k.sib.push_back(std::move(g));
    }
  }
  // parameter offsets, node order; a group's filters back to back at its first member
  for (int j = 0; j < n_nodes; ++j) {
    ModNode& q = k.nodes[j];
    const ralpb_node_desc& d = q.d;
    if (d.op != RALPB_NODE_CONV) continue;
    if (q.grp >= 0 && k.sib[q.grp].members[0] == j) {
      ModGroup& g = k.sib[q.grp];
      g.w_off = *off;
      for (int i : g.members) k.nodes[i].w_off = *off + static_cast<long long>(k.nodes[i].grp_col) * q.cin;
      *off = al4(*off + static_cast<long long>(g.ncat) * q.cin);
    } else if (q.grp < 0) {
      q.w_off = *off;
      *off = al4(*off + static_cast<long long>(d.cout) * q.K());
    }
    q.b_off = *off;
    const long long nb = d.bn ? 2LL * d.cout : d.cout;
    *off = al4(*off + nb);
    runs->emplace_back(q.w_off, static_cast<long long>(d.cout) * q.K());
    runs->emplace_back(q.b_off, nb);
    *count += static_cast<long long>(d.cout) * q.K() + nb;
  }
  return 0;
}

int module_alloc(Model* m, ModuleBufs& k, std::string* why) {
  long long col = 16, dz = 16;
  for (ModNode& q : k.nodes) {
    const long long rout = static_cast<long long>(k.n) * q.ho * q.wo;
    const int c_out = q.d.op == RALPB_NODE_CONV ? q.d.cout : q.cin;
    if (q.d.op == RALPB_NODE_CONV && q.same) {
      // the padded input copy, (pre-activation) output, and the gradients, all with zero borders
      const size_t pix = static_cast<size_t>(k.n) * (q.h + 2 * q.p) * (q.w + 2 * q.p);
      const size_t wpad = static_cast<size_t>(q.d.cout) * q.d.kh * q.d.kw * q.cpad;
      if (!(q.wbf = galloc<bf16>(m, wpad, why)) || !(q.wdb = galloc<bf16>(m, wpad, why)) ||
          !(q.xp = galloc_zero<bf16>(m, pix * q.cpad, why)) || !(q.z = galloc_zero<bf16>(m, pix * q.d.cout, why)) ||
          !(q.dzp = galloc_zero<bf16>(m, pix * q.d.cout, why)) || !(q.dxp = galloc_zero<bf16>(m, pix * q.cpad, why)))
        return 1;
      if (q.cpad != q.cin && !(q.gw = galloc<float>(m, wpad, why))) return 1;
      if (q.d.bn && (!(q.stats = galloc<float>(m, 2 * static_cast<size_t>(q.d.cout) * k.groups, why)) ||
                     !(q.mask = galloc<uint8_t>(m, static_cast<size_t>(rout) * q.d.cout / 8, why))))
        return 1;
      dz = std::max(dz, rout * q.d.cout);
    } else if (q.d.op == RALPB_NODE_CONV && q.grp >= 0) {
      ModGroup& g = k.sib[q.grp];
      if (g.members[0] == &q - k.nodes.data()) {
        const size_t rz = static_cast<size_t>(rout) * g.ncat;
        if (!(g.wbf = galloc<bf16>(m, static_cast<size_t>(g.ncat) * q.cin, why)) || !(g.dz = galloc<bf16>(m, rz, why)))
          return 1;
        if (q.d.bn && (!(g.z = galloc<bf16>(m, rz, why)) ||
                       !(g.stats = galloc<float>(m, 2 * static_cast<size_t>(g.ncat) * k.groups, why))))
          return 1;
        if (!res_epilogue()) col = std::max(col, static_cast<long long>(k.n) * q.h * q.w * q.cin);   // add-pass path
      }
      if (q.d.bn && !(q.mask = galloc<uint8_t>(m, static_cast<size_t>(rout) * q.d.cout / 8, why))) return 1;
    } else if (q.d.op == RALPB_NODE_CONV) {
      if (!(q.wbf = galloc<bf16>(m, static_cast<size_t>(q.d.cout) * q.K(), why))) return 1;
      if (q.d.bn) {
        if (!(q.z = galloc<bf16>(m, static_cast<size_t>(rout) * q.d.cout, why))) return 1;
        if (!(q.stats = galloc<float>(m, 2 * static_cast<size_t>(q.d.cout) * k.groups, why))) return 1;
        if (!(q.mask = galloc<uint8_t>(m, static_cast<size_t>(rout) * q.d.cout / 8, why))) return 1;
      }
      if (!q.direct) col = std::max(col, rout * q.K());
      else if (!res_epilogue()) col = std::max(col, static_cast<long long>(k.n) * q.h * q.w * q.cin);   // add-pass path
      dz = std::max(dz, rout * q.d.cout);
    } else if (q.d.op == RALPB_NODE_MAXPOOL) {
      if (!(q.idx = galloc<uint8_t>(m, static_cast<size_t>(rout) * q.cin, why))) return 1;
    }
    if (!q.d.output) {
      if (!(q.y = galloc<bf16>(m, static_cast<size_t>(rout) * c_out, why))) return 1;
      if (!(q.dy = galloc<bf16>(m, static_cast<size_t>(rout) * c_out, why))) return 1;
    }
  }
  if (!(k.col = galloc<bf16>(m, static_cast<size_t>(col), why)) || !(k.dz = galloc<bf16>(m, static_cast<size_t>(dz), why)))
    return 1;
  k.col_elems = col; k.dz_elems = dz;
  return 0;
}

int module_prep(Model* m, ModuleBufs& k, cudaStream_t s, std::string* why, std::vector<CastJob>* casts) {
  auto cast = [&](const float* x, long long n, bf16* y) -> int {
    if (casts != nullptr) {
      casts->push_back(CastJob{x, y, n});
      return 0;
    }
    RALPB_TRY(cast_bf16(x, n, y, s));
    ++m->launches;
    return 0;
  };
  for (const ModGroup& g : k.sib) {
    if (g.wbf == nullptr) continue;   // a layer this rank does not run (not allocated)
    if (cast(m->P + g.w_off, static_cast<long long>(g.ncat) * k.nodes[g.members[0]].cin, g.wbf)) return 1;
  }
  for (ModNode& q : k.nodes) {
    if (q.d.op != RALPB_NODE_CONV || q.wbf == nullptr) continue;
    if (q.same && q.cpad != q.cin) {   // via the zero-extended fp32 filters
      const long long rows = static_cast<long long>(q.d.cout) * q.d.kh * q.d.kw;
      filter_pad_kernel<<<grid_for(rows * q.cpad, 256), 256, 0, s>>>(m->P + q.w_off, rows, q.cin, q.cpad, q.gw);
      RALPB_TRY(cudaGetLastError());
      RALPB_TRY(conv_weight_prep(q.gw, q.d.cout, q.d.kh * q.d.kw, q.cpad, q.wbf, q.wdb, s));
      ++m->launches;
    } else if (q.same) {   // [cout][taps][cin] forward copy and the tap-reversed transpose for backward-data
      RALPB_TRY(conv_weight_prep(m->P + q.w_off, q.d.cout, q.d.kh * q.d.kw, q.cin, q.wbf, q.wdb, s));
      ++m->launches;
    } else if (cast(m->P + q.w_off, static_cast<long long>(q.d.cout) * q.K(), q.wbf)) {
      return 1;
    }
  }
  return 0;
}

void module_param_runs(const ModuleBufs& k, std::vector<std::pair<long long, long long>>* w_runs,
                       std::vector<std::pair<long long, long long>>* b_runs) {
  for (const ModNode& q : k.nodes) {
    if (q.d.op != RALPB_NODE_CONV) continue;
    w_runs->emplace_back(q.w_off, static_cast<long long>(q.d.cout) * q.K());
    b_runs->emplace_back(q.b_off, q.d.bn ? 2LL * q.d.cout : q.d.cout);
  }
}

int module_forward(Model* m, ModuleBufs& k, const bf16* x, bf16* y, std::string* why) {
  cudaStream_t s = m->stream;
  for (ModNode& q : k.nodes) {
    const ralpb_node_desc& d = q.d;
    const bf16* src = d.input < 0 ? x : k.nodes[d.input].y;
    const int lds = q.cin;   // inputs are contiguous (the module input or a non-output node)
    const long long rout = static_cast<long long>(k.n) * q.ho * q.wo;
    bf16* dst = d.output ? y + q.out_off : q.y;
    const int ldd = d.output ? k.cout : (d.op == RALPB_NODE_CONV ? d.cout : q.cin);
    if (d.op == RALPB_NODE_CONV && q.grp >= 0) {
      const ModGroup& g = k.sib[q.grp];
      if (!d.bn) {   // bias + ReLU epilogue into this node's destination, filters from the group copy
        if (gemm_fwd(m, src, rout, q.cin, g.wbf + static_cast<long long>(q.grp_col) * q.cin, d.cout, dst, ldd,
                     m->P + q.b_off, 1, why))
          return 1;
        continue;
      }
      if (g.members[0] != &q - k.nodes.data()) continue;   // ran with the group's first member
      if (gemm_fwd(m, src, rout, q.cin, g.wbf, g.ncat, g.z, g.ncat, nullptr, 0, why)) return 1;
      RALPB_TRY(bn_stats(Act4{g.z, 0, g.ncat}, k.n, q.ho, q.wo, g.ncat, kBnEps, m->bn_work, g.stats, g.stats + g.ncat, s,
                         k.groups, 2LL * g.ncat));
      m->launches += 2;
      for (int i : g.members) {
        const ModNode& r = k.nodes[i];
        BnApply ap{};
        ap.x = Act4{g.z + r.grp_col, 0, g.ncat};
        ap.mean = g.stats + r.grp_col; ap.rstd = g.stats + g.ncat + r.grp_col;
        ap.gamma = m->P + r.b_off; ap.beta = m->P + r.b_off + r.d.cout; ap.relu = 1;
        ap.y = r.d.output ? MutAct4{y + r.out_off, 0, k.cout} : MutAct4{r.y, 0, r.d.cout};
        ap.mask_out = r.mask;
        ap.n = k.n; ap.h = r.ho; ap.w = r.wo; ap.c = r.d.cout;
        ap.groups = k.groups; ap.stat_stride = 2LL * g.ncat;
        RALPB_TRY(bn_apply(ap, s));
        ++m->launches;
      }
    } else if (d.op == RALPB_NODE_CONV && q.same) {
      // implicit GEMM over a padded copy of the input (slab / flat kernels of conv.cuh): no patch
      // matrix; the (pre-activation) output lands in the interior of z
      const ConvGeom g{k.n, q.h, q.w, q.cpad, d.cout, d.kh, q.p};
      const long long tin = static_cast<long long>(k.n) * q.h * q.w * (q.cin / 8);
      pad_copy_kernel<<<grid_for(tin, 256), 256, 0, s>>>(src, lds, k.n, q.h, q.w, q.cin, q.p, q.xp, q.cpad);
      RALPB_TRY(cudaGetLastError());
      RALPB_TRY(conv_fwd(g, q.xp, q.wbf, d.bn ? nullptr : m->P + q.b_off, q.z, d.bn ? 0 : 1, s, why));
      m->launches += 2;
      if (d.bn) {
        RALPB_TRY(bn_stats(Act4{q.z, q.p + q.crop}, k.n, q.ho, q.wo, d.cout, kBnEps, m->bn_work, q.stats,
                           q.stats + d.cout, s,
                           k.groups, 2LL * d.cout));
        BnApply ap{};
        ap.x = Act4{q.z, q.p + q.crop}; ap.mean = q.stats; ap.rstd = q.stats + d.cout;
        ap.gamma = m->P + q.b_off; ap.beta = m->P + q.b_off + d.cout; ap.relu = 1;
        ap.y = MutAct4{dst, 0, ldd};
        ap.mask_out = q.mask;
        ap.n = k.n; ap.h = q.ho; ap.w = q.wo; ap.c = d.cout;
        ap.groups = k.groups; ap.stat_stride = 2LL * d.cout;
        RALPB_TRY(bn_apply(ap, s));
        m->launches += 3;
      } else {
        const long long tout = rout * (d.cout / 8);
        unpad_kernel<<<grid_for(tout, 256), 256, 0, s>>>(q.z, d.cout, k.n, q.ho, q.wo, d.cout, q.p + q.crop, dst, ldd, 0);
        RALPB_TRY(cudaGetLastError());
        ++m->launches;
      }
    } else if (d.op == RALPB_NODE_CONV) {
      const bf16* a = src;
      if (!q.direct) {
        const long long total = rout * 32;   // a warp per patch row
        im2col_gen_kernel<<<grid_for(total, 256), 256, 0, s>>>(src, lds, k.n, q.h, q.w, q.cin, d.kh, d.kw, d.stride,
                                                               d.pad_h, d.pad_w, q.ho, q.wo, k.col);
        RALPB_TRY(cudaGetLastError());
        ++m->launches;
        a = k.col;
      }
      if (d.bn) {
        if (gemm_fwd(m, a, rout, q.K(), q.wbf, d.cout, q.z, d.cout, nullptr, 0, why)) return 1;
        RALPB_TRY(bn_stats(Act4{q.z, 0}, k.n, q.ho, q.wo, d.cout, kBnEps, m->bn_work, q.stats, q.stats + d.cout, s,
                           k.groups, 2LL * d.cout));
        BnApply ap{};
        ap.x = Act4{q.z, 0}; ap.mean = q.stats; ap.rstd = q.stats + d.cout;
        ap.gamma = m->P + q.b_off; ap.beta = m->P + q.b_off + d.cout; ap.relu = 1;
        ap.y = MutAct4{dst, 0, ldd};
        ap.mask_out = q.mask;
        ap.n = k.n; ap.h = q.ho; ap.w = q.wo; ap.c = d.cout;
        ap.groups = k.groups; ap.stat_stride = 2LL * d.cout;
        RALPB_TRY(bn_apply(ap, s));
        m->launches += 3;
      } else {
        if (gemm_fwd(m, a, rout, q.K(), q.wbf, d.cout, dst, ldd, m->P + q.b_off, 1, why)) return 1;
      }
    } else if (d.op == RALPB_NODE_MAXPOOL) {
      const long long total = rout * (q.cin / 8);
      auto kern = d.kh == 3 && d.kw == 3 ? maxpool_gen_fwd_kernel<3> : maxpool_gen_fwd_kernel<0>;
      kern<<<grid_for(total, 256), 256, 0, s>>>(src, lds, k.n, q.h, q.w, q.cin, d.kh, d.kw, d.stride, d.pad_h, d.pad_w,
                                                q.ho, q.wo, dst, ldd, q.idx);
      RALPB_TRY(cudaGetLastError());
      ++m->launches;
    } else {
      const long long total = rout * (q.cin / 8);
      if (d.kh == 3 && d.kw == 3 && d.stride == 1 && d.pad_h == 1 && d.pad_w == 1 && q.h > 1 && q.w > 1)
        avgpool3_fwd_kernel<<<grid_for(total, 256), 256, 0, s>>>(src, lds, k.n, q.h, q.w, q.cin, dst, ldd);
      else
        avgpool_gen_fwd_kernel<<<grid_for(total, 256), 256, 0, s>>>(src, lds, k.n, q.h, q.w, q.cin, d.kh, d.kw,
                                                                    d.stride, d.pad_h, d.pad_w, q.ho, q.wo, dst, ldd);
      RALPB_TRY(cudaGetLastError());
      ++m->launches;
    }
  }
  return 0;
}

int module_backward(Model* m, ModuleBufs& k, const bf16* x, const bf16* y, const bf16* dy, bf16* dx, std::string* why) {
  cudaStream_t s = m->stream;
  float *P = m->P, *G = m->G;
  // which gradient buffers have received their first contribution (reverse node order)
  std::vector<char> started(k.nodes.size() + 1, 0);   // [0] = the module input, [j + 1] = node j
  for (int j = static_cast<int>(k.nodes.size()) - 1; j >= 0; --j) {
    ModNode& q = k.nodes[j];
    const ralpb_node_desc& d = q.d;
    const bf16* src = d.input < 0 ? x : k.nodes[d.input].y;
    const int lds = q.cin;
    const long long rin = static_cast<long long>(k.n) * q.h * q.w;
    const long long rout = static_cast<long long>(k.n) * q.ho * q.wo;
    const bf16* g_out = d.output ? dy + q.out_off : q.dy;    // gradient w.r.t. this node's output
    const bf16* v_out = d.output ? y + q.out_off : q.y;      // ... and the output itself
    const int ldo = d.output ? k.cout : (d.op == RALPB_NODE_CONV ? d.cout : q.cin);
    bf16* g_in = d.input < 0 ? dx : k.nodes[d.input].dy;     // gradient w.r.t. its input (may be null)
    char& st = started[d.input + 1];
    const int acc = st ? 1 : 0;
    if (d.op == RALPB_NODE_CONV && q.grp >= 0) {
      const ModGroup& g = k.sib[q.grp];
      if (!d.bn) {   // dz = dy * relu'(y) into the group's gradient columns; bias gradient = column sums
        RALPB_TRY(relu_grad_colsum(g_out, ldo, v_out, ldo, k.n, q.ho, q.wo, d.cout, g.dz + q.grp_col, g.ncat, 0,
                                   G + q.b_off, s));
        ++m->launches;
      } else {
        BnBackward bb{};
        bb.dy = Act4{g_out, 0, ldo}; bb.y = Act4{v_out, 0, ldo}; bb.relu_mask = 1; bb.x = Act4{g.z + q.grp_col, 0, g.ncat};
        bb.mask_in = q.mask;
        bb.mean = g.stats + q.grp_col; bb.rstd = g.stats + g.ncat + q.grp_col; bb.gamma = P + q.b_off;
        bb.dgamma = G + q.b_off; bb.dbeta = G + q.b_off + d.cout;
        bb.dx = MutAct4{g.dz + q.grp_col, 0, g.ncat};
        bb.n = k.n; bb.h = q.ho; bb.w = q.wo; bb.c = d.cout;
        bb.groups = k.groups; bb.stat_stride = 2LL * g.ncat;
        RALPB_TRY(bn_backward(bb, m->bn_work, s));
        m->launches += 3;
      }
      if (g.members[0] != j) continue;   // the group's contractions run once every member's dz is in
      if (gemm_wgrad(m, g.dz, rout, g.ncat, src, q.cin, G + g.w_off, why)) return 1;
      if (g_in != nullptr) {
        if (!acc || res_epilogue()) {
          if (gemm_dgrad(m, g.dz, rout, g.ncat, g.wbf, q.cin, g_in, why, acc ? g_in : nullptr)) return 1;
        } else {
          if (gemm_dgrad(m, g.dz, rout, g.ncat, g.wbf, q.cin, k.col, why)) return 1;
          RALPB_TRY(add_act(Act4{g_in, 0}, Act4{k.col, 0}, MutAct4{g_in, 0}, k.n, q.h, q.w, q.cin, s));
          ++m->launches;
        }
        st = 1;
      }
    } else if (d.op == RALPB_NODE_CONV && q.same) {
      const ConvGeom g{k.n, q.h, q.w, q.cpad, d.cout, d.kh, q.p};
      if (d.bn) {   // dz (padded) from the batch-norm backward
        BnBackward bb{};
        bb.dy = Act4{g_out, 0, ldo}; bb.y = Act4{v_out, 0, ldo}; bb.relu_mask = 1; bb.x = Act4{q.z, q.p + q.crop};
        bb.mask_in = q.mask;
        bb.mean = q.stats; bb.rstd = q.stats + d.cout; bb.gamma = P + q.b_off;
        bb.dgamma = G + q.b_off; bb.dbeta = G + q.b_off + d.cout;
        bb.dx = MutAct4{q.dzp, q.p + q.crop};   // (a cropped ring of the same conv's outputs stays 0)
        bb.n = k.n; bb.h = q.ho; bb.w = q.wo; bb.c = d.cout;
        bb.groups = k.groups; bb.stat_stride = 2LL * d.cout;
        RALPB_TRY(bn_backward(bb, m->bn_work, s));
        m->launches += 3;
      } else {      // dz = dy * relu'(y) straight into the padded buffer; bias gradient = its column sums
        RALPB_TRY(relu_grad_colsum(g_out, ldo, v_out, ldo, k.n, q.ho, q.wo, d.cout, q.dzp, d.cout, q.p + q.crop,
                                   G + q.b_off, s));
        ++m->launches;
      }
      if (q.cpad != q.cin) {   // into the padded scratch, then onto the descriptor's filters
        const long long rows = static_cast<long long>(d.cout) * d.kh * d.kw;
        RALPB_TRY(cudaMemsetAsync(q.gw, 0, static_cast<size_t>(rows) * q.cpad * sizeof(float), s));
        RALPB_TRY(conv_wgrad(g, q.xp, q.dzp, q.gw, nullptr, s, why));
        filter_unpad_add_kernel<<<grid_for(rows * q.cin, 256), 256, 0, s>>>(q.gw, rows, q.cin, q.cpad, G + q.w_off);
        RALPB_TRY(cudaGetLastError());
        m->launches += 2;
      } else {
        RALPB_TRY(conv_wgrad(g, q.xp, q.dzp, G + q.w_off, nullptr, s, why));
        ++m->launches;
      }
      if (g_in != nullptr) {
        RALPB_TRY(conv_dgrad(g, q.dzp, q.wdb, nullptr, q.dxp, nullptr, s, why));
        const long long tin = rin * (q.cin / 8);
        unpad_kernel<<<grid_for(tin, 256), 256, 0, s>>>(q.dxp, q.cpad, k.n, q.h, q.w, q.cin, q.p, g_in, lds, acc);
        RALPB_TRY(cudaGetLastError());
        m->launches += 2;
        st = 1;
      }
    } else if (d.op == RALPB_NODE_CONV) {
      // dz: the gradient w.r.t. the pre-activation (bn: w.r.t. the pre-batch-norm output)
      if (d.bn) {
        BnBackward bb{};
        bb.dy = Act4{g_out, 0, ldo}; bb.y = Act4{v_out, 0, ldo}; bb.relu_mask = 1; bb.x = Act4{q.z, 0};
        bb.mask_in = q.mask;
        bb.mean = q.stats; bb.rstd = q.stats + d.cout; bb.gamma = P + q.b_off;
        bb.dgamma = G + q.b_off; bb.dbeta = G + q.b_off + d.cout;
        bb.dx = MutAct4{k.dz, 0};
        bb.n = k.n; bb.h = q.ho; bb.w = q.wo; bb.c = d.cout;
        bb.groups = k.groups; bb.stat_stride = 2LL * d.cout;
        RALPB_TRY(bn_backward(bb, m->bn_work, s));
        m->launches += 3;
      } else {
        RALPB_TRY(relu_grad_colsum(g_out, ldo, v_out, ldo, k.n, q.ho, q.wo, d.cout, k.dz, d.cout, 0, G + q.b_off, s));
        ++m->launches;
      }
      // backward-filter
      if (q.direct) {
        if (gemm_wgrad(m, k.dz, rout, d.cout, src, q.cin, G + q.w_off, why)) return 1;
      } else {
        const long long total = rout * 32;   // a warp per patch row
        im2col_gen_kernel<<<grid_for(total, 256), 256, 0, s>>>(src, lds, k.n, q.h, q.w, q.cin, d.kh, d.kw, d.stride,
                                                               d.pad_h, d.pad_w, q.ho, q.wo, k.col);
        RALPB_TRY(cudaGetLastError());
        ++m->launches;
        if (gemm_wgrad(m, k.dz, rout, d.cout, k.col, q.K(), G + q.w_off, why)) return 1;
      }
      // backward-data
      if (g_in != nullptr) {
        if (q.direct && (!acc || res_epilogue())) {   // a later contribution: summed in the GEMM epilogue
          if (gemm_dgrad(m, k.dz, rout, d.cout, q.wbf, q.cin, g_in, why, acc ? g_in : nullptr)) return 1;
        } else if (q.direct) {   // RALPB_RES_EPI=0: via the patch workspace and an add pass
          if (gemm_dgrad(m, k.dz, rout, d.cout, q.wbf, q.cin, k.col, why)) return 1;
          RALPB_TRY(add_act(Act4{g_in, 0}, Act4{k.col, 0}, MutAct4{g_in, 0}, k.n, q.h, q.w, q.cin, s));
          ++m->launches;
        } else {
          if (gemm_dgrad(m, k.dz, rout, d.cout, q.wbf, q.K(), k.col, why)) return 1;
          const long long total = rin * ((q.cin / 8 + kChunk - 1) / kChunk);
          if (d.stride == 1)
            col2im_gen_kernel<true><<<grid_for(total, 256), 256, 0, s>>>(k.col, k.n, q.h, q.w, q.cin, d.kh, d.kw, 1,
                                                                         d.pad_h, d.pad_w, q.ho, q.wo, g_in, lds, acc);
          else
            col2im_gen_kernel<false><<<grid_for(total, 256), 256, 0, s>>>(k.col, k.n, q.h, q.w, q.cin, d.kh, d.kw,
                                                                          d.stride, d.pad_h, d.pad_w, q.ho, q.wo, g_in,
                                                                          lds, acc);
          RALPB_TRY(cudaGetLastError());
          ++m->launches;
        }
        st = 1;
      }
    } else if (g_in != nullptr) {
      const long long total = rin * (q.cin / 8);
      const int gr = grid_for(total, 256);
      const bool s1 = d.stride == 1;
      if (d.op == RALPB_NODE_MAXPOOL) {
        const bool k3 = d.kh == 3 && d.kw == 3;
        auto kern = s1 ? (k3 ? maxpool_gen_bwd_kernel<true, 3> : maxpool_gen_bwd_kernel<true>)
                       : (k3 ? maxpool_gen_bwd_kernel<false, 3> : maxpool_gen_bwd_kernel<false>);
        kern<<<gr, 256, 0, s>>>(q.idx, g_out, ldo, k.n, q.h, q.w, q.cin, d.kh, d.kw, d.stride, d.pad_h, d.pad_w, q.ho,
                                q.wo, g_in, lds, acc);
      } else {
        if (d.kh == 3 && d.kw == 3 && s1 && d.pad_h == 1 && d.pad_w == 1 && q.h > 1 && q.w > 1) {
          avgpool3_bwd_kernel<<<gr, 256, 0, s>>>(g_out, ldo, k.n, q.h, q.w, q.cin, g_in, lds, acc);
          RALPB_TRY(cudaGetLastError());
          ++m->launches;
          st = 1;
          continue;
        }
        auto kern = s1 ? avgpool_gen_bwd_kernel<true> : avgpool_gen_bwd_kernel<false>;
        kern<<<gr, 256, 0, s>>>(g_out, ldo, k.n, q.h, q.w, q.cin, d.kh, d.kw, d.stride, d.pad_h, d.pad_w, q.ho, q.wo,
                                g_in, lds, acc);
      }
      RALPB_TRY(cudaGetLastError());
      ++m->launches;
      st = 1;
    }
  }
  if (dx != nullptr && !started[0]) RALPB_TRY(cudaMemsetAsync(dx, 0, static_cast<size_t>(k.n) * k.h * k.w * k.cin * 2, s));
  return 0;
}

}  // namespace ralpb
