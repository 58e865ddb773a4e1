#include <algorithm>
#include "elementwise.cuh"
#include "gemm_host.cuh"
#include "ptx.cuh"

namespace ralpb {

static int grid_for(long long work, int threads) {
  long long blocks = (work + threads - 1) / threads;
  long long cap = static_cast<long long>(num_sms()) * 16;
  return static_cast<int>(std::max<long long>(1, std::min(blocks, cap)));
}

// ------------------------------------------------------------------ input packing
__global__ void pack_input_kernel(const float* __restrict__ x, int n, int h, int w, int c,
                                  __nv_bfloat16* __restrict__ out, int cp, int pad) {
  const int hp = h + 2 * pad, wp = w + 2 * pad;
  const long long total = static_cast<long long>(n) * hp * wp;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long img = i / (hp * wp);
    int r = static_cast<int>(i - img * hp * wp);
    int ph = r / wp, pw = r - (r / wp) * wp;
    int ih = ph - pad, iw = pw - pad;
    bool in = ih >= 0 && ih < h && iw >= 0 && iw < w;
    const float* src = x + ((img * h + ih) * w + iw) * c;
    __nv_bfloat16* dst = out + i * cp;
    for (int ch = 0; ch < cp; ch += 2) {
      float a = (in && ch < c) ? src[ch] : 0.f;
      float b = (in && ch + 1 < c) ? src[ch + 1] : 0.f;
      *reinterpret_cast<__nv_bfloat162*>(dst + ch) = __floats2bfloat162_rn(a, b);
    }
  }
}

cudaError_t pack_input(const float* x, int n, int h, int w, int c, __nv_bfloat16* out, int cp,
                       int pad, cudaStream_t s) {
  long long total = static_cast<long long>(n) * (h + 2 * pad) * (w + 2 * pad);
  pack_input_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, n, h, w, c, out, cp, pad);
  return cudaGetLastError();
}

// One thread = 8 consecutive columns of one im2col row (a 16-byte store).
__global__ void pack_im2col_kernel(const float* __restrict__ x, int n, int h, int w, int c, int k, int st, int p,
                                   int ho, int wo, int po, int kpad, __nv_bfloat16* __restrict__ out) {
  const int hop = ho + 2 * po, wop = wo + 2 * po;
  const int groups = kpad / 8;
  const int kk = k * k * c;
  const long long total = static_cast<long long>(n) * hop * wop * groups;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % groups);
    const long long row = i / groups;
    const long long img = row / (static_cast<long long>(hop) * wop);
    const int rem = static_cast<int>(row - img * hop * wop);
    const int oy = rem / wop - po, ox = rem % wop - po;
    const bool interior = oy >= 0 && oy < ho && ox >= 0 && ox < wo;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int j = g * 8 + e;
      float val = 0.f;
      if (interior) {
        if (j < kk) {
          const int ch = j % c, tap = j / c;
          const int iy = oy * st + tap / k - p, ix = ox * st + tap % k - p;
          if (iy >= 0 && iy < h && ix >= 0 && ix < w) val = x[((img * h + iy) * w + ix) * c + ch];
        } else if (j == kk) {
          val = 1.f;
        }
      }
      v[e] = __float2bfloat16_rn(val);
    }
    *reinterpret_cast<uint4*>(out + row * kpad + g * 8) = *reinterpret_cast<const uint4*>(v);
  }
}

// Fully unrolled variant (one thread = one patch row, all columns in registers) for the
// common small first layers, e.g. VGG's 3x3x3 (+bias) -> 32 columns.
template <int K, int C, int KPAD>
__global__ void pack_im2col_row_kernel(const float* __restrict__ x, int n, int h, int w, int st, int p, int ho,
                                       int wo, int po, __nv_bfloat16* __restrict__ out) {
  const int hop = ho + 2 * po, wop = wo + 2 * po;
  const int rows = n * hop * wop;
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < rows; row += gridDim.x * blockDim.x) {
    const int img = row / (hop * wop);
    const int rem = row - img * hop * wop;
    const int py = rem / wop;
    const int oy = py - po, ox = rem - py * wop - po;
    const bool interior = oy >= 0 && oy < ho && ox >= 0 && ox < wo;
    const float* base = x + static_cast<long long>(img) * h * w * C;
    __align__(16) __nv_bfloat16 v[KPAD];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int iy = oy * st + r - p;
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const int ix = ox * st + s - p;
        const bool in = interior && iy >= 0 && iy < h && ix >= 0 && ix < w;
        const float* src = base + (static_cast<long long>(in ? iy : 0) * w + (in ? ix : 0)) * C;
#pragma unroll
        for (int ch = 0; ch < C; ++ch) v[(r * K + s) * C + ch] = __float2bfloat16_rn(in ? __ldg(src + ch) : 0.f);
      }
    }
    v[K * K * C] = __float2bfloat16_rn(interior ? 1.f : 0.f);
#pragma unroll
    for (int j = K * K * C + 1; j < KPAD; ++j) v[j] = __float2bfloat16_rn(0.f);
    uint4* o = reinterpret_cast<uint4*>(out + static_cast<long long>(row) * KPAD);
#pragma unroll
    for (int q = 0; q < KPAD / 8; ++q) o[q] = reinterpret_cast<const uint4*>(v)[q];
  }
}

// Large first-layer filters (AlexNet's 11x11x3 -> 363 (+bias) columns, kpad 384; ResNet's /
// GoogLeNet's 7x7x3 stem -> 147 (+ones), kpad 192).  One CTA per row of the padded output grid
// (img, py): the K image rows its patches read are staged in shared memory as fp32 with coalesced
// loads (zero outside the image; each image row is staged by ~K/st output rows instead of being
// gathered column by column by every patch), then each warp builds whole patch rows from shared
// memory: lane l owns columns [l*KPAD/32, (l+1)*KPAD/32), index arithmetic by compile-time
// constants, 8-byte stores (4-byte when KPAD/32 is not a multiple of 4).
template <int K, int C, int KPAD>
__global__ void __launch_bounds__(256) pack_im2col_smem_kernel(const float* __restrict__ x, int n, int h, int w, int st,
                                                               int p, int ho, int wo, int po,
                                                               __nv_bfloat16* __restrict__ out) {
  constexpr int PER = KPAD / 32, KK = K * K * C;
  static_assert(PER % 2 == 0, "lane span must be a multiple of 2 columns");
  extern __shared__ float sx[];   // [K][w * C]
  const int hop = ho + 2 * po, wop = wo + 2 * po;
  const int rowlen = w * C;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int gr = blockIdx.x; gr < n * hop; gr += gridDim.x) {
    const int img = gr / hop, py = gr - img * hop;
    const int oy = py - po;
    const bool row_in = oy >= 0 && oy < ho;
    __syncthreads();   // the previous row's patches are built
    if (row_in) {
      const float* xi = x + static_cast<long long>(img) * h * rowlen;
      for (int i = threadIdx.x; i < K * rowlen; i += blockDim.x) {
        const int r = i / rowlen;
        const int iy = oy * st - p + r;
        sx[i] = (iy >= 0 && iy < h) ? __ldg(xi + static_cast<long long>(iy) * rowlen + (i - r * rowlen)) : 0.f;
      }
    }
    __syncthreads();
    for (int px = warp; px < wop; px += nwarps) {
      const int ox = px - po;
      const bool interior = row_in && ox >= 0 && ox < wo;
      const int x0 = ox * st - p;
      float v[PER];
      if constexpr (PER % C == 0) {
        // the lane's columns are PER / C whole taps: their (row, column) offsets are per-lane
        // constants (tap_r / tap_s), so a value is one bounds test and one shared-memory load
#pragma unroll
        for (int t = 0; t < PER / C; ++t) {
          const int tap = lane * (PER / C) + t;
          const int r = tap / K, sc = tap - r * K;
          const int ix = x0 + sc;
          const bool ok = interior && tap < K * K && ix >= 0 && ix < w;
#pragma unroll
          for (int ch = 0; ch < C; ++ch)
            v[t * C + ch] = ok ? sx[r * rowlen + ix * C + ch] : 0.f;
          if (tap == K * K) v[t * C] = interior ? 1.f : 0.f;   // the ones (bias) column
        }
      } else {
#pragma unroll
        for (int e = 0; e < PER; ++e) {
          const int j = lane * PER + e;
          float val = 0.f;
          if (interior) {
            if (j < KK) {
              const int ch = j % C, tap = j / C;
              const int r = tap / K, ix = x0 + tap % K;
              if (ix >= 0 && ix < w) val = sx[r * rowlen + ix * C + ch];
            } else if (j == KK) {
              val = 1.f;
            }
          }
          v[e] = val;
        }
      }
      uint32_t pk[PER / 2];
#pragma unroll
      for (int e2 = 0; e2 < PER / 2; ++e2) pk[e2] = pack_bf16(v[2 * e2], v[2 * e2 + 1]);
      __nv_bfloat16* orow = out + (static_cast<long long>(gr) * wop + px) * KPAD + lane * PER;
      if constexpr (PER % 4 == 0) {
        uint2* dst = reinterpret_cast<uint2*>(orow);
#pragma unroll
        for (int e4 = 0; e4 < PER / 4; ++e4) dst[e4] = make_uint2(pk[2 * e4], pk[2 * e4 + 1]);
      } else {
        uint32_t* dst = reinterpret_cast<uint32_t*>(orow);
#pragma unroll
        for (int e2 = 0; e2 < PER / 2; ++e2) dst[e2] = pk[e2];
      }
    }
  }
}

template <int K, int C, int KPAD>
cudaError_t launch_im2col_smem(const float* x, int n, int h, int w, int st, int p, int ho, int wo, int po,
                               __nv_bfloat16* out, cudaStream_t s) {
  const size_t smem = sizeof(float) * K * static_cast<size_t>(w) * C;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(pack_im2col_smem_kernel<K, C, KPAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const long long rows = static_cast<long long>(n) * (ho + 2 * po);
  const int grid = static_cast<int>(std::min<long long>(rows, static_cast<long long>(num_sms()) * 16));
  pack_im2col_smem_kernel<K, C, KPAD><<<grid, 256, smem, s>>>(x, n, h, w, st, p, ho, wo, po, out);
  return cudaGetLastError();
}

cudaError_t pack_im2col(const float* x, int n, int h, int w, int c, int k, int st, int p, int ho, int wo,
                        int po, int kpad, __nv_bfloat16* out, cudaStream_t s) {
  if (k == 11 && c == 3 && kpad == 384) return launch_im2col_smem<11, 3, 384>(x, n, h, w, st, p, ho, wo, po, out, s);
  if (k == 7 && c == 3 && kpad == 192) return launch_im2col_smem<7, 3, 192>(x, n, h, w, st, p, ho, wo, po, out, s);
  if (kpad % 8 != 0 || kpad < k * k * c + 1) return cudaErrorInvalidValue;
  const long long rows = static_cast<long long>(n) * (ho + 2 * po) * (wo + 2 * po);
  if (k == 3 && c == 3 && kpad == 32 && rows < (1LL << 31)) {
    pack_im2col_row_kernel<3, 3, 32><<<grid_for(rows, 256), 256, 0, s>>>(x, n, h, w, st, p, ho, wo, po, out);
    return cudaGetLastError();
  }
  const long long total = static_cast<long long>(n) * (ho + 2 * po) * (wo + 2 * po) * (kpad / 8);
  pack_im2col_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, n, h, w, c, k, st, p, ho, wo, po, kpad, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ max pool
// One thread = one output position x 8 channels.
__global__ void maxpool_fwd_kernel(const __nv_bfloat16* __restrict__ x, int n, int h, int w, int c,
                                   int pi, int k, int st, __nv_bfloat16* __restrict__ y, int po,
                                   int oh, int ow, uint8_t* __restrict__ idx) {
  const int ohp = oh + 2 * po, owp = ow + 2 * po;
  const int hp = h + 2 * pi, wp = w + 2 * pi;
  const int cv = c / 8;
  // 32-bit index arithmetic (the launcher checks n * ohp * owp * cv < 2^31)
  const int total = n * ohp * owp * cv;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int pos = i / cv;
    const int cg = i - pos * cv;
    const long long img = pos / (ohp * owp);
    const int r = pos - static_cast<int>(img) * ohp * owp;
    const int py = r / owp, px = r - py * owp;
    int oy = py - po, ox = px - po;
    uint4 res = make_uint4(0, 0, 0, 0);
    if (oy >= 0 && oy < oh && ox >= 0 && ox < ow) {
      float m[8];
      int a[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) { m[e] = -INFINITY; a[e] = 0; }
      for (int ky = 0; ky < k; ++ky) {
        for (int kx = 0; kx < k; ++kx) {
          long long src = ((img * hp + oy * st + ky + pi) * wp + ox * st + kx + pi) * c + cg * 8;
          uint4 u = *reinterpret_cast<const uint4*>(x + src);
          const __nv_bfloat16* hb = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float v = __bfloat162float(hb[e]);
            if (v > m[e]) { m[e] = v; a[e] = ky * k + kx; }   // first max, row-major
          }
        }
      }
      __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&res);
#pragma unroll
      for (int e = 0; e < 8; ++e) ob[e] = __float2bfloat16_rn(m[e]);
      if (idx != nullptr) {
        uint2 iw;
        uint8_t* ib = reinterpret_cast<uint8_t*>(&iw);
#pragma unroll
        for (int e = 0; e < 8; ++e) ib[e] = m[e] > 0.f ? static_cast<uint8_t>(a[e]) : uint8_t(255);
        *reinterpret_cast<uint2*>(idx + ((img * oh + oy) * ow + ox) * c + cg * 8) = iw;
      }
    }
    *reinterpret_cast<uint4*>(y + static_cast<long long>(pos) * c + cg * 8) = res;
  }
}

cudaError_t maxpool_fwd(const __nv_bfloat16* x, int n, int h, int w, int c, int pad_in, int k,
                        int st, __nv_bfloat16* y, int pad_out, cudaStream_t s, uint8_t* idx) {
  if (idx != nullptr && k * k > 255) return cudaErrorInvalidValue;
  if (c % 8 != 0) return cudaErrorInvalidValue;
  int oh = (h - k) / st + 1, ow = (w - k) / st + 1;
  long long total = static_cast<long long>(n) * (oh + 2 * pad_out) * (ow + 2 * pad_out) * (c / 8);
  if (total >= (1LL << 31)) return cudaErrorInvalidValue;
  maxpool_fwd_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, n, h, w, c, pad_in, k, st, y, pad_out, oh, ow, idx);
  return cudaGetLastError();
}

// Bias gradient of the convolution feeding a max-pool, fused into the pool backward: every
// thread keeps a fixed 8-channel group (the block size and the grid stride are multiples of
// c/8), sums the bf16 values it stores, and the block folds them through shared memory into
// one global atomic per channel.
constexpr int kPoolColsumMax = 1024;
__device__ __forceinline__ void block_colsum_flush(const float* csum, int cg, int c, float* s_col, float* colsum) {
  for (int i = threadIdx.x; i < c; i += blockDim.x) s_col[i] = 0.f;
  __syncthreads();
#pragma unroll
  for (int e = 0; e < 8; ++e) atomicAdd(&s_col[cg * 8 + e], csum[e]);
  __syncthreads();
  for (int i = threadIdx.x; i < c; i += blockDim.x) atomicAdd(colsum + i, s_col[i]);
}

static int pool_threads(int c) {  // a multiple of c/8 (fixed channel group per thread)
  const int cv = c / 8;
  return cv <= 256 ? (256 / cv) * cv : 256;
}

// One thread = one input position x 8 channels; loops over the windows covering it.
__global__ void maxpool_bwd_kernel(const __nv_bfloat16* __restrict__ x,
                                   const __nv_bfloat16* __restrict__ dy, int n, int h, int w, int c,
                                   int pi, int k, int st, int po, int oh, int ow,
                                   __nv_bfloat16* __restrict__ dx, float* __restrict__ colsum) {
  __shared__ float s_col[kPoolColsumMax];
  float csum[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const int hp = h + 2 * pi, wp = w + 2 * pi;
  const int ohp = oh + 2 * po, owp = ow + 2 * po;
  const int cv = c / 8;
  const long long total = static_cast<long long>(n) * hp * wp * cv;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int cg = static_cast<int>(i % cv);
    long long pos = i / cv;
    long long img = pos / (hp * wp);
    int r = static_cast<int>(pos - img * hp * wp);
    int py = r / wp, px = r - (r / wp) * wp;
    int iy = py - pi, ix = px - pi;
    float g[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) g[e] = 0.f;
    if (iy >= 0 && iy < h && ix >= 0 && ix < w) {
      uint4 xs = *reinterpret_cast<const uint4*>(x + pos * c + cg * 8);
      const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(&xs);
      // windows oy with oy*st <= iy < oy*st + k
      const int oy0 = iy - k + 1 > 0 ? (iy - k + st) / st : 0;
      const int ox0 = ix - k + 1 > 0 ? (ix - k + st) / st : 0;
      for (int oy = oy0; oy <= iy / st && oy < oh; ++oy) {
        for (int ox = ox0; ox <= ix / st && ox < ow; ++ox) {
          // first argmax (row-major) of window (oy, ox), per channel
          float best[8];
          int arg[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) { best[e] = -INFINITY; arg[e] = -1; }
          for (int ky = 0; ky < k; ++ky) {
            for (int kx = 0; kx < k; ++kx) {
              long long src = ((img * hp + oy * st + ky + pi) * wp + ox * st + kx + pi) * c + cg * 8;
              uint4 u = *reinterpret_cast<const uint4*>(x + src);
              const __nv_bfloat16* hb = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                float v = __bfloat162float(hb[e]);
                if (v > best[e]) { best[e] = v; arg[e] = ky * k + kx; }
              }
            }
          }
          const int mine = (iy - oy * st) * k + (ix - ox * st);
          long long dsrc = ((img * ohp + oy + po) * owp + ox + po) * c + cg * 8;
          uint4 du = *reinterpret_cast<const uint4*>(dy + dsrc);
          const __nv_bfloat16* db = reinterpret_cast<const __nv_bfloat16*>(&du);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (arg[e] == mine) g[e] += __bfloat162float(db[e]);
        }
      }
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (!(__bfloat162float(xb[e]) > 0.f)) g[e] = 0.f;
    }
    uint4 res;
    __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&res);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      ob[e] = __float2bfloat16_rn(g[e]);
      csum[e] += __bfloat162float(ob[e]);
    }
    *reinterpret_cast<uint4*>(dx + pos * c + cg * 8) = res;
  }
  if (colsum != nullptr) block_colsum_flush(csum, threadIdx.x % cv, c, s_col, colsum);
}

// Disjoint windows (stride == window == K): one thread per output window x 8 channels reads
// the K*K inputs and dy once and writes the K*K input gradients.  Positions no window covers
// and the padding border are never written (the executor's gradient buffers are zeroed once).
#ifndef RALPB_POOL_ILP
#define RALPB_POOL_ILP 1  // 2 and 4 measured slower (tools/probe_pool.py: 610 vs 705 vs 978 us)
#endif
template <int K>
__global__ void maxpool_bwd_disjoint_kernel(const __nv_bfloat16* __restrict__ x,
                                            const __nv_bfloat16* __restrict__ dy, int n, int h, int w, int c,
                                            int pi, int po, int oh, int ow, __nv_bfloat16* __restrict__ dx,
                                            float* __restrict__ colsum) {
  __shared__ float s_col[kPoolColsumMax];
  float csum[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const int cv = c >> 3;
  const int total = n * oh * ow * cv;
  const int hp = h + 2 * pi, wp = w + 2 * pi;
  // RALPB_POOL_ILP windows per thread per iteration: all their loads are issued before any
  // compare, so each thread keeps ILP * (K*K + 1) 16-byte loads in flight.
  const int stride = gridDim.x * blockDim.x;
  for (int i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < total; i0 += RALPB_POOL_ILP * stride) {
    long long base_u[RALPB_POOL_ILP];
    uint4 xv_u[RALPB_POOL_ILP][K * K];
    uint4 dv_u[RALPB_POOL_ILP];
#pragma unroll
    for (int u = 0; u < RALPB_POOL_ILP; ++u) {
      const int i = i0 + u * stride;
      if (i >= total) break;
      const int cg = i % cv;
      int t = i / cv;
      const int ox = t % ow;
      t /= ow;
      const int oy = t % oh;
      const int img = t / oh;
      base_u[u] = ((static_cast<long long>(img) * hp + oy * K + pi) * wp + ox * K + pi) * c + cg * 8;
      const long long dyo =
          ((static_cast<long long>(img) * (oh + 2 * po) + oy + po) * (ow + 2 * po) + ox + po) * c + cg * 8;
#pragma unroll
      for (int q = 0; q < K * K; ++q)
        xv_u[u][q] = *reinterpret_cast<const uint4*>(x + base_u[u] + (static_cast<long long>(q / K) * wp + q % K) * c);
      dv_u[u] = *reinterpret_cast<const uint4*>(dy + dyo);
    }
#pragma unroll
    for (int u = 0; u < RALPB_POOL_ILP; ++u) {
    if (i0 + u * stride >= total) break;
    const long long base = base_u[u];
    const uint4* xv = xv_u[u];
    const __nv_bfloat16* db = reinterpret_cast<const __nv_bfloat16*>(&dv_u[u]);
    int arg[8];
    float best[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) { best[e] = -INFINITY; arg[e] = -1; }
#pragma unroll
    for (int q = 0; q < K * K; ++q) {
      const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(&xv[q]);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float v = __bfloat162float(xb[e]);
        if (v > best[e]) { best[e] = v; arg[e] = q; }
      }
    }
#pragma unroll
    for (int q = 0; q < K * K; ++q) {
      const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(&xv[q]);
      uint4 out;
      __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&out);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const bool hit = arg[e] == q && __bfloat162float(xb[e]) > 0.f;
        ob[e] = hit ? db[e] : __float2bfloat16_rn(0.f);
        if (hit) csum[e] += __bfloat162float(db[e]);
      }
      *reinterpret_cast<uint4*>(dx + base + (static_cast<long long>(q / K) * wp + q % K) * c) = out;
    }
    }
  }
  if (colsum != nullptr) block_colsum_flush(csum, threadIdx.x % cv, c, s_col, colsum);
}

// 2x2/2 pool backward from the argmax bytes the fused conv+pool forward recorded
// (conv_slab.cuh): reads 1 byte + 2 bytes per pooled element, writes the 4 input gradients --
// the conv output itself is never read back.
__global__ void maxpool_bwd_idx_kernel(const uint8_t* __restrict__ idx, const __nv_bfloat16* __restrict__ dy, int n,
                                       int oh, int ow, int c, int po, int pi, __nv_bfloat16* __restrict__ dx,
                                       float* __restrict__ colsum) {
  __shared__ float s_col[kPoolColsumMax];
  float csum[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const int cv = c >> 3;
  const long long total = static_cast<long long>(n) * oh * ow * cv;
  const int hp = 2 * oh + 2 * pi, wp = 2 * ow + 2 * pi;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int cg = static_cast<int>(i % cv);
    const long long pix = i / cv;
    const int ox = static_cast<int>(pix % ow);
    const long long t = pix / ow;
    const int oy = static_cast<int>(t % oh);
    const long long img = t / oh;
    const uint2 iw = *reinterpret_cast<const uint2*>(idx + pix * c + cg * 8);
    const uint4 dv = *reinterpret_cast<const uint4*>(dy + ((img * (oh + 2 * po) + oy + po) * (ow + 2 * po) + ox + po) * c + cg * 8);
    const __nv_bfloat16* db = reinterpret_cast<const __nv_bfloat16*>(&dv);
    const uint8_t* ib = reinterpret_cast<const uint8_t*>(&iw);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 out;
      __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&out);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const bool hit = ib[e] == q;
        ob[e] = hit ? db[e] : __float2bfloat16_rn(0.f);
        if (hit) csum[e] += __bfloat162float(db[e]);
      }
      const long long o = ((img * hp + 2 * oy + (q >> 1) + pi) * wp + 2 * ox + (q & 1) + pi) * c + cg * 8;
      *reinterpret_cast<uint4*>(dx + o) = out;
    }
  }
  if (colsum != nullptr) block_colsum_flush(csum, threadIdx.x % cv, c, s_col, colsum);
}

// General k/stride pool backward from argmax bytes (maxpool_fwd with idx): one thread per input
// position x 8 channels gathers dy from the (at most ceil(k/st)^2) windows whose recorded
// argmax is this position -- 8 + 16 bytes per covering window instead of re-reading the
// k*k inputs of every window.
// KC / STC > 0: the window and stride as compile-time constants (AlexNet's overlapping 3/2 pools:
// the covering-window bounds and position arithmetic fold into a few instructions; the kernel is
// instruction-bound on these L2-resident tensors).
template <int KC, int STC>
__global__ void maxpool_bwd_gather_kernel(const uint8_t* __restrict__ idx, const __nv_bfloat16* __restrict__ dy,
                                          int n, int h, int w, int c, int pi, int k_rt, int st_rt, int po, int oh,
                                          int ow, __nv_bfloat16* __restrict__ dx, float* __restrict__ colsum) {
  const int k = KC > 0 ? KC : k_rt;
  const int st = STC > 0 ? STC : st_rt;
  __shared__ float s_col[kPoolColsumMax];
  float csum[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const int cv = c >> 3;
  // 32-bit index arithmetic (the launcher checks n * h * w * cv < 2^31)
  const int total = n * h * w * cv;
  const int hp = h + 2 * pi, wp = w + 2 * pi;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int pix = i / cv;
    const int cg = i - pix * cv;
    const int t = pix / w;
    const int ix = pix - t * w;
    const long long img = t / h;
    const int iy = t - static_cast<int>(img) * h;
    float g[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const int oy0 = iy - k + 1 > 0 ? (iy - k + st) / st : 0;
    const int ox0 = ix - k + 1 > 0 ? (ix - k + st) / st : 0;
    if constexpr (KC > 0 && STC > 0) {
      // compile-time window count per axis: every covering window's idx and dy are loaded at once
      // (the runtime loop serialised a dependent idx -> dy load chain per window)
      constexpr int NW = (KC + STC - 1) / STC;
      const int oy_hi = min(iy / st, oh - 1), ox_hi = min(ix / st, ow - 1);
      uint2 iw[NW][NW];
      uint4 dv[NW][NW];
#pragma unroll
      for (int a = 0; a < NW; ++a)
#pragma unroll
        for (int b = 0; b < NW; ++b) {
          const int oy = oy_hi - a, ox = ox_hi - b;
          iw[a][b] = make_uint2(0xffffffffu, 0xffffffffu);
          dv[a][b] = make_uint4(0, 0, 0, 0);
          if (oy >= oy0 && ox >= ox0) {
            const long long o = (img * oh + oy) * ow + ox;
            iw[a][b] = *reinterpret_cast<const uint2*>(idx + o * c + cg * 8);
            dv[a][b] = *reinterpret_cast<const uint4*>(dy + ((img * (oh + 2 * po) + oy + po) * (ow + 2 * po) + ox + po) * c +
                                                       cg * 8);
          }
        }
#pragma unroll
      for (int a = 0; a < NW; ++a)
#pragma unroll
        for (int b = 0; b < NW; ++b) {
          const int mine = (iy - (oy_hi - a) * st) * k + (ix - (ox_hi - b) * st);
          const uint8_t* ib = reinterpret_cast<const uint8_t*>(&iw[a][b]);
          const __nv_bfloat16* db = reinterpret_cast<const __nv_bfloat16*>(&dv[a][b]);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (ib[e] == mine) g[e] += __bfloat162float(db[e]);
        }
    } else {
      for (int oy = oy0; oy <= iy / st && oy < oh; ++oy) {
        for (int ox = ox0; ox <= ix / st && ox < ow; ++ox) {
          const int mine = (iy - oy * st) * k + (ix - ox * st);
          const long long o = (img * oh + oy) * ow + ox;
          const uint2 iw = *reinterpret_cast<const uint2*>(idx + o * c + cg * 8);
          const uint8_t* ib = reinterpret_cast<const uint8_t*>(&iw);
          bool any = false;
#pragma unroll
          for (int e = 0; e < 8; ++e) any |= ib[e] == mine;
          if (!any) continue;
          const uint4 dv = *reinterpret_cast<const uint4*>(dy + ((img * (oh + 2 * po) + oy + po) * (ow + 2 * po) + ox + po) * c + cg * 8);
          const __nv_bfloat16* db = reinterpret_cast<const __nv_bfloat16*>(&dv);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (ib[e] == mine) g[e] += __bfloat162float(db[e]);
        }
      }
    }
    uint4 res;
    __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&res);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      ob[e] = __float2bfloat16_rn(g[e]);
      csum[e] += __bfloat162float(ob[e]);
    }
    *reinterpret_cast<uint4*>(dx + ((img * hp + iy + pi) * wp + ix + pi) * c + cg * 8) = res;
  }
  if (colsum != nullptr) block_colsum_flush(csum, threadIdx.x % cv, c, s_col, colsum);
}

cudaError_t maxpool_bwd_gather(const uint8_t* idx, const __nv_bfloat16* dy, int n, int h, int w, int c, int pad_in,
                               int k, int st, int pad_out, __nv_bfloat16* dx, float* colsum, cudaStream_t s) {
  if (c % 8 != 0 || (colsum != nullptr && (c > kPoolColsumMax || c / 8 > 256))) return cudaErrorInvalidValue;
  const int oh = (h - k) / st + 1, ow = (w - k) / st + 1;
  const int threads = pool_threads(c);
  const long long work = static_cast<long long>(n) * h * w * (c / 8);
  if (work >= (1LL << 31)) return cudaErrorInvalidValue;
  // with a column sum, 4 resident blocks per SM (each block flushes c atomics at its end); without,
  // a full SM of threads (RALPB_POOL_GATHER_BLOCKS overrides the per-SM block count)
  static const int bps = [] { const char* e = getenv("RALPB_POOL_GATHER_BLOCKS"); return e ? atoi(e) : 8; }();
  const int grid = static_cast<int>(std::max<long long>(1, std::min((work + threads - 1) / threads,
                                                                   static_cast<long long>(num_sms()) *
                                                                       (colsum != nullptr ? 4 : bps))));
  // idx + dy read, dx written (interior)
  const double bytes = static_cast<double>(n) * c * (static_cast<double>(oh) * ow * 3.0 + static_cast<double>(h) * w * 2.0);
  launch_timed([&] {
    if (k == 3 && st == 2)
      maxpool_bwd_gather_kernel<3, 2><<<grid, threads, 0, s>>>(idx, dy, n, h, w, c, pad_in, k, st, pad_out, oh, ow, dx,
                                                               colsum);
    else
      maxpool_bwd_gather_kernel<0, 0><<<grid, threads, 0, s>>>(idx, dy, n, h, w, c, pad_in, k, st, pad_out, oh, ow, dx,
                                                               colsum);
  }, s, KIND_POOL_BWD, 0.0, bytes);
  return cudaGetLastError();
}

cudaError_t maxpool_bwd_idx(const uint8_t* idx, const __nv_bfloat16* dy, int n, int oh, int ow, int c, int pad_out,
                            int pad_in, __nv_bfloat16* dx, float* colsum, cudaStream_t s) {
  if (c % 8 != 0 || (colsum != nullptr && (c > kPoolColsumMax || c / 8 > 256))) return cudaErrorInvalidValue;
  const int threads = pool_threads(c);
  const long long work = static_cast<long long>(n) * oh * ow * (c / 8);
  const int grid = static_cast<int>(std::max<long long>(1, std::min((work + threads - 1) / threads,
                                                                   static_cast<long long>(num_sms()) * 16)));
  const double bytes = static_cast<double>(n) * oh * ow * c * (1.0 + 2.0 + 4 * 2.0);   // idx, dy, 4 dx
  launch_timed([&] { maxpool_bwd_idx_kernel<<<grid, threads, 0, s>>>(idx, dy, n, oh, ow, c, pad_out, pad_in, dx, colsum); },
               s, KIND_POOL_BWD, 0.0, bytes);
  return cudaGetLastError();
}

cudaError_t maxpool_bwd(const __nv_bfloat16* x, const __nv_bfloat16* dy, int n, int h, int w,
                        int c, int pad_in, int k, int st, int pad_out, __nv_bfloat16* dx, float* colsum,
                        cudaStream_t s) {
  if (c % 8 != 0) return cudaErrorInvalidValue;
  if (colsum != nullptr && (c > kPoolColsumMax || c / 8 > 256)) return cudaErrorInvalidValue;
  int oh = (h - k) / st + 1, ow = (w - k) / st + 1;
  const long long windows = static_cast<long long>(n) * oh * ow * (c / 8);
  const int threads = pool_threads(c);
  // (with a fused column sum: one global atomic per channel per block)
  auto grid = [&](long long work) {
    const long long cap = static_cast<long long>(num_sms()) * 16;
    return static_cast<int>(std::max<long long>(1, std::min((work + threads - 1) / threads, cap)));
  };
  // x (interior) + dy read, dx (interior) written
  const double bytes = static_cast<double>(n) * c * (static_cast<double>(h) * w * 4.0 + static_cast<double>(oh) * ow * 2.0);
  if (k == st && k == 2 && windows < (1LL << 31)) {
    launch_timed([&] {
      maxpool_bwd_disjoint_kernel<2><<<grid(windows), threads, 0, s>>>(x, dy, n, h, w, c, pad_in, pad_out, oh, ow, dx,
                                                                       colsum);
    }, s, KIND_POOL_BWD, 0.0, bytes);
    return cudaGetLastError();
  }
  long long total = static_cast<long long>(n) * (h + 2 * pad_in) * (w + 2 * pad_in) * (c / 8);
  launch_timed([&] {
    maxpool_bwd_kernel<<<grid(total), threads, 0, s>>>(x, dy, n, h, w, c, pad_in, k, st, pad_out, oh, ow, dx, colsum);
  }, s, KIND_POOL_BWD, 0.0, bytes);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ softmax cross-entropy
__device__ __forceinline__ float block_reduce(float v, float* sh, bool is_max) {
  for (int o = 16; o > 0; o >>= 1) {
    float u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, u) : v + u;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  v = lane < nw ? sh[lane] : (is_max ? -INFINITY : 0.f);
  for (int o = 16; o > 0; o >>= 1) {
    float u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, u) : v + u;
  }
  return v;
}

__global__ void softmax_xent_kernel(const float* __restrict__ logits, int classes, long long ld,
                                    const int32_t* __restrict__ labels, float scale,
                                    float* __restrict__ row_loss, __nv_bfloat16* __restrict__ dl,
                                    long long ld_d) {
  __shared__ float sh[32];
  const int row = blockIdx.x;
  const float* z = logits + row * ld;
  float mx = -INFINITY;
  for (int j = threadIdx.x; j < classes; j += blockDim.x) mx = fmaxf(mx, z[j]);
  mx = block_reduce(mx, sh, true);
  float se = 0.f;
  for (int j = threadIdx.x; j < classes; j += blockDim.x) se += expf(z[j] - mx);
  se = block_reduce(se, sh, false);
  const float lse = mx + logf(se);
  const int lab = labels[row];
  for (int j = threadIdx.x; j < classes; j += blockDim.x) {
    float pj = expf(z[j] - lse);
    float g = (pj - (j == lab ? 1.f : 0.f)) * scale;
    dl[row * ld_d + j] = __float2bfloat16_rn(g);
  }
  if (threadIdx.x == 0) row_loss[row] = lse - z[lab];
}

cudaError_t softmax_xent(const float* logits, int rows, int classes, long long ld,
                         const int32_t* labels, float scale, float* row_loss,
                         __nv_bfloat16* dlogits, long long ld_d, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  softmax_xent_kernel<<<rows, 256, 0, s>>>(logits, classes, ld, labels, scale, row_loss, dlogits, ld_d);
  return cudaGetLastError();
}

__global__ void reduce_sum_kernel(const float* __restrict__ x, int n, float scale, float* out) {
  __shared__ float sh[32];
  float v = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += x[i];
  v = block_reduce(v, sh, false);
  if (threadIdx.x == 0) out[0] = v * scale;
}

cudaError_t reduce_sum(const float* x, int n, float scale, float* out, cudaStream_t s) {
  reduce_sum_kernel<<<1, 1024, 0, s>>>(x, n, scale, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ SGD momentum
// Optionally also writes the bf16 copy of the updated parameters (the GEMM operand), so the
// fp32 master is not re-read by a separate cast.
__global__ void sgd_kernel(float* __restrict__ p, float* __restrict__ v, const float* __restrict__ g,
                           long long n, float lr, float mu, float gs, __nv_bfloat16* __restrict__ out) {
  long long n4 = n / 4;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float4 pv = reinterpret_cast<float4*>(p)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    float4 gv = reinterpret_cast<const float4*>(g)[i];
    vv.x = mu * vv.x + gs * gv.x; pv.x -= lr * vv.x;
    vv.y = mu * vv.y + gs * gv.y; pv.y -= lr * vv.y;
    vv.z = mu * vv.z + gs * gv.z; pv.z -= lr * vv.z;
    vv.w = mu * vv.w + gs * gv.w; pv.w -= lr * vv.w;
    reinterpret_cast<float4*>(v)[i] = vv;
    reinterpret_cast<float4*>(p)[i] = pv;
    if (out != nullptr) {
      uint2 b;
      b.x = pack_bf16(pv.x, pv.y);
      b.y = pack_bf16(pv.z, pv.w);
      reinterpret_cast<uint2*>(out)[i] = b;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    long long i = n4 * 4 + threadIdx.x;
    v[i] = mu * v[i] + gs * g[i];
    p[i] -= lr * v[i];
    if (out != nullptr) out[i] = __float2bfloat16_rn(p[i]);
  }
}

cudaError_t sgd_momentum(float* p, float* v, const float* g, long long n, float lr, float mu,
                         float gscale, cudaStream_t s) {
  return sgd_momentum_bf16(p, v, g, n, lr, mu, gscale, nullptr, s);
}

cudaError_t sgd_momentum_bf16(float* p, float* v, const float* g, long long n, float lr, float mu,
                              float gscale, __nv_bfloat16* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  // p, v, g read; p, v (+ the bf16 copy) written
  launch_timed([&] { sgd_kernel<<<grid_for(n / 4 + 1, 256), 256, 0, s>>>(p, v, g, n, lr, mu, gscale, out); }, s, KIND_SGD,
               0.0, static_cast<double>(n) * (20.0 + (out != nullptr ? 2.0 : 0.0)));
  return cudaGetLastError();
}

// ------------------------------------------------------------------ bias gradients
// Block = 256 threads covering up to 256*8 channels of a row strip; partial sums in
// registers, one atomic per (block, channel).
__global__ void colsum_kernel(const __nv_bfloat16* __restrict__ dy, long long rows, int c,
                              long long ld, float* __restrict__ db, long long rows_per_block) {
  const int cv = c / 8;
  const int tx = threadIdx.x % 32;       // channel-group lane
  const int ty = threadIdx.x / 32;       // row lane (8 rows in flight)
  long long r0 = blockIdx.x * rows_per_block;
  long long r1 = min(rows, r0 + rows_per_block);
  const int cg = blockIdx.y * 32 + tx;
  const bool valid = cg < cv;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  if (valid) {
    long long r = r0 + ty;
    for (; r + 24 < r1; r += 32) {  // four independent 16-byte loads in flight
      uint4 u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) u[q] = *reinterpret_cast<const uint4*>(dy + (r + 8 * q) * ld + cg * 8);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const __nv_bfloat16* hb = reinterpret_cast<const __nv_bfloat16*>(&u[q]);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += __bfloat162float(hb[e]);
      }
    }
    for (; r < r1; r += 8) {
      uint4 u = *reinterpret_cast<const uint4*>(dy + r * ld + cg * 8);
      const __nv_bfloat16* hb = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += __bfloat162float(hb[e]);
    }
  }
  __shared__ float sh[8][32][9];
#pragma unroll
  for (int e = 0; e < 8; ++e) sh[ty][tx][e] = acc[e];
  __syncthreads();
  if (ty == 0 && valid) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      float t = 0.f;
      for (int j = 0; j < 8; ++j) t += sh[j][tx][e];
      atomicAdd(db + cg * 8 + e, t);
    }
  }
}

// Narrow / ragged widths (e.g. a 10-class logit layer): one thread per column strip.
__global__ void colsum_scalar_kernel(const __nv_bfloat16* __restrict__ dy, long long rows, int c,
                                     long long ld, float* __restrict__ db) {
  const int col = threadIdx.x % 32 + 32 * blockIdx.y;
  const int lane_r = threadIdx.x / 32;
  if (col >= c) return;
  float acc = 0.f;
  for (long long r = blockIdx.x * 8 + lane_r; r < rows; r += 8LL * gridDim.x)
    acc += __bfloat162float(dy[r * ld + col]);
  atomicAdd(db + col, acc);
}

cudaError_t colsum_bf16(const __nv_bfloat16* dy, long long rows, int c, long long ld, float* db,
                        cudaStream_t s) {
  if (c % 8 != 0 || ld % 8 != 0) {
    colsum_scalar_kernel<<<dim3(64, (c + 31) / 32), 256, 0, s>>>(dy, rows, c, ld, db);
    return cudaGetLastError();
  }
  int cv = c / 8;
  int gy = (cv + 31) / 32;
  long long want_blocks = static_cast<long long>(num_sms()) * 8 / gy + 1;
  long long rpb = std::max<long long>(64, (rows + want_blocks - 1) / want_blocks);
  long long gx = (rows + rpb - 1) / rpb;
  colsum_kernel<<<dim3(static_cast<unsigned>(gx), gy), 256, 0, s>>>(dy, rows, c, ld, db, rpb);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ partial sums (RALP_MPS)
__global__ void sum_partials_kernel(PartialSum ps, int rows, int cols, long long ld, const float* __restrict__ bias,
                                    int relu, __nv_bfloat16* __restrict__ out_bf16, float* __restrict__ out_f32,
                                    long long ld_out) {
  const long long total = static_cast<long long>(rows) * cols;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / cols;
    const int c = static_cast<int>(i - r * cols);
    float v = bias != nullptr ? bias[c] : 0.f;
    for (int p = 0; p < ps.n; ++p) v += ps.part[p][r * ld + c];
    if (relu) v = fmaxf(v, 0.f);
    if (out_bf16 != nullptr) out_bf16[r * ld_out + c] = __float2bfloat16_rn(v);
    else out_f32[r * ld_out + c] = v;
  }
}

cudaError_t sum_partials(const PartialSum& ps, int rows, int cols, long long ld, const float* bias, int relu,
                         __nv_bfloat16* out_bf16, float* out_f32, long long ld_out, cudaStream_t s) {
  const long long total = static_cast<long long>(rows) * cols;
  if (total == 0) return cudaSuccess;
  sum_partials_kernel<<<grid_for(total, 256), 256, 0, s>>>(ps, rows, cols, ld, bias, relu, out_bf16, out_f32, ld_out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ weight re-layouts
// All conv layers' filter copies in one launch: every block transposes 32 (co) x 32 (ci) of one tap
// through shared memory, so both the forward copy wf [co][t][ci] and the tap-reversed transpose
// wd [ci][taps-1-t][co] are written with coalesced rows.
__global__ void __launch_bounds__(256) conv_weight_prep_kernel(const __grid_constant__ WeightPrepBatch b) {
  __shared__ float tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (long long blk = blockIdx.x; blk < b.total_blocks; blk += gridDim.x) {
    int k = 0;
    while (k + 1 < b.n && blk >= b.job[k + 1].block0) ++k;
    const WeightPrepJob& J = b.job[k];
    long long r = blk - J.block0;
    const int tci = static_cast<int>(r % J.tiles_ci);
    r /= J.tiles_ci;
    const int tco = static_cast<int>(r % J.tiles_co);
    const int t = static_cast<int>(r / J.tiles_co);
    const int co0 = tco * 32, ci0 = tci * 32;
    for (int yy = ty; yy < 32; yy += 8) {
      const int co = co0 + yy, ci = ci0 + tx;
      if (co < J.co && ci < J.ci) {
        const long long i = (static_cast<long long>(co) * J.taps + t) * J.ci + ci;
        const float v = J.w[i];
        if (J.wf != nullptr) J.wf[i] = __float2bfloat16_rn(v);
        tile[yy][tx] = v;
      }
    }
    __syncthreads();
    if (J.wd != nullptr) {
      for (int yy = ty; yy < 32; yy += 8) {
        const int ci = ci0 + yy, co = co0 + tx;
        if (co < J.co && ci < J.ci)
          J.wd[(static_cast<long long>(ci) * J.taps + (J.taps - 1 - t)) * J.co + co] = __float2bfloat16_rn(tile[tx][yy]);
      }
    }
    __syncthreads();
  }
}

cudaError_t conv_weight_prep_batch(const WeightPrepJob* jobs, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (n > kMaxPrepJobs) return cudaErrorInvalidValue;
  WeightPrepBatch b;
  b.n = n;
  long long blocks = 0;
  for (int i = 0; i < n; ++i) {
    b.job[i] = jobs[i];
    b.job[i].tiles_co = (jobs[i].co + 31) / 32;
    b.job[i].tiles_ci = (jobs[i].ci + 31) / 32;
    b.job[i].block0 = blocks;
    blocks += static_cast<long long>(b.job[i].tiles_co) * b.job[i].tiles_ci * jobs[i].taps;
  }
  b.total_blocks = blocks;
  const int grid = static_cast<int>(std::min<long long>(blocks, static_cast<long long>(num_sms()) * 8));
  conv_weight_prep_kernel<<<grid, 256, 0, s>>>(b);
  return cudaGetLastError();
}

cudaError_t conv_weight_prep(const float* w, int co, int taps, int ci, __nv_bfloat16* wf,
                             __nv_bfloat16* wd, cudaStream_t s) {
  WeightPrepJob j{};
  j.w = w; j.wf = wf; j.wd = wd; j.co = co; j.taps = taps; j.ci = ci;
  return conv_weight_prep_batch(&j, 1, s);
}

__global__ void cast_kernel(const float* __restrict__ x, long long n, __nv_bfloat16* __restrict__ y) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    y[i] = __float2bfloat16_rn(x[i]);
}

cudaError_t cast_bf16(const float* x, long long n, __nv_bfloat16* y, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  cast_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, n, y);
  return cudaGetLastError();
}

struct CastBatch {
  CastJob j[kMaxCastJobs];
  long long start[kMaxCastJobs + 1];   // first 4-element chunk of each job
  int n;
};
// thread = one 4-element chunk of one job (jobs located by binary search over the chunk starts)
__global__ void cast_batch_kernel(const __grid_constant__ CastBatch b) {
  const long long total = b.start[b.n];
  for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < total;
       v += static_cast<long long>(gridDim.x) * blockDim.x) {
    int lo = 0, hi = b.n - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (b.start[mid] <= v) lo = mid; else hi = mid - 1;
    }
    const CastJob& j = b.j[lo];
    const long long o = (v - b.start[lo]) * 4;
    if (o + 4 <= j.n) {
      const float4 f = *reinterpret_cast<const float4*>(j.x + o);
      __nv_bfloat162 p0 = __floats2bfloat162_rn(f.x, f.y), p1 = __floats2bfloat162_rn(f.z, f.w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&p0);
      u.y = *reinterpret_cast<uint32_t*>(&p1);
      *reinterpret_cast<uint2*>(j.y + o) = u;
    } else {
      for (long long e = o; e < j.n; ++e) j.y[e] = __float2bfloat16_rn(j.x[e]);
    }
  }
}

cudaError_t cast_bf16_batch(const CastJob* jobs, int n, cudaStream_t s) {
  for (int base = 0; base < n; base += kMaxCastJobs) {
    CastBatch b{};
    b.n = std::min(kMaxCastJobs, n - base);
    b.start[0] = 0;
    for (int i = 0; i < b.n; ++i) {
      b.j[i] = jobs[base + i];
      if ((reinterpret_cast<uintptr_t>(b.j[i].x) & 15) || (reinterpret_cast<uintptr_t>(b.j[i].y) & 7))
        return cudaErrorMisalignedAddress;
      b.start[i + 1] = b.start[i] + (b.j[i].n + 3) / 4;
    }
    if (b.start[b.n] == 0) continue;
    cast_batch_kernel<<<grid_for(b.start[b.n], 256), 256, 0, s>>>(b);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace ralpb

namespace ralpb {

// out = act(acc + bias) [* (mask > 0)] for split-K GEMM results (fp32 accumulators).
__global__ void gemm_finalize_kernel(const float* __restrict__ acc, int rows, int cols, long long ld_acc,
                                     const float* __restrict__ bias, int relu, const __nv_bfloat16* __restrict__ mask,
                                     long long ld_mask, __nv_bfloat16* __restrict__ out_bf16, float* __restrict__ out_f32,
                                     long long ld_out) {
  const long long total = static_cast<long long>(rows) * cols;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / cols;
    const int c = static_cast<int>(i - r * cols);
    float v = acc[r * ld_acc + c];
    if (bias != nullptr) v += bias[c];
    if (relu) v = fmaxf(v, 0.f);
    if (mask != nullptr && !(__bfloat162float(mask[r * ld_mask + c]) > 0.f)) v = 0.f;
    if (out_bf16 != nullptr) out_bf16[r * ld_out + c] = __float2bfloat16_rn(v);
    if (out_f32 != nullptr) out_f32[r * ld_out + c] = v;
  }
}

cudaError_t gemm_finalize(const float* acc, int rows, int cols, long long ld_acc, const float* bias, int relu,
                          const __nv_bfloat16* mask, long long ld_mask, __nv_bfloat16* out_bf16, float* out_f32,
                          long long ld_out, cudaStream_t s) {
  const long long total = static_cast<long long>(rows) * cols;
  if (total <= 0) return cudaSuccess;
  gemm_finalize_kernel<<<grid_for(total, 256), 256, 0, s>>>(acc, rows, cols, ld_acc, bias, relu, mask, ld_mask,
                                                            out_bf16, out_f32, ld_out);
  return cudaGetLastError();
}

}  // namespace ralpb
