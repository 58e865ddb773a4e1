// Kernels of the parity precision: fp32-accurate (hi, lo) bf16 pairs (see pair.cuh).  Every
// contraction runs on the tcgen05 GEMM engine; these are the HBM-bound passes around it
// (operand layouts, the finishing sums with bias / ReLU / mask, pools, loss).
#include <algorithm>
#include "gemm_host.cuh"
#include "pair.cuh"

namespace ralpb {

namespace {

int grid_for(long long work, int threads) {
  const long long blocks = (work + threads - 1) / threads;
  const long long cap = static_cast<long long>(num_sms()) * 16;
  return static_cast<int>(std::max<long long>(1, std::min(blocks, cap)));
}

constexpr int kMaxPieces = 3;

// v -> P bf16 pieces, most significant first: piece_a = bf16_rn(v - sum_{b<a} piece_b).
__device__ __forceinline__ void split(float v, int P, __nv_bfloat16* pc) {
  float r = v;
#pragma unroll
  for (int a = 0; a < kMaxPieces; ++a) {
    if (a < P) {
      pc[a] = __float2bfloat16_rn(r);
      r -= __bfloat162float(pc[a]);
    }
  }
}
__device__ __forceinline__ bool border_row(long long q, int img_rows, int wp, int pad, int h, int w) {
  const int r = static_cast<int>(q % img_rows);
  const int ph = r / wp, pw = r - (r / wp) * wp;
  return ph < pad || ph >= h + pad || pw < pad || pw >= w + pad;
}

#define GRID_STRIDE(i, total) \
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < (total); \
       i += static_cast<long long>(gridDim.x) * blockDim.x)

// ------------------------------------------------------------------ operand layouts
__global__ void pair_im2col_kernel(const float* __restrict__ x, int n, int h, int w, int c, int k, int st, int p,
                                   int ho, int wo, int po, int kpad, __nv_bfloat16* __restrict__ out, int P) {
  const int hop = ho + 2 * po, wop = wo + 2 * po;
  const int kk = k * k * c;
  const long long total = static_cast<long long>(n) * hop * wop * kpad;
  GRID_STRIDE(i, total) {
    const int j = static_cast<int>(i % kpad);
    const long long row = i / kpad;
    const long long img = row / (static_cast<long long>(hop) * wop);
    const int rem = static_cast<int>(row - img * hop * wop);
    const int oy = rem / wop - po, ox = rem % wop - po;
    float v = 0.f;
    if (oy >= 0 && oy < ho && ox >= 0 && ox < wo) {
      if (j < kk) {
        const int ch = j % c, tap = j / c;
        const int iy = oy * st + tap / k - p, ix = ox * st + tap % k - p;
        if (iy >= 0 && iy < h && ix >= 0 && ix < w) v = x[((img * h + iy) * w + ix) * c + ch];
      } else if (j == kk) {
        v = 1.f;
      }
    }
    __nv_bfloat16 pc[kMaxPieces];
    split(v, P, pc);
    for (int a = 0; a < P; ++a) out[(row * P + a) * kpad + j] = pc[a];
  }
}

__global__ void pair_prep_conv_kernel(const float* __restrict__ w, int co, int taps, int ci,
                                      __nv_bfloat16* __restrict__ wf2, __nv_bfloat16* __restrict__ wd2, int P) {
  const long long total = static_cast<long long>(co) * taps * ci;
  GRID_STRIDE(i, total) {
    const int c = static_cast<int>(i % ci);
    const long long ot = i / ci;
    const int t = static_cast<int>(ot % taps);
    const int o = static_cast<int>(ot / taps);
    __nv_bfloat16 pc[kMaxPieces];
    split(w[i], P, pc);
    for (int a = 0; a < P; ++a)
      for (int b = 0; b < P; ++b) {
        // forward: rows (a, o), columns (t, b, c)
        wf2[((static_cast<long long>(a) * co + o) * taps + t) * P * ci + b * ci + c] = pc[a];
        // backward-data: rows (a, c), columns (taps-1-t, b, o)
        if (wd2 != nullptr)
          wd2[((static_cast<long long>(a) * ci + c) * taps + (taps - 1 - t)) * P * co + b * co + o] = pc[a];
      }
  }
}

__global__ void pair_prep_mat_kernel(const float* __restrict__ w, int out, int ld_out, int groups, int c,
                                     __nv_bfloat16* __restrict__ bf, __nv_bfloat16* __restrict__ bd, int P) {
  const long long in = static_cast<long long>(groups) * c;
  const long long total = static_cast<long long>(ld_out) * in;
  GRID_STRIDE(i, total) {
    const long long k = i % in;
    const int n = static_cast<int>(i / in);
    const int g = static_cast<int>(k / c), cc = static_cast<int>(k - static_cast<long long>(g) * c);
    __nv_bfloat16 pc[kMaxPieces];
    split(n < out ? w[static_cast<long long>(n) * in + k] : 0.f, P, pc);
    for (int a = 0; a < P; ++a)
      for (int b = 0; b < P; ++b) {
        const long long col = (static_cast<long long>(g) * P + b) * c + cc;
        const long long row = static_cast<long long>(a) * ld_out + n;
        bf[row * P * in + col] = pc[a];
        if (bd != nullptr) bd[row * P * in + col] = pc[b];
      }
  }
}

// ------------------------------------------------------------------ finishing passes
__global__ void pair_finish_kernel(PairFinish f) {
  const long long total = f.rows * f.n;
  GRID_STRIDE(i, total) {
    const int n = static_cast<int>(i % f.n);
    const long long q = i / f.n;
    if (f.border && border_row(q, f.img_rows, f.wp, f.pad, f.h, f.w)) continue;
    const int P = f.pieces;
    const float* a = f.acc + q * P * f.ld;
    float v = 0.f;
    for (int b = 0; b < P; ++b) v += a[b * f.ld + n];
    if (f.bias != nullptr) v += f.bias[n];
    if (f.relu) v = fmaxf(v, 0.f);
    if (f.mask != nullptr && !(__bfloat162float(f.mask[q * P * f.ld + n]) > 0.f)) v = 0.f;
    if (f.out2 != nullptr) {
      __nv_bfloat16 pc[kMaxPieces];
      split(v, P, pc);
      for (int b = 0; b < P; ++b) f.out2[(q * P + b) * f.ld + n] = pc[b];
    }
    if (f.out_f32 != nullptr) f.out_f32[q * f.ld_f32 + n] = v;
  }
}

__global__ void pair_finish_groups_kernel(PairFinishGroups f) {
  const long long row_elems = static_cast<long long>(f.groups) * f.c;
  const long long total = f.rows * row_elems;
  GRID_STRIDE(i, total) {
    const long long k = i % row_elems;
    const long long q = i / row_elems;
    if (f.border && border_row(q, f.img_rows, f.wp, f.pad, f.h, f.w)) continue;
    const int P = f.pieces;
    const int g = static_cast<int>(k / f.c), c = static_cast<int>(k - static_cast<long long>(g) * f.c);
    const long long base = q * P * row_elems + static_cast<long long>(g) * P * f.c;
    float v = 0.f;
    for (int b = 0; b < P; ++b) v += f.acc[base + b * f.c + c];
    if (f.mask != nullptr && !(__bfloat162float(f.mask[base + c]) > 0.f)) v = 0.f;
    __nv_bfloat16 pc[kMaxPieces];
    split(v, P, pc);
    for (int b = 0; b < P; ++b) f.out2[base + b * f.c + c] = pc[b];
  }
}

// ------------------------------------------------------------------ max pool
__global__ void pair_pool_fwd_kernel(const __nv_bfloat16* __restrict__ x, int n, int h, int w, int c, int pi, int k,
                                     int st, __nv_bfloat16* __restrict__ y, int po, int oh, int ow,
                                     uint8_t* __restrict__ idx, int P) {
  const int hp = h + 2 * pi, wp = w + 2 * pi;
  const long long total = static_cast<long long>(n) * oh * ow * c;
  GRID_STRIDE(i, total) {
    const int ch = static_cast<int>(i % c);
    const long long pos = i / c;
    const int ox = static_cast<int>(pos % ow);
    const long long t = pos / ow;
    const int oy = static_cast<int>(t % oh);
    const long long img = t / oh;
    float best = 0.f;
    long long best_px = 0;
    int arg = -1;
    for (int ky = 0; ky < k; ++ky)
      for (int kx = 0; kx < k; ++kx) {
        const long long px = (img * hp + oy * st + ky + pi) * wp + ox * st + kx + pi;
        // pieces decrease in magnitude, so summing from the least significant is exact enough and
        // ordering matches the value they carry
        float v = 0.f;
        for (int b = P - 1; b >= 0; --b) v += __bfloat162float(x[(px * P + b) * c + ch]);
        if (arg < 0 || v > best) { best = v; best_px = px; arg = ky * k + kx; }
      }
    const long long op = (img * (oh + 2 * po) + oy + po) * (ow + 2 * po) + ox + po;
    for (int b = 0; b < P; ++b) y[(op * P + b) * c + ch] = x[(best_px * P + b) * c + ch];
    idx[i] = best > 0.f ? static_cast<uint8_t>(arg) : static_cast<uint8_t>(255);
  }
}

// One thread per input element: gathers every window that covers it.
__global__ void pair_pool_bwd_kernel(const uint8_t* __restrict__ idx, const __nv_bfloat16* __restrict__ dy, int n,
                                     int h, int w, int c, int pi, int k, int st, int po, __nv_bfloat16* __restrict__ dx,
                                     float* __restrict__ colsum, int P) {
  const int oh = (h - k) / st + 1, ow = (w - k) / st + 1;
  const int hp = h + 2 * pi, wp = w + 2 * pi;
  const long long total = static_cast<long long>(n) * h * w * c;
  GRID_STRIDE(i, total) {
    const int ch = static_cast<int>(i % c);
    const long long pos = i / c;
    const int x0 = static_cast<int>(pos % w);
    const long long t = pos / w;
    const int y0 = static_cast<int>(t % h);
    const long long img = t / h;
    float acc = 0.f;
    // windows (oy, ox) with oy*st <= y0 < oy*st + k
    const int oy_lo = y0 >= k ? (y0 - k) / st + 1 : 0, oy_hi = min(oh - 1, y0 / st);
    const int ox_lo = x0 >= k ? (x0 - k) / st + 1 : 0, ox_hi = min(ow - 1, x0 / st);
    for (int oy = oy_lo; oy <= oy_hi; ++oy)
      for (int ox = ox_lo; ox <= ox_hi; ++ox) {
        const int pos_in_win = (y0 - oy * st) * k + (x0 - ox * st);
        if (idx[((img * oh + oy) * ow + ox) * c + ch] != pos_in_win) continue;
        const long long op = (img * (oh + 2 * po) + oy + po) * (ow + 2 * po) + ox + po;
        for (int b = P - 1; b >= 0; --b) acc += __bfloat162float(dy[(op * P + b) * c + ch]);
      }
    __nv_bfloat16 pc[kMaxPieces];
    split(acc, P, pc);
    const long long px = (img * hp + y0 + pi) * wp + x0 + pi;
    for (int b = 0; b < P; ++b) dx[(px * P + b) * c + ch] = pc[b];
    if (colsum != nullptr && acc != 0.f) atomicAdd(colsum + ch, acc);
  }
}

// ------------------------------------------------------------------ reductions
// One block per 32 columns x (rows / gridDim.y) rows; warp-shuffle-free fp32 partial sums.
__global__ void pair_colsum_kernel(const __nv_bfloat16* __restrict__ x2, long long rows, int n, int ld,
                                   float* __restrict__ db, int P) {
  const int col = blockIdx.x * 32 + (threadIdx.x & 31);
  const int r0 = threadIdx.x >> 5;
  const int rstep = blockDim.x >> 5;
  if (col >= n) return;
  float acc = 0.f;
  for (long long r = blockIdx.y * static_cast<long long>(rstep) + r0; r < rows;
       r += static_cast<long long>(gridDim.y) * rstep)
    for (int b = P - 1; b >= 0; --b) acc += __bfloat162float(x2[(r * P + b) * ld + col]);
  atomicAdd(db + col, acc);
}

__global__ void pair_reduce_wgrad_kernel(const float* __restrict__ S, int m_rows, int m_valid, int t_count, int c,
                                         float* __restrict__ g, long long g_ld, int P) {
  const long long tc = static_cast<long long>(t_count) * c;
  const long long total = static_cast<long long>(m_valid) * tc;
  GRID_STRIDE(i, total) {
    const long long r = i % tc;
    const int m = static_cast<int>(i / tc);
    const int t = static_cast<int>(r / c), cc = static_cast<int>(r - static_cast<long long>(t) * c);
    float v = 0.f;
    for (int a = P - 1; a >= 0; --a) {
      const float* row = S + (static_cast<long long>(a) * m_rows + m) * t_count * P * c + static_cast<long long>(t) * P * c;
      for (int b = P - 1; b >= 0; --b) v += row[b * c + cc];
    }
    g[m * g_ld + r] = v;
  }
}

__global__ void pair_softmax_kernel(const float* __restrict__ logits, int rows, int classes, int ld,
                                    const int32_t* __restrict__ labels, float scale, float* __restrict__ row_loss,
                                    __nv_bfloat16* __restrict__ d2, int P) {
  // one warp per row
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const float* z = logits + static_cast<long long>(warp) * ld;
  float mx = -INFINITY;
  for (int j = lane; j < classes; j += 32) mx = fmaxf(mx, z[j]);
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  double sum = 0.0;
  for (int j = lane; j < classes; j += 32) sum += exp(static_cast<double>(z[j] - mx));
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const double lse = log(sum) + mx;
  const int lab = labels[warp];
  if (lane == 0) row_loss[warp] = static_cast<float>(lse - z[lab]);
  __nv_bfloat16* d = d2 + static_cast<long long>(warp) * P * ld;
  for (int j = lane; j < classes; j += 32) {
    const float p = static_cast<float>(exp(static_cast<double>(z[j]) - lse));
    const float v = (p - (j == lab ? 1.f : 0.f)) * scale;
    __nv_bfloat16 pc[kMaxPieces];
    split(v, P, pc);
    for (int b = 0; b < P; ++b) d[b * ld + j] = pc[b];
  }
}

}  // namespace

cudaError_t pair_pack_im2col(const float* x, int n, int h, int w, int c, int k, int st, int p, int ho, int wo, int po,
                             int kpad, __nv_bfloat16* out, int P, cudaStream_t s) {
  const long long total = static_cast<long long>(n) * (ho + 2 * po) * (wo + 2 * po) * kpad;
  pair_im2col_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, n, h, w, c, k, st, p, ho, wo, po, kpad, out, P);
  return cudaGetLastError();
}

cudaError_t pair_prep_conv(const float* w, int co, int taps, int ci, __nv_bfloat16* wf2, __nv_bfloat16* wd2, int P,
                           cudaStream_t s) {
  const long long total = static_cast<long long>(co) * taps * ci;
  pair_prep_conv_kernel<<<grid_for(total, 256), 256, 0, s>>>(w, co, taps, ci, wf2, wd2, P);
  return cudaGetLastError();
}

cudaError_t pair_prep_mat(const float* w, int out, int ld_out, int groups, int c, __nv_bfloat16* bf,
                          __nv_bfloat16* bd, int P, cudaStream_t s) {
  const long long total = static_cast<long long>(ld_out) * groups * c;
  pair_prep_mat_kernel<<<grid_for(total, 256), 256, 0, s>>>(w, out, ld_out, groups, c, bf, bd, P);
  return cudaGetLastError();
}

cudaError_t pair_finish(const PairFinish& f, cudaStream_t s) {
  pair_finish_kernel<<<grid_for(f.rows * f.n, 256), 256, 0, s>>>(f);
  return cudaGetLastError();
}

cudaError_t pair_finish_groups(const PairFinishGroups& f, cudaStream_t s) {
  pair_finish_groups_kernel<<<grid_for(f.rows * f.groups * static_cast<long long>(f.c), 256), 256, 0, s>>>(f);
  return cudaGetLastError();
}

cudaError_t pair_maxpool_fwd(const __nv_bfloat16* x, int n, int h, int w, int c, int pi, int k, int st,
                             __nv_bfloat16* y, int po, uint8_t* idx, int P, cudaStream_t s) {
  const int oh = (h - k) / st + 1, ow = (w - k) / st + 1;
  const long long total = static_cast<long long>(n) * oh * ow * c;
  pair_pool_fwd_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, n, h, w, c, pi, k, st, y, po, oh, ow, idx, P);
  return cudaGetLastError();
}

cudaError_t pair_maxpool_bwd(const uint8_t* idx, const __nv_bfloat16* dy, int n, int h, int w, int c, int pi, int k,
                             int st, int po, __nv_bfloat16* dx, float* colsum, int P, cudaStream_t s) {
  const long long total = static_cast<long long>(n) * h * w * c;
  pair_pool_bwd_kernel<<<grid_for(total, 256), 256, 0, s>>>(idx, dy, n, h, w, c, pi, k, st, po, dx, colsum, P);
  return cudaGetLastError();
}

cudaError_t pair_colsum(const __nv_bfloat16* x2, long long rows, int n, int ld, float* db, int P, cudaStream_t s) {
  const int gx = (n + 31) / 32;
  const long long want = std::max<long long>(1, 4LL * num_sms() / gx);
  const int gy = static_cast<int>(std::min<long long>(want, (rows + 7) / 8));
  pair_colsum_kernel<<<dim3(gx, std::max(gy, 1)), 256, 0, s>>>(x2, rows, n, ld, db, P);
  return cudaGetLastError();
}

cudaError_t pair_reduce_wgrad(const float* S, int m_rows, int m_valid, int t_count, int c, float* g, long long g_ld,
                              int P, cudaStream_t s) {
  const long long total = static_cast<long long>(m_valid) * t_count * c;
  pair_reduce_wgrad_kernel<<<grid_for(total, 256), 256, 0, s>>>(S, m_rows, m_valid, t_count, c, g, g_ld, P);
  return cudaGetLastError();
}

cudaError_t pair_softmax_xent(const float* logits, int rows, int classes, int ld, const int32_t* labels, float scale,
                              float* row_loss, __nv_bfloat16* dlogits2, int P, cudaStream_t s) {
  const int threads = 256;
  const int blocks = (rows * 32 + threads - 1) / threads;
  pair_softmax_kernel<<<blocks, threads, 0, s>>>(logits, rows, classes, ld, labels, scale, row_loss, dlogits2, P);
  return cudaGetLastError();
}

}  // namespace ralpb
