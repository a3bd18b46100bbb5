// Memory-bound kernels of the training step (HBM-bound; vectorised NHWC).
//   layout conversion     NCHW fp32 <-> NHWC views (input tiles, reference tensors)
//   avgpool / upsample    ops.py:133-141 forward, ops.py:186-194 VJPs
//   add / relu mask       elementwise-add VJP fan-out (ops.py:197-198), relu VJP (ops.py:176-177)
//   bias gradient         bias_add VJP sum over N,H,W (ops.py:172-175), deterministic two-pass
//   weight packing        fp32 HWIO master -> bf16 fprop / dgrad operand layouts
#include <cuda_bf16.h>

#include <algorithm>

#include "internal.h"

namespace b2 {

__device__ __forceinline__ float ld_bf(const b2h* p) { return h_to_f(*p); }
__device__ __forceinline__ float bf16_lo(uint32_t v) { return h_lo(v); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return h_hi(v); }

static int grid1d(long long total, int per_thread = 1) {
  long long blocks = (total / per_thread + 255) / 256;
  return static_cast<int>(std::max<long long>(1, std::min<long long>(blocks, 16LL * num_sms())));
}

// ------------------------------------------------------------------ layout
__global__ void k_nchw_to_nhwc(const float* __restrict__ x, void* __restrict__ y, int f32, int n, int c, int h, int w,
                               int cs) {
  // one thread per (n, y, x, channel-pair) reading strided NCHW; fine for input tiles
  const long long hw = static_cast<long long>(h) * w;
  const long long total = n * hw * c;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    // i enumerates NCHW order -> coalesced reads
    long long pix = i % hw;
    long long r = i / hw;
    int ch = static_cast<int>(r % c);
    long long img = r / c;
    const long long d = (img * hw + pix) * cs + ch;
    if (f32)
      reinterpret_cast<float*>(y)[d] = x[i];
    else
      reinterpret_cast<b2h*>(y)[d] = f_to_h(x[i]);
  }
}
constexpr int HALO_COLS = 256;  // one thread per pixel column of a row
__device__ __forceinline__ uint32_t halo_pack2(float a, float b) {  // a -> low half
  const b2h2 t = h2_from(a, b);
  return *reinterpret_cast<const uint32_t*>(&t);
}
// NCHW fp32 -> NHWC bf16 with zeroed halo columns.  One thread per pixel: each of its c channel
// loads is a coalesced 128-byte warp access of one plane row, and its 2c output bytes are
// written as 16-byte pieces adjacent to the neighbouring threads' (no shared-memory transpose).
__global__ void __launch_bounds__(HALO_COLS) k_nchw_to_nhwc_halo(const float* __restrict__ x,
                                                                 b2h* __restrict__ y, int c, int h, int w,
                                                                 int wp, int left) {
  const int col = blockIdx.x * HALO_COLS + threadIdx.x, row = blockIdx.y, img = blockIdx.z;
  const long long plane = static_cast<long long>(h) * w;
  b2h* dst_row = y + (static_cast<long long>(img) * h + row) * wp * c;
  const int vec = c / 8;  // 16-byte pieces per pixel
  if (col < w) {
    const float* src = x + static_cast<long long>(img) * c * plane + static_cast<long long>(row) * w + col;
    uint4* dst = reinterpret_cast<uint4*>(dst_row + static_cast<long long>(left + col) * c);
    for (int pc = 0; pc < vec; ++pc) {
      float v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = __ldg(src + (pc * 8 + e) * plane);
      uint4 o;
      o.x = halo_pack2(v[0], v[1]);
      o.y = halo_pack2(v[2], v[3]);
      o.z = halo_pack2(v[4], v[5]);
      o.w = halo_pack2(v[6], v[7]);
      dst[pc] = o;
    }
  }
  if (blockIdx.x == 0) {  // zero halo columns of this row
    const int nh = wp - w;
    for (int i = threadIdx.x; i < nh * vec; i += HALO_COLS) {
      const int k = i / vec, pc = i - k * vec;
      const int hc = k < left ? k : w + k;
      *reinterpret_cast<uint4*>(dst_row + static_cast<long long>(hc) * c + pc * 8) = make_uint4(0, 0, 0, 0);
    }
  }
}

__global__ void k_nhwc_to_nchw(const void* __restrict__ x, int f32, float* __restrict__ y, int n, int c, int h, int w,
                               int cs) {
  const long long hw = static_cast<long long>(h) * w;
  const long long total = n * hw * c;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long pix = i % hw;
    long long r = i / hw;
    int ch = static_cast<int>(r % c);
    long long img = r / c;
    long long src = (img * hw + pix) * cs + ch;
    y[i] = f32 ? reinterpret_cast<const float*>(x)[src] : h_to_f(reinterpret_cast<const b2h*>(x)[src]);
  }
}

// ------------------------------------------------------------------ pool / upsample
// 8-channel (16 B) vector helpers; G = 8 on aligned views, 1 otherwise
template <int G>
__device__ __forceinline__ void ldv(const b2h* p, float* v) {
  if constexpr (G == 8) {
    uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[2 * e] = h_lo(w[e]);
      v[2 * e + 1] = h_hi(w[e]);
    }
  } else {
    v[0] = ld_bf(p);
  }
}
template <int G>
__device__ __forceinline__ void ldv_rw(const b2h* p, float* v) {  // plain load (data written in place)
  if constexpr (G == 8) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[2 * e] = h_lo(w[e]);
      v[2 * e + 1] = h_hi(w[e]);
    }
  } else {
    v[0] = ld_bf(p);
  }
}
template <int G>
__device__ __forceinline__ void stv(b2h* p, const float* v) {
  if constexpr (G == 8) {
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      b2h2 t = h2_from(v[2 * e], v[2 * e + 1]);
      w[e] = *reinterpret_cast<uint32_t*>(&t);
    }
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  } else {
    *p = f_to_h(v[0]);
  }
}
// d <- mask(m) * v  [+ d]
template <int G>
__device__ __forceinline__ void finish(float* v, const b2h* m, b2h* d, int acc) {
  if (m) {
    float mv[G];
    ldv<G>(m, mv);
#pragma unroll
    for (int e = 0; e < G; ++e)
      if (!(mv[e] > 0.f)) v[e] = 0.f;
  }
  if (acc) {
    float o[G];
    ldv_rw<G>(d, o);
#pragma unroll
    for (int e = 0; e < G; ++e) v[e] += o[e];
  }
  stv<G>(d, v);
}

template <int G>
__global__ void k_avgpool_fwd(const b2h* __restrict__ x, int xs, b2h* __restrict__ y, int ys,
                              int n, int ho, int wo, int c, int k) {
  const int W = wo * k;
  const int cg = c / G;
  const long long total = static_cast<long long>(n) * ho * wo * cg;
  const float inv = 1.f / (k * k);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i % cg) * G;
    const long long op = i / cg;
    const int ox = static_cast<int>(op % wo);
    const long long r = op / wo;
    const int oy = static_cast<int>(r % ho);
    const long long img = r / ho;
    float s[G] = {};
    if constexpr (G == 8) {
      if (k == 4) {  // the stem pool: all 16 loads in flight, then summed in the generic order
        uint4 raw[16];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b)
            raw[4 * a + b] = __ldg(reinterpret_cast<const uint4*>(
                x + ((img * ho * 4 + oy * 4 + a) * W + ox * 4 + b) * xs + ch));
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const uint32_t w4[4] = {raw[t].x, raw[t].y, raw[t].z, raw[t].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            s[2 * e] += h_lo(w4[e]);
            s[2 * e + 1] += h_hi(w4[e]);
          }
        }
#pragma unroll
        for (int e = 0; e < G; ++e) s[e] *= inv;
        stv<G>(y + op * ys + ch, s);
        continue;
      }
    }
    for (int a = 0; a < k; ++a) {
      const b2h* row = x + ((img * ho * k + oy * k + a) * W + ox * k) * xs + ch;
      for (int b = 0; b < k; ++b) {
        float v[G];
        ldv<G>(row + static_cast<long long>(b) * xs, v);
#pragma unroll
        for (int e = 0; e < G; ++e) s[e] += v[e];
      }
    }
#pragma unroll
    for (int e = 0; e < G; ++e) s[e] *= inv;
    stv<G>(y + op * ys + ch, s);
  }
}
// dx[p] (+)= mask(x)[p] * dy[pool(p)] / k^2
template <int G>
__global__ void k_avgpool_bwd(const b2h* __restrict__ dy, int dys, b2h* __restrict__ dx, int dxs,
                              const b2h* __restrict__ mask, int ms, int n, int h, int w, int c, int k,
                              int acc) {
  // one thread per (pooled pixel, channel group): dy read once, the k x k outputs written from it;
  // 32-bit index math (the launcher checks the pooled element count fits)
  const int cg = c / G;
  const int wo = w / k, ho = h / k;
  const int total = n * ho * wo * cg;
  const float inv = 1.f / (k * k);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int ch = (i % cg) * G;
    const int q = i / cg;  // (img * ho + yo) * wo + xo
    const int xo = q % wo, r = q / wo;
    const int yo = r % ho, img = r / ho;
    float v[G];
    ldv<G>(dy + static_cast<long long>(q) * dys + ch, v);
#pragma unroll
    for (int e = 0; e < G; ++e) v[e] *= inv;
    const long long p0 = (static_cast<long long>(img) * h + yo * k) * w + xo * k;
    if constexpr (G == 8) {
      if (k == 4 && mask && !acc) {  // the stem pool: all 16 mask loads in flight before any store
        uint4 mr[16];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b)
            mr[4 * a + b] = __ldg(reinterpret_cast<const uint4*>(mask + (p0 + a * w + b) * ms + ch));
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const uint32_t mw[4] = {mr[4 * a + b].x, mr[4 * a + b].y, mr[4 * a + b].z, mr[4 * a + b].w};
            float o[8];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              o[2 * e] = h_lo(mw[e]) > 0.f ? v[2 * e] : 0.f;
              o[2 * e + 1] = h_hi(mw[e]) > 0.f ? v[2 * e + 1] : 0.f;
            }
            stv<8>(dx + (p0 + a * w + b) * dxs + ch, o);
          }
        continue;
      }
    }
    if (k == 2) {   // 2x2 pool (the Tiramisu transitions): the mask / accumulated loads of the four
                    // outputs in flight before any store, same per-output arithmetic as finish()
      const long long pp[4] = {p0, p0 + 1, p0 + w, p0 + w + 1};
      float mv[4][G], ov[4][G];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (mask) ldv<G>(mask + pp[u] * ms + ch, mv[u]);
        if (acc) ldv_rw<G>(dx + pp[u] * dxs + ch, ov[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float o[G];
#pragma unroll
        for (int e = 0; e < G; ++e) {
          o[e] = v[e];
          if (mask && !(mv[u][e] > 0.f)) o[e] = 0.f;
          if (acc) o[e] += ov[u][e];
        }
        stv<G>(dx + pp[u] * dxs + ch, o);
      }
      continue;
    }
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) {
        const long long p = p0 + static_cast<long long>(a) * w + b;
        float o[G];
#pragma unroll
        for (int e = 0; e < G; ++e) o[e] = v[e];
        finish<G>(o, mask ? mask + p * ms + ch : nullptr, dx + p * dxs + ch, acc);
      }
  }
}
template <int G>
__global__ void k_upsample_fwd(const b2h* __restrict__ x, int xs, b2h* __restrict__ y, int ys,
                               int n, int h, int w, int c, int f) {
  // one thread per (input pixel, channel group): read once, write the f x f replicas
  const int W = w * f;
  const int cg = c / G;
  const long long total = static_cast<long long>(n) * h * w * cg;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i % cg) * G;
    const long long sp = i / cg;  // (img * h + yy) * w + xx
    const int xx = static_cast<int>(sp % w);
    const long long r = sp / w;   // img * h + yy
    float v[G];
    ldv<G>(x + sp * xs + ch, v);
    const long long o = r * f * W + static_cast<long long>(xx) * f;  // output pixel (img, yy*f, xx*f)
    for (int a = 0; a < f; ++a)
      for (int b = 0; b < f; ++b) stv<G>(y + (o + static_cast<long long>(a) * W + b) * ys + ch, v);
  }
}
// dx[q] (+)= mask(x)[q] * sum over the f x f block of dy
template <int G>
__global__ void k_upsample_bwd(const b2h* __restrict__ dy, int dys, b2h* __restrict__ dx, int dxs,
                               const b2h* __restrict__ mask, int ms, int n, int h, int w, int c, int f,
                               int acc) {
  const int W = w * f;
  const int cg = c / G;
  const long long total = static_cast<long long>(n) * h * w * cg;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i % cg) * G;
    const long long q = i / cg;
    const int xx = static_cast<int>(q % w);
    const long long r = q / w;
    const int yy = static_cast<int>(r % h);
    const long long img = r / h;
    float s[G] = {};
    if (f == 2) {   // the four dy loads in flight at once, summed in the same order
      const long long r0 = (img * h * f + yy * f) * W + xx * f, r1 = r0 + W;
      float v[4][G];
      ldv<G>(dy + r0 * dys + ch, v[0]);
      ldv<G>(dy + (r0 + 1) * dys + ch, v[1]);
      ldv<G>(dy + r1 * dys + ch, v[2]);
      ldv<G>(dy + (r1 + 1) * dys + ch, v[3]);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int e = 0; e < G; ++e) s[e] += v[u][e];
    } else {
      for (int a = 0; a < f; ++a) {
        const long long rowp = (img * h * f + yy * f + a) * W + xx * f;
        for (int b = 0; b < f; ++b) {
          float v[G];
          ldv<G>(dy + (rowp + b) * dys + ch, v);
#pragma unroll
          for (int e = 0; e < G; ++e) s[e] += v[e];
        }
      }
    }
    finish<G>(s, mask ? mask + q * ms + ch : nullptr, dx + q * dxs + ch, acc);
  }
}

// ------------------------------------------------------------------ add / mask
template <int G>
__global__ void k_add(const b2h* __restrict__ x, int xs, b2h* __restrict__ y, int ys,
                      const b2h* __restrict__ mask, int ms, long long npix, int c, int acc) {
  const int cg = c / G;
  const long long total = npix * cg;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i % cg) * G;
    const long long p = i / cg;
    float v[G];
    ldv_rw<G>(x + p * xs + ch, v);
    finish<G>(v, mask ? mask + p * ms + ch : nullptr, y + p * ys + ch, acc);
  }
}
template <int G>
__global__ void k_relu_mask(b2h* __restrict__ g, int gs, const b2h* __restrict__ a, int as,
                            long long npix, int c) {
  const int cg = c / G;
  const long long total = npix * cg;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i % cg) * G;
    const long long p = i / cg;
    float v[G];
    ldv_rw<G>(g + p * gs + ch, v);
    finish<G>(v, a + p * as + ch, g + p * gs + ch, 0);
  }
}

// ------------------------------------------------------------------ bias gradient
// pass 1: block b sums a contiguous pixel range; threads own channel groups and
//         stride over rows, rows are folded in shared memory -> part[b][c]
// pass 2: out[c] (+)= sum_b part[b][c] in a fixed order (deterministic)
template <int G>
__global__ void k_colsum_partial(const b2h* __restrict__ g, int gs, long long npix, int c,
                                 float* __restrict__ part) {
  extern __shared__ float red[];
  const int cg = c / G;
  const int lanes = cg < static_cast<int>(blockDim.x) ? cg : static_cast<int>(blockDim.x);
  const int rows = blockDim.x / lanes;
  const int row = threadIdx.x / lanes, lane = threadIdx.x - row * lanes;
  const long long per = (npix + gridDim.x - 1) / gridDim.x;
  const long long p0 = blockIdx.x * per;
  const long long p1 = p0 + per < npix ? p0 + per : npix;
  if (row < rows) {
    for (int grp = lane; grp < cg; grp += lanes) {
      float s[G] = {};
      for (long long p = p0 + row; p < p1; p += rows) {
        float v[G];
        ldv<G>(g + p * gs + grp * G, v);
#pragma unroll
        for (int e = 0; e < G; ++e) s[e] += v[e];
      }
#pragma unroll
      for (int e = 0; e < G; ++e) red[row * c + grp * G + e] = s[e];
    }
  }
  __syncthreads();
  for (int ch = threadIdx.x; ch < c; ch += blockDim.x) {
    float s = 0.f;
    for (int r = 0; r < rows; ++r) s += red[r * c + ch];
    part[static_cast<long long>(blockIdx.x) * c + ch] = s;
  }
}
__global__ void k_colsum_final(const float* __restrict__ part, int nb, int c, float* __restrict__ out, int acc) {
  __shared__ float red[8][33];
  const int ch = blockIdx.x * 32 + threadIdx.x;
  float s = 0.f;
  if (ch < c)
    for (int b = threadIdx.y; b < nb; b += 8) s += part[static_cast<long long>(b) * c + ch];
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && ch < c) {
    float t = 0.f;
    for (int y = 0; y < 8; ++y) t += red[y][threadIdx.x];
    out[ch] = acc ? out[ch] + t : t;
  }
}

static int colsum_blocks(long long npix) {
  return static_cast<int>(std::max<long long>(1, std::min<long long>((npix + 31) / 32, 2LL * num_sms())));
}


// dx[p][ci] (+)= mask * sum_k dy[p][k] * w[ci][k]   (1x1 conv, k = dy channels <= 8)
// weights transposed into shared memory as [k][cin] so a thread's 8 channels are 2 float4 reads
template <int G>
__global__ void k_dgrad_1x1_small(const b2h* __restrict__ dy, int dys, int kc,
                                  const float* __restrict__ w, int cin, b2h* __restrict__ dx, int dxs,
                                  const b2h* __restrict__ mask, int ms, long long npix, int acc) {
  extern __shared__ float wsm[];  // [kc][cin]
  for (int i = threadIdx.x; i < cin * kc; i += blockDim.x) {
    const int ci = i / kc, k = i - ci * kc;
    wsm[k * cin + ci] = w[i];
  }
  __syncthreads();
  const int cg = cin / G;
  const long long total = npix * cg;
  const bool dy_vec = (dys % 8) == 0 && ((reinterpret_cast<uintptr_t>(dy) & 15) == 0);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i % cg) * G;
    const long long p = i / cg;
    float d[8];
    if (dy_vec) {
      ldv<8>(dy + p * dys, d);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) d[k] = k < kc ? ld_bf(dy + p * dys + k) : 0.f;
    }
    float v[G];
#pragma unroll
    for (int e = 0; e < G; ++e) v[e] = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k >= kc) break;
      const float* wr = wsm + k * cin + ch;
      if constexpr (G == 8) {
        const float4 a = *reinterpret_cast<const float4*>(wr);
        const float4 b = *reinterpret_cast<const float4*>(wr + 4);
        v[0] += d[k] * a.x;
        v[1] += d[k] * a.y;
        v[2] += d[k] * a.z;
        v[3] += d[k] * a.w;
        v[4] += d[k] * b.x;
        v[5] += d[k] * b.y;
        v[6] += d[k] * b.z;
        v[7] += d[k] * b.w;
      } else {
        v[0] += d[k] * wr[0];
      }
    }
    finish<G>(v, mask ? mask + p * ms + ch : nullptr, dx + p * dxs + ch, acc);
  }
}

// Backward of a 1x1 conv with few output channels (the 3-class head), one pass over its input:
//   dW[ci][k] partial  = sum_p x[p][ci] * dy[p][k]      (per-block partials, fixed order)
//   db[k]     partial  = sum_p dy[p][k]
//   dx[p][ci] (+)= [x > 0] * sum_k w[ci][k] * dy[p][k]  (optional; x doubles as the relu mask)
// A warp-sized group of threads covers one pixel's channels (8 per thread, 16-byte accesses).
constexpr int HEAD_THREADS = 256;
template <int KC, bool DYV>
__global__ void __launch_bounds__(HEAD_THREADS, 2) k_head_backward(
    const b2h* __restrict__ dy, int dys, const float* __restrict__ w, int cin,
    const b2h* __restrict__ x, int xs, b2h* __restrict__ dx, int dxs, int acc, int mask_dx,
    int npix, float* __restrict__ dwp, float* __restrict__ dbp) {
  constexpr int kc = KC;
  extern __shared__ float hsm[];  // w^T [kc][cin], then reduction scratch [ppb][cin * kc + kc]
  float* wsm = hsm;
  float* red = hsm + kc * cin;
  for (int i = threadIdx.x; i < cin * kc; i += blockDim.x) {
    const int ci = i / kc, k = i - ci * kc;
    wsm[k * cin + ci] = w[i];
  }
  __syncthreads();
  const int cg = cin / 8;
  const int g = threadIdx.x % cg, pl = threadIdx.x / cg, ppb = blockDim.x / cg;
  const int ch = g * 8;
  float aw[8][KC];
  float ab[KC];
#pragma unroll
  for (int k = 0; k < KC; ++k) ab[k] = 0.f;
#pragma unroll
  for (int e = 0; e < 8; ++e)
#pragma unroll
    for (int k = 0; k < KC; ++k) aw[e][k] = 0.f;
  // U pixels per iteration: all their loads are issued before any use (memory-level parallelism)
  constexpr int U = 8;
  const int stride = gridDim.x * ppb;
  for (int p0 = blockIdx.x * ppb + pl; p0 < npix; p0 += U * stride) {
    uint4 xr[U];
    float d[U][KC];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int p = p0 + u * stride;
      xr[u] = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int k = 0; k < KC; ++k) d[u][k] = 0.f;
      if (p < npix) {
        const long long pp = p;
        xr[u] = __ldg(reinterpret_cast<const uint4*>(x + pp * xs + ch));
        if constexpr (DYV) {
          const uint4 r = __ldg(reinterpret_cast<const uint4*>(dy + pp * dys));
          const uint32_t q[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
          for (int k = 0; k < KC; ++k) d[u][k] = (k & 1) ? bf16_hi(q[k >> 1]) : bf16_lo(q[k >> 1]);
        } else {
#pragma unroll
          for (int k = 0; k < KC; ++k) d[u][k] = ld_bf(dy + pp * dys + k);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int p = p0 + u * stride;
      if (p >= npix) break;
      const uint32_t q[4] = {xr[u].x, xr[u].y, xr[u].z, xr[u].w};
      float xv[8];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        xv[2 * e] = bf16_lo(q[e]);
        xv[2 * e + 1] = bf16_hi(q[e]);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e)
#pragma unroll
        for (int k = 0; k < KC; ++k) aw[e][k] += xv[e] * d[u][k];
      if (g == 0) {
#pragma unroll
        for (int k = 0; k < KC; ++k) ab[k] += d[u][k];
      }
      if (dx) {
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = 0.f;
#pragma unroll
        for (int k = 0; k < KC; ++k) {
          const float4 a = *reinterpret_cast<const float4*>(wsm + k * cin + ch);
          const float4 b = *reinterpret_cast<const float4*>(wsm + k * cin + ch + 4);
          v[0] += d[u][k] * a.x;
          v[1] += d[u][k] * a.y;
          v[2] += d[u][k] * a.z;
          v[3] += d[u][k] * a.w;
          v[4] += d[u][k] * b.x;
          v[5] += d[u][k] * b.y;
          v[6] += d[u][k] * b.z;
          v[7] += d[u][k] * b.w;
        }
        if (mask_dx) {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (!(xv[e] > 0.f)) v[e] = 0.f;
        }
        b2h* o = dx + static_cast<long long>(p) * dxs + ch;
        if (acc) {
          float old[8];
          ldv_rw<8>(o, old);
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] += old[e];
        }
        stv<8>(o, v);
      }
    }
  }
  // block partials: the ppb threads of each channel group meet in shared memory (fixed order)
  const int row = cin * kc + kc;
#pragma unroll
  for (int e = 0; e < 8; ++e)
#pragma unroll
    for (int k = 0; k < KC; ++k) red[pl * row + (ch + e) * kc + k] = aw[e][k];
  if (g == 0) {
#pragma unroll
    for (int k = 0; k < KC; ++k) red[pl * row + cin * kc + k] = ab[k];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < row; i += blockDim.x) {
    float sum = 0.f;
    for (int q = 0; q < ppb; ++q) sum += red[q * row + i];
    if (i < cin * kc)
      dwp[static_cast<long long>(blockIdx.x) * cin * kc + i] = sum;
    else
      dbp[static_cast<long long>(blockIdx.x) * kc + (i - cin * kc)] = sum;
  }
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
static bool vec_ok(const b2dl_act& a) { return a.c % 8 == 0 && a.c_stride % 8 == 0 && aligned16(a.ptr); }
static bool vec_ok(const b2dl_act& a, const b2dl_act& b) { return vec_ok(a) && vec_ok(b); }
static bool vec_ok(const b2dl_act& a, const b2dl_act& b, const b2dl_act& m) {
  return vec_ok(a, b) && (!m.ptr || (m.c_stride % 8 == 0 && aligned16(m.ptr)));
}

// ------------------------------------------------------------------ weight packing
// master HWIO fp32 [taps][cin][cout] -> fprop [cout][taps][cin_pad] and dgrad [cin][taps'][cout_pad]
__global__ void k_pack_fprop(const float* __restrict__ w, b2h* __restrict__ out, int taps, int cin,
                             int cout, int cin_pad) {
  const long long total = static_cast<long long>(cout) * taps * cin_pad;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int ci = static_cast<int>(i % cin_pad);
    long long r = i / cin_pad;
    int t = static_cast<int>(r % taps);
    int co = static_cast<int>(r / taps);
    out[i] = f_to_h(ci < cin ? w[(static_cast<long long>(t) * cin + ci) * cout + co] : 0.f);
  }
}
__global__ void k_pack_dgrad(const float* __restrict__ w, b2h* __restrict__ out, int taps, int cin,
                             int cout, int cout_pad) {
  const long long total = static_cast<long long>(cin) * taps * cout_pad;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int co = static_cast<int>(i % cout_pad);
    long long r = i / cout_pad;
    int tf = static_cast<int>(r % taps);
    int ci = static_cast<int>(r / taps);
    int t = taps - 1 - tf;
    out[i] = f_to_h(co < cout ? w[(static_cast<long long>(t) * cin + ci) * cout + co] : 0.f);
  }
}

}  // namespace b2

using namespace b2;
#define BF(p) reinterpret_cast<b2h*>(p)
#define CBF(p) reinterpret_cast<const b2h*>(p)

extern "C" int b2dl_nchw_to_nhwc(const float* x, b2dl_act y, int dst_f32, void* stream) {
  if (!x || !y.ptr) return B2DL_E_VALUE;
  long long total = static_cast<long long>(y.n) * y.c * y.h * y.w;
  k_nchw_to_nhwc<<<grid1d(total), 256, 0, as_stream(stream)>>>(x, y.ptr, dst_f32, y.n, y.c, y.h, y.w, y.c_stride);
  return check_launch();
}

extern "C" int b2dl_nchw_to_nhwc_halo(const float* x, int n, int c, int h, int w, void* y, int wp, int left,
                                      void* stream) {
  if (!x || !y || n < 1 || h < 1 || w < 1 || left < 0 || wp < w + left) return B2DL_E_VALUE;
  if (c < 8 || c > 64 || c % 8 || (reinterpret_cast<uintptr_t>(y) & 15)) return B2DL_E_ALIGN;
  dim3 grid(cdiv(w, HALO_COLS), h, n);
  k_nchw_to_nhwc_halo<<<grid, HALO_COLS, 0, as_stream(stream)>>>(x, BF(y), c, h, w, wp, left);
  return check_launch();
}

extern "C" int b2dl_nhwc_to_nchw(b2dl_act x, int src_f32, float* y, void* stream) {
  if (!y || !x.ptr) return B2DL_E_VALUE;
  long long total = static_cast<long long>(x.n) * x.c * x.h * x.w;
  k_nhwc_to_nchw<<<grid1d(total), 256, 0, as_stream(stream)>>>(x.ptr, src_f32, y, x.n, x.c, x.h, x.w, x.c_stride);
  return check_launch();
}

#define B2_LAUNCH_G(KERN, VEC, GRIDN, ...)                                                   \
  do {                                                                                      \
    if (VEC)                                                                                \
      KERN<8><<<grid1d(GRIDN, 8), 256, 0, as_stream(stream)>>>(__VA_ARGS__);                \
    else                                                                                    \
      KERN<1><<<grid1d(GRIDN), 256, 0, as_stream(stream)>>>(__VA_ARGS__);                   \
  } while (0)

extern "C" int b2dl_avgpool_fwd(b2dl_act x, b2dl_act y, int k, void* stream) {
  if (k < 1 || x.h % k || x.w % k || y.h != x.h / k || y.w != x.w / k || y.c != x.c || y.n != x.n) return B2DL_E_VALUE;
  long long total = static_cast<long long>(y.n) * y.h * y.w * y.c;
  B2_LAUNCH_G(k_avgpool_fwd, vec_ok(x, y), total, CBF(x.ptr), x.c_stride, BF(y.ptr), y.c_stride, y.n, y.h, y.w, y.c, k);
  return check_launch();
}

extern "C" int b2dl_avgpool_bwd(b2dl_act dy, b2dl_act dx, int k, int accumulate, b2dl_act mask, void* stream) {
  if (k < 1 || dx.h != dy.h * k || dx.w != dy.w * k || dx.c != dy.c) return B2DL_E_VALUE;
  long long total = static_cast<long long>(dx.n) * dx.h * dx.w * dx.c;
  if (static_cast<long long>(dy.n) * dy.h * dy.w * dy.c > 0x7fffffffLL) return B2DL_E_VALUE;
  total /= static_cast<long long>(k) * k;   // threads walk pooled pixels
  B2_LAUNCH_G(k_avgpool_bwd, vec_ok(dy, dx, mask), total, CBF(dy.ptr), dy.c_stride, BF(dx.ptr), dx.c_stride,
              CBF(mask.ptr), mask.c_stride, dx.n, dx.h, dx.w, dx.c, k, accumulate);
  return check_launch();
}

extern "C" int b2dl_upsample_fwd(b2dl_act x, b2dl_act y, int f, void* stream) {
  if (f < 1 || y.h != x.h * f || y.w != x.w * f || y.c != x.c) return B2DL_E_VALUE;
  long long total = static_cast<long long>(x.n) * x.h * x.w * x.c;
  B2_LAUNCH_G(k_upsample_fwd, vec_ok(x, y), total, CBF(x.ptr), x.c_stride, BF(y.ptr), y.c_stride, x.n, x.h, x.w, x.c,
              f);
  return check_launch();
}

extern "C" int b2dl_upsample_bwd(b2dl_act dy, b2dl_act dx, int f, int accumulate, b2dl_act mask, void* stream) {
  if (f < 1 || dy.h != dx.h * f || dy.w != dx.w * f || dy.c != dx.c) return B2DL_E_VALUE;
  long long total = static_cast<long long>(dx.n) * dx.h * dx.w * dx.c;
  B2_LAUNCH_G(k_upsample_bwd, vec_ok(dy, dx, mask), total, CBF(dy.ptr), dy.c_stride, BF(dx.ptr), dx.c_stride,
              CBF(mask.ptr), mask.c_stride, dx.n, dx.h, dx.w, dx.c, f, accumulate);
  return check_launch();
}

extern "C" int b2dl_add(b2dl_act x, b2dl_act y, int accumulate, b2dl_act mask, void* stream) {
  if (x.c != y.c || x.h != y.h || x.w != y.w || x.n != y.n) return B2DL_E_VALUE;
  long long npix = static_cast<long long>(x.n) * x.h * x.w;
  B2_LAUNCH_G(k_add, vec_ok(x, y, mask), npix * x.c, CBF(x.ptr), x.c_stride, BF(y.ptr), y.c_stride, CBF(mask.ptr),
              mask.c_stride, npix, x.c, accumulate);
  return check_launch();
}

extern "C" int b2dl_relu_mask(b2dl_act g, b2dl_act act, void* stream) {
  if (g.c != act.c || g.h != act.h || g.w != act.w || g.n != act.n) return B2DL_E_VALUE;
  long long npix = static_cast<long long>(g.n) * g.h * g.w;
  B2_LAUNCH_G(k_relu_mask, vec_ok(g, act), npix * g.c, BF(g.ptr), g.c_stride, CBF(act.ptr), act.c_stride, npix, g.c);
  return check_launch();
}

static int colsum_rows(int c, bool vec) {
  const int cg = vec ? c / 8 : c;
  const int lanes = cg < 256 ? cg : 256;
  return 256 / lanes;
}

extern "C" size_t b2dl_bias_grad_workspace_size(b2dl_act g) {
  long long npix = static_cast<long long>(g.n) * g.h * g.w;
  return static_cast<size_t>(colsum_blocks(npix)) * g.c * sizeof(float) + 256;
}

extern "C" int b2dl_bias_grad(b2dl_act g, float* out, int accumulate, void* workspace, size_t workspace_bytes,
                              void* stream) {
  long long npix = static_cast<long long>(g.n) * g.h * g.w;
  if (!out || workspace_bytes < b2dl_bias_grad_workspace_size(g)) return B2DL_E_VALUE;
  const int nb = colsum_blocks(npix);
  float* part = reinterpret_cast<float*>(workspace);
  const bool vec = vec_ok(g);
  const size_t smem = static_cast<size_t>(colsum_rows(g.c, vec)) * g.c * sizeof(float);
  if (smem > 48 * 1024) return B2DL_E_VALUE;
  if (vec)
    k_colsum_partial<8><<<nb, 256, smem, as_stream(stream)>>>(CBF(g.ptr), g.c_stride, npix, g.c, part);
  else
    k_colsum_partial<1><<<nb, 256, smem, as_stream(stream)>>>(CBF(g.ptr), g.c_stride, npix, g.c, part);
  int rc = check_launch();
  if (rc) return rc;
  k_colsum_final<<<(g.c + 31) / 32, dim3(32, 8), 0, as_stream(stream)>>>(part, nb, g.c, out, accumulate);
  return check_launch();
}

extern "C" int b2dl_pack_weights(const float* w_hwio, int kh, int kw, int cin, int cout, void* fprop_packed,
                                 void* dgrad_packed, void* stream) {
  const int taps = kh * kw;
  cudaStream_t st = as_stream(stream);
  if (fprop_packed) {
    const int cp = b2dl_cin_pad(cin);
    k_pack_fprop<<<grid1d(static_cast<long long>(cout) * taps * cp), 256, 0, st>>>(w_hwio, BF(fprop_packed), taps,
                                                                                  cin, cout, cp);
    int rc = check_launch();
    if (rc) return rc;
  }
  if (dgrad_packed) {
    const int cp = b2dl_cin_pad(cout);
    k_pack_dgrad<<<grid1d(static_cast<long long>(cin) * taps * cp), 256, 0, st>>>(w_hwio, BF(dgrad_packed), taps, cin,
                                                                                 cout, cp);
    return check_launch();
  }
  return B2DL_OK;
}

// W'[ci][i*K'+j][co] = sum over taps (ti, tj) of W_hwio[ti*k+tj][ci][co] whose block offset
// b = i + t - (k - 1) lies in [0, f) on both axes (K' = k + f - 1): the input gradient of a k x k
// "same" conv over a nearest x f upsampling, summed over each f x f block, as one K'-tap conv
// with input stride f over dy.
__global__ void k_pack_upsampled_dgrad(const float* __restrict__ w, b2h* __restrict__ out, int k, int cin,
                                       int cout, int f, int cp) {
  const int kk = k + f - 1;
  const long long total = static_cast<long long>(cin) * kk * kk * cp;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int co = static_cast<int>(idx % cp);
    const long long r = idx / cp;
    const int o = static_cast<int>(r % (kk * kk));
    const int ci = static_cast<int>(r / (kk * kk));
    const int i = o / kk, j = o - i * kk;
    float v = 0.f;
    if (co < cout)
      for (int ti = 0; ti < k; ++ti) {
        const int bi = i + ti - (k - 1);
        if (bi < 0 || bi >= f) continue;
        for (int tj = 0; tj < k; ++tj) {
          const int bj = j + tj - (k - 1);
          if (bj < 0 || bj >= f) continue;
          v += w[(static_cast<long long>(ti * k + tj) * cin + ci) * cout + co];
        }
      }
    out[idx] = f_to_h(v);
  }
}

extern "C" int b2dl_pack_upsampled_dgrad(const float* w_hwio, int k, int cin, int cout, int f, void* out,
                                         void* stream) {
  if (!w_hwio || !out || k < 1 || k % 2 == 0 || f < 1 || cin < 1 || cout < 1) return B2DL_E_VALUE;
  const int cp = b2dl_cin_pad(cout), kk = k + f - 1;
  k_pack_upsampled_dgrad<<<grid1d(static_cast<long long>(cin) * kk * kk * cp), 256, 0, as_stream(stream)>>>(
      w_hwio, BF(out), k, cin, cout, f, cp);
  return check_launch();
}

// Phase decomposition of a "same" k x k conv over a nearest x f upsampling: output row f*i + a
// reads upsampled row f*i + a + t - P (P = (k-1)/2), i.e. low-resolution row i + d(a, t) with
// d(a, t) = floor((a + t - P) / f).  Per phase a the offsets form the range [d(a,0), d(a,k-1)];
// merged weights sum the taps that land on the same offset.  Output: the phases (a, b) in
// row-major order, each a bf16 HWIO block [ka * kb][cin][cout] (ka = d(a,k-1) - d(a,0) + 1).
__device__ __host__ inline int up_floordiv(int v, int f) { return v >= 0 ? v / f : -((-v + f - 1) / f); }

struct UpTaps {
  uint32_t mask[256];   // per merged tap (phase blocks in order): bit ty*k+tx set if that tap is summed in
};

__global__ void k_pack_upsampled_fprop(const float* __restrict__ w, b2h* __restrict__ out, long long per,
                                       int taps, int kk, const UpTaps tab) {
  const long long total = static_cast<long long>(taps) * per;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long e = idx % per;
    const uint32_t m = tab.mask[idx / per];
    float v = 0.f;
    for (int t = 0; t < kk; ++t)
      if (m >> t & 1u) v += w[t * per + e];
    out[idx] = f_to_h(v);
  }
}

extern "C" int b2dl_upsampled_fprop_taps(int k, int f) {
  if (k < 1 || k % 2 == 0 || f < 1) return -1;
  const int P = (k - 1) / 2;
  int S = 0;
  for (int a = 0; a < f; ++a) S += up_floordiv(a + k - 1 - P, f) - up_floordiv(a - P, f) + 1;
  return S * S;
}

extern "C" int b2dl_pack_upsampled_fprop(const float* w_hwio, int k, int cin, int cout, int f, void* out,
                                         void* stream) {
  if (!w_hwio || !out || k < 1 || k % 2 == 0 || k > 5 || f < 2 || f > 8 || cin < 1 || cout < 1) return B2DL_E_VALUE;
  const int P = (k - 1) / 2;
  UpTaps tab{};
  int T = 0;
  for (int a = 0; a < f; ++a) {
    const int a0 = up_floordiv(a - P, f), ka = up_floordiv(a + k - 1 - P, f) - a0 + 1;
    for (int b = 0; b < f; ++b) {
      const int b0 = up_floordiv(b - P, f), kb = up_floordiv(b + k - 1 - P, f) - b0 + 1;
      for (int dy = 0; dy < ka; ++dy)
        for (int dx = 0; dx < kb; ++dx) {
          if (T >= 256) return B2DL_E_VALUE;
          uint32_t m = 0;
          for (int ty = 0; ty < k; ++ty)
            for (int tx = 0; tx < k; ++tx)
              if (up_floordiv(a + ty - P, f) - a0 == dy && up_floordiv(b + tx - P, f) - b0 == dx) m |= 1u << (ty * k + tx);
          tab.mask[T++] = m;
        }
    }
  }
  const long long per = static_cast<long long>(cin) * cout;
  k_pack_upsampled_fprop<<<grid1d(T * per), 256, 0, as_stream(stream)>>>(w_hwio, BF(out), per, T, k * k, tab);
  return check_launch();
}

// Weight gradient of a "same" K x K conv over a nearest x f upsampling, from the low-resolution
// input: dW[t] = sum_q x_up[q] dy[q + P - t] = sum_i x[i] G_t[i] with
//   G_t[i] = sum over the f x f block of low-resolution pixel i of dy shifted by P - t
// (zero outside the image).  One thread per (pixel i, 8 channels): the (f+K-1)^2 dy pixels
// around the block, K horizontal window sums per row, accumulated into the K*K outputs.
// G: [n][h][w][K*K][c] bf16, so dW = x^T G is one 1x1 wgrad with K*K*c output channels.
// The K*K shifted F x F block sums of a (F+K-1)^2 window of W words (2 bf16 channels each):
// horizontal window sums per row first, then vertical sums of those (each element converted once).
template <int K, int F, int W>
__device__ __forceinline__ void upw_block_sums(const uint32_t (&v)[F + K - 1][F + K - 1][W], float (&o)[K * K][2 * W]) {
  float rs[F + K - 1][K][2 * W];
#pragma unroll
  for (int rr = 0; rr < F + K - 1; ++rr) {
    float e[F + K - 1][2 * W];
#pragma unroll
    for (int cc = 0; cc < F + K - 1; ++cc)
#pragma unroll
      for (int u = 0; u < W; ++u) {
        e[cc][2 * u] = bf16_lo(v[rr][cc][u]);
        e[cc][2 * u + 1] = bf16_hi(v[rr][cc][u]);
      }
#pragma unroll
    for (int tx = 0; tx < K; ++tx)
#pragma unroll
      for (int ch = 0; ch < 2 * W; ++ch) {
        float a = 0.f;
#pragma unroll
        for (int q = 0; q < F; ++q) a += e[K - 1 - tx + q][ch];
        rs[rr][tx][ch] = a;
      }
  }
#pragma unroll
  for (int ty = 0; ty < K; ++ty)
#pragma unroll
    for (int tx = 0; tx < K; ++tx)
#pragma unroll
      for (int ch = 0; ch < 2 * W; ++ch) {
        float a = 0.f;
#pragma unroll
        for (int u = 0; u < F; ++u) a += rs[K - 1 - ty + u][tx][ch];
        o[ty * K + tx][ch] = a;
      }
}

// W words (2W channels) per thread: grid (w * c/(2W) / 256, h, n), one thread per (low-resolution
// pixel, 2W channels); a warp covers 64W channels of one pixel (128-byte lines per dy row segment
// for W = 1, 256 for W = 2).  32-bit index math and an unpredicated interior path: the kernel is
// instruction-bound, so wider words amortise the address arithmetic over more channels.
template <int K, int F, int W>
__global__ void __launch_bounds__(256) k_upsampled_wgrad_sums(const b2h* __restrict__ dy, int dys, int H,
                                                              int Wd, int c, b2h* __restrict__ g) {
  constexpr int P = (K - 1) / 2, R = F + K - 1, CPT = 2 * W;
  const int h = H / F, w = Wd / F, cv = c / CPT;
  const int t = blockIdx.x * 256 + threadIdx.x;
  if (t >= w * cv) return;
  const int j = t / cv, ch = (t - j * cv) * CPT;
  const int i = blockIdx.y, b = blockIdx.z;
  const int y0 = F * i - (K - 1 - P), x0 = F * j - (K - 1 - P);
  const b2h* img = dy + static_cast<size_t>(b) * H * Wd * dys + ch;
  uint32_t v[R][R][W];
  auto ld = [&](const b2h* ptr, uint32_t (&dst)[W]) {
    if constexpr (W == 2) {
      const uint2 u = __ldg(reinterpret_cast<const uint2*>(ptr));
      dst[0] = u.x;
      dst[1] = u.y;
    } else {
      dst[0] = __ldg(reinterpret_cast<const uint32_t*>(ptr));
    }
  };
  if (y0 >= 0 && y0 + R <= H && x0 >= 0 && x0 + R <= Wd) {
    const b2h* p0 = img + (static_cast<size_t>(y0) * Wd + x0) * dys;
#pragma unroll
    for (int rr = 0; rr < R; ++rr)
#pragma unroll
      for (int cc = 0; cc < R; ++cc) ld(p0 + (rr * Wd + cc) * dys, v[rr][cc]);
  } else {
#pragma unroll
    for (int rr = 0; rr < R; ++rr)
#pragma unroll
      for (int cc = 0; cc < R; ++cc) {
        const int y = y0 + rr, x = x0 + cc;
        if (y >= 0 && y < H && x >= 0 && x < Wd) {
          ld(img + (static_cast<size_t>(y) * Wd + x) * dys, v[rr][cc]);
        } else {
#pragma unroll
          for (int u = 0; u < W; ++u) v[rr][cc][u] = 0u;
        }
      }
  }
  b2h* out = g + ((static_cast<size_t>(b) * h + i) * w + j) * (K * K) * c + ch;
  // tap (ty, tx) sums rows / cols [K-1-ty, K-1-ty+F) of the loaded window
  float o[K * K][CPT];
  upw_block_sums<K, F, W>(v, o);
#pragma unroll
  for (int q = 0; q < K * K; ++q) {
    uint32_t wd[W];
#pragma unroll
    for (int u = 0; u < W; ++u) {
      const b2h2 hv = h2_from(o[q][2 * u], o[q][2 * u + 1]);
      wd[u] = *reinterpret_cast<const uint32_t*>(&hv);
    }
    if constexpr (W == 2)
      *reinterpret_cast<uint2*>(out + q * c) = make_uint2(wd[0], wd[1]);
    else
      *reinterpret_cast<uint32_t*>(out + q * c) = wd[0];
  }
}

// dW[t][ci][co] = sum_s ws[s][ci][t][co]; db[co] = sum_b bsum[b][center][co]   (fixed order)
__global__ void k_upsampled_wgrad_reduce(const float* __restrict__ ws, int wp, const float* __restrict__ bsum, int bp,
                                         int cin, int taps, int cout, int center, float* __restrict__ dw,
                                         float* __restrict__ db) {
  const int c4 = cout / 4;
  const long long nw = static_cast<long long>(taps) * cin * c4;
  const long long part = static_cast<long long>(cin) * taps * cout;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < nw + c4;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    if (idx < nw) {
      const int co = static_cast<int>(idx % c4) * 4;
      const long long r = idx / c4;
      const int ci = static_cast<int>(r % cin), t = static_cast<int>(r / cin);
      const float* src = ws + (static_cast<long long>(ci) * taps + t) * cout + co;
#pragma unroll 8
      for (int k = 0; k < wp; ++k) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(src + k * part));
        s.x += v.x;
        s.y += v.y;
        s.z += v.z;
        s.w += v.w;
      }
      *reinterpret_cast<float4*>(dw + (static_cast<long long>(t) * cin + ci) * cout + co) = s;
    } else if (db) {
      const int co = static_cast<int>(idx - nw) * 4;
      const float* src = bsum + static_cast<long long>(center) * cout + co;
#pragma unroll 8
      for (int k = 0; k < bp; ++k) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(src + static_cast<long long>(k) * taps * cout));
        s.x += v.x;
        s.y += v.y;
        s.z += v.z;
        s.w += v.w;
      }
      *reinterpret_cast<float4*>(db + co) = s;
    }
  }
}

extern "C" int b2dl_upsampled_wgrad_sums(b2dl_act dy, int k, int f, void* g, void* stream) {
  if (!dy.ptr || !g || f < 2 || f > 8 || dy.h % f || dy.w % f) return B2DL_E_VALUE;
  if (dy.c % 2 || dy.c_stride % 2 || reinterpret_cast<uintptr_t>(dy.ptr) & 3) return B2DL_E_ALIGN;
  if (dy.n > 65535 || dy.h / f > 65535 || static_cast<long long>(dy.w / f) * dy.c / 2 > 0x7fffffffLL)
    return B2DL_E_VALUE;
  // 4 channels per thread where 8-byte loads are aligned
  const bool w2 = dy.c % 4 == 0 && dy.c_stride % 4 == 0 && (reinterpret_cast<uintptr_t>(dy.ptr) & 7) == 0;
  const int cpt = w2 ? 4 : 2;
  const dim3 grid(cdiv(static_cast<long long>(dy.w / f) * (dy.c / cpt), 256), dy.h / f, dy.n);
#define B2_UPW(KV, FV)                                                                                     \
  if (k == KV && f == FV) {                                                                               \
    if (w2)                                                                                               \
      k_upsampled_wgrad_sums<KV, FV, 2><<<grid, 256, 0, as_stream(stream)>>>(CBF(dy.ptr), dy.c_stride, dy.h,  \
                                                                            dy.w, dy.c, BF(g));           \
    else                                                                                                  \
      k_upsampled_wgrad_sums<KV, FV, 1><<<grid, 256, 0, as_stream(stream)>>>(CBF(dy.ptr), dy.c_stride, dy.h,  \
                                                                            dy.w, dy.c, BF(g));           \
    return check_launch();                                                                                \
  }
  B2_UPW(3, 4)
  B2_UPW(3, 2)
  B2_UPW(1, 4)
  B2_UPW(1, 2)
#undef B2_UPW
  return B2DL_E_VALUE;
}

extern "C" int b2dl_upsampled_wgrad_reduce(const void* partials, int w_parts, int b_parts, size_t b_offset, int cin,
                                           int k, int cout, float* dw, float* db, void* stream) {
  if (!partials || !dw || cin < 1 || cout % 4 || k < 1 || k % 2 == 0 || w_parts < 1 ||
      (reinterpret_cast<uintptr_t>(partials) | reinterpret_cast<uintptr_t>(dw) | b_offset) & 15 ||
      (db && (reinterpret_cast<uintptr_t>(db) & 15)))
    return B2DL_E_VALUE;
  const int taps = k * k, center = (k / 2) * k + k / 2;
  const float* ws = static_cast<const float*>(partials);
  const float* bs = reinterpret_cast<const float*>(static_cast<const char*>(partials) + b_offset);
  k_upsampled_wgrad_reduce<<<grid1d(static_cast<long long>(taps) * cin * cout / 4 + cout / 4), 256, 0,
                             as_stream(stream)>>>(ws, w_parts, bs, b_parts, cin, taps, cout, center, dw, db);
  return check_launch();
}

extern "C" int b2dl_head_backward_parts(void) { return 4 * num_sms(); }

extern "C" int b2dl_head_backward(b2dl_act dy, const float* w_hwio, b2dl_act x, b2dl_act dx, int accumulate,
                                  int mask_dx, float* dw_partials, float* db_partials, void* stream) {
  if (!dy.ptr || !w_hwio || !x.ptr || !dw_partials || !db_partials || dy.c < 1 || dy.c > 8 || dy.n != x.n ||
      dy.h != x.h || dy.w != x.w)
    return B2DL_E_VALUE;
  if (dx.ptr && (dx.n != x.n || dx.h != x.h || dx.w != x.w || dx.c != x.c)) return B2DL_E_VALUE;
  const int cin = x.c;
  if (cin % 8 || HEAD_THREADS % (cin / 8) || !vec_ok(x) || (dx.ptr && !vec_ok(dx))) return B2DL_E_ALIGN;
  const long long npix = static_cast<long long>(x.n) * x.h * x.w;
  if (npix > 0x7fffffffLL) return B2DL_E_VALUE;
  const int ppb = HEAD_THREADS / (cin / 8);
  const size_t smem = (static_cast<size_t>(dy.c) * cin + static_cast<size_t>(ppb) * (cin * dy.c + dy.c)) * sizeof(float);
  if (smem > 48 * 1024) return B2DL_E_VALUE;
  const bool dyv = (dy.c_stride % 8) == 0 && aligned16(dy.ptr);
#define B2_HEAD(K)                                                                                             \
  case K:                                                                                                      \
    if (dyv)                                                                                                   \
      k_head_backward<K, true><<<b2dl_head_backward_parts(), HEAD_THREADS, smem, as_stream(stream)>>>(         \
          CBF(dy.ptr), dy.c_stride, w_hwio, cin, CBF(x.ptr), x.c_stride, BF(dx.ptr), dx.c_stride, accumulate,  \
          mask_dx, static_cast<int>(npix), dw_partials, db_partials);                                          \
    else                                                                                                       \
      k_head_backward<K, false><<<b2dl_head_backward_parts(), HEAD_THREADS, smem, as_stream(stream)>>>(        \
          CBF(dy.ptr), dy.c_stride, w_hwio, cin, CBF(x.ptr), x.c_stride, BF(dx.ptr), dx.c_stride, accumulate,  \
          mask_dx, static_cast<int>(npix), dw_partials, db_partials);                                          \
    break;
  switch (dy.c) {
    B2_HEAD(1)
    B2_HEAD(2)
    B2_HEAD(3)
    B2_HEAD(4)
    B2_HEAD(5)
    B2_HEAD(6)
    B2_HEAD(7)
    B2_HEAD(8)
  }
#undef B2_HEAD
  return check_launch();
}

extern "C" int b2dl_dgrad_1x1_small(b2dl_act dy, const float* w_hwio, b2dl_act dx, int accumulate, b2dl_act mask,
                                    void* stream) {
  if (!dy.ptr || !w_hwio || !dx.ptr || dy.c < 1 || dy.c > 8 || dy.n != dx.n || dy.h != dx.h || dy.w != dx.w)
    return B2DL_E_VALUE;
  const long long npix = static_cast<long long>(dx.n) * dx.h * dx.w;
  const size_t smem = static_cast<size_t>(dx.c) * dy.c * sizeof(float);
  if (smem > 48 * 1024) return B2DL_E_VALUE;
  if (vec_ok(dx, dx, mask))
    k_dgrad_1x1_small<8><<<grid1d(npix * dx.c, 8), 256, smem, as_stream(stream)>>>(
        CBF(dy.ptr), dy.c_stride, dy.c, w_hwio, dx.c, BF(dx.ptr), dx.c_stride, CBF(mask.ptr), mask.c_stride, npix,
        accumulate);
  else
    k_dgrad_1x1_small<1><<<grid1d(npix * dx.c), 256, smem, as_stream(stream)>>>(
        CBF(dy.ptr), dy.c_stride, dy.c, w_hwio, dx.c, BF(dx.ptr), dx.c_stride, CBF(mask.ptr), mask.c_stride, npix,
        accumulate);
  return check_launch();
}
