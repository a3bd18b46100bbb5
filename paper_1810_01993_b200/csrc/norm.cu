// Training-mode batch normalisation (+ residual + relu, fused into the normalising pass) and
// bilinear upsampling, NHWC, bf16 or fp32 storage -- the north-star items the reference lacks
// (float64 oracle in oracle/deskdl_port.py pinned by finite differences).
//
//   forward   stats: per-block partial sums of x and x^2 (fp64, fixed order) -> per-channel
//             mean / rstd / scale = gamma*rstd / shift = beta - mean*scale;
//             apply: y = relu?(x*scale + shift (+ residual))
//   backward  reduce: per-block partial sums of gy and gy*xhat (fp64, fixed order) ->
//             dbeta, dgamma and dx = gamma*rstd*(gy - dbeta/M - xhat*dgamma/M)
//   bilinear  half-pixel centres, source clamped at 0 (align_corners=False); the VJP gathers
//             each input pixel's contributions from the outputs whose taps reach it, so it is
//             deterministic (no atomics).
// All passes are HBM streams: 16-byte vectors over channels, pixels split across blocks.
#include <cuda_bf16.h>

#include <algorithm>

#include "internal.h"

namespace b2 {

// ---- element access: V consecutive channels of type T as floats
template <typename T, int V>
struct Vec;
template <>
struct Vec<b2h, 8> {
  static __device__ __forceinline__ void load(const b2h* p, float* v) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[2 * e] = h_lo(w[e]);
      v[2 * e + 1] = h_hi(w[e]);
    }
  }
  static __device__ __forceinline__ void store(b2h* p, const float* v) {
    uint4 u;
    uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const b2h2 h = h2_from(v[2 * e], v[2 * e + 1]);
      w[e] = *reinterpret_cast<const uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(p) = u;
  }
};
template <>
struct Vec<float, 4> {
  static __device__ __forceinline__ void load(const float* p, float* v) {
    const float4 u = *reinterpret_cast<const float4*>(p);
    v[0] = u.x;
    v[1] = u.y;
    v[2] = u.z;
    v[3] = u.w;
  }
  static __device__ __forceinline__ void store(float* p, const float* v) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <typename T>
struct Vec<T, 1> {
  static __device__ __forceinline__ void load(const T* p, float* v) { v[0] = static_cast<float>(*p); }
  static __device__ __forceinline__ void store(T* p, const float* v) { *p = static_cast<T>(v[0]); }
};
template <>
struct Vec<b2h, 1> {
  static __device__ __forceinline__ void load(const b2h* p, float* v) { v[0] = h_to_f(*p); }
  static __device__ __forceinline__ void store(b2h* p, const float* v) { *p = f_to_h(v[0]); }
};

constexpr int BN_THREADS = 256;

// partial[b][0][c] = sum of a, partial[b][1][c] = sum of a*b' over block b's pixels, where for the
// forward a = x, b' = x; for the backward a = gy, b' = xhat = (x - mean) * rstd.
template <typename T, int V, bool BWD>
__global__ void __launch_bounds__(BN_THREADS) k_bn_reduce(const T* __restrict__ x, int xs, const T* __restrict__ gy,
                                                          int gs, const float* __restrict__ stats, long long npix,
                                                          int c, double* __restrict__ part) {
  extern __shared__ double red[];  // [rows][2][c]
  const int groups = c / V;
  const int lanes = groups < BN_THREADS ? groups : BN_THREADS;
  const int rows = BN_THREADS / lanes;
  const int row = threadIdx.x / lanes, lane = threadIdx.x - row * lanes;
  const long long per = (npix + gridDim.x - 1) / gridDim.x;
  const long long p0 = blockIdx.x * per, p1 = min(npix, p0 + per);
  for (int g = lane; g < groups; g += lanes) {
    double s[V], q[V];
#pragma unroll
    for (int e = 0; e < V; ++e) s[e] = q[e] = 0.0;
    float mean[V], rstd[V];
    if constexpr (BWD) {
#pragma unroll
      for (int e = 0; e < V; ++e) {
        mean[e] = stats[g * V + e];
        rstd[e] = stats[c + g * V + e];
      }
    }
    if (threadIdx.x < rows * lanes) {
      auto accum = [&](const float* xv, const float* gv) {
        if constexpr (BWD) {
#pragma unroll
          for (int e = 0; e < V; ++e) {
            s[e] += gv[e];
            q[e] += static_cast<double>(gv[e]) * ((xv[e] - mean[e]) * rstd[e]);
          }
        } else {
#pragma unroll
          for (int e = 0; e < V; ++e) {
            s[e] += xv[e];
            q[e] += static_cast<double>(xv[e]) * xv[e];
          }
        }
      };
      // U pixels' loads in flight per thread (one load in flight left the pass latency-bound)
      constexpr int U = BWD ? 4 : 8;   // two input streams backward, one forward
      long long p = p0 + row;
      for (; p + (U - 1) * rows < p1; p += U * rows) {
        float xv[U][V], gv[U][V];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          Vec<T, V>::load(x + (p + u * rows) * xs + g * V, xv[u]);
          if constexpr (BWD) Vec<T, V>::load(gy + (p + u * rows) * gs + g * V, gv[u]);
        }
        // the U pixels are summed in fp32 first (fixed order), then folded into the fp64 sums:
        // a quarter of the f32 -> f64 conversions and fp64 adds, which bound the pass
        float sf[V], qf[V];
#pragma unroll
        for (int e = 0; e < V; ++e) {
          if constexpr (BWD) {
            sf[e] = gv[0][e];
            qf[e] = gv[0][e] * ((xv[0][e] - mean[e]) * rstd[e]);
          } else {
            sf[e] = xv[0][e];
            qf[e] = xv[0][e] * xv[0][e];
          }
        }
#pragma unroll
        for (int u = 1; u < U; ++u)
#pragma unroll
          for (int e = 0; e < V; ++e) {
            if constexpr (BWD) {
              sf[e] += gv[u][e];
              qf[e] = fmaf(gv[u][e], (xv[u][e] - mean[e]) * rstd[e], qf[e]);
            } else {
              sf[e] += xv[u][e];
              qf[e] = fmaf(xv[u][e], xv[u][e], qf[e]);
            }
          }
#pragma unroll
        for (int e = 0; e < V; ++e) {
          s[e] += sf[e];
          q[e] += qf[e];
        }
      }
      for (; p < p1; p += rows) {
        float xv[V], gv[V];
        Vec<T, V>::load(x + p * xs + g * V, xv);
        if constexpr (BWD) Vec<T, V>::load(gy + p * gs + g * V, gv);
        accum(xv, gv);
      }
    }
    if (threadIdx.x < rows * lanes) {
#pragma unroll
      for (int e = 0; e < V; ++e) {
        red[(row * 2 + 0) * c + g * V + e] = s[e];
        red[(row * 2 + 1) * c + g * V + e] = q[e];
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * c; i += blockDim.x) {
    const int k = i / c, ch = i - k * c;
    double t = 0.0;
    for (int r = 0; r < rows; ++r) t += red[(r * 2 + k) * c + ch];
    part[(static_cast<long long>(blockIdx.x) * 2 + k) * c + ch] = t;
  }
}

// Sum of the per-block partials of channel ch in a fixed order: FIN_ROWS threads per channel
// each take every FIN_ROWS-th block, then a fixed-shape tree over the rows (deterministic).
constexpr int FIN_CH = 32, FIN_ROWS = 16;
template <typename P>
__device__ __forceinline__ void fin_sums(const P* __restrict__ part, int blocks, int c, double* red, double& s,
                                         double& q) {
  const int lc = threadIdx.x % FIN_CH, r = threadIdx.x / FIN_CH;
  const int ch = blockIdx.x * FIN_CH + lc;
  double a = 0.0, b = 0.0;
  if (ch < c)
    for (int k = r; k < blocks; k += FIN_ROWS) {
      a += part[(static_cast<long long>(k) * 2) * c + ch];
      b += part[(static_cast<long long>(k) * 2 + 1) * c + ch];
    }
  red[(r * 2) * FIN_CH + lc] = a;
  red[(r * 2 + 1) * FIN_CH + lc] = b;
  __syncthreads();
  s = q = 0.0;
  if (r == 0)
    for (int k = 0; k < FIN_ROWS; ++k) {
      s += red[(k * 2) * FIN_CH + lc];
      q += red[(k * 2 + 1) * FIN_CH + lc];
    }
}

// Fold conv-epilogue statistics partials [tiles][2][c] (fp32) into [G][2][c] fp64 rows: block
// (channel group, g) sums its contiguous tile range with FIN_ROWS strided threads per channel and
// a fixed-order fold -- deterministic, and wide enough for 10^4+ tiles.
__global__ void __launch_bounds__(FIN_CH * FIN_ROWS) k_bn_fold_partials(const float* __restrict__ part, int tiles,
                                                                        int c, double* __restrict__ fold) {
  __shared__ double red[FIN_ROWS * 2 * FIN_CH];
  const int lc = threadIdx.x % FIN_CH, r = threadIdx.x / FIN_CH;
  const int ch = blockIdx.x * FIN_CH + lc, g = blockIdx.y, G = gridDim.y;
  const long long per = (tiles + G - 1) / G;
  const long long lo = g * per, hi = min(static_cast<long long>(tiles), lo + per);
  double a = 0.0, b = 0.0;
  if (ch < c)
    for (long long k = lo + r; k < hi; k += FIN_ROWS) {
      a += part[(k * 2) * c + ch];
      b += part[(k * 2 + 1) * c + ch];
    }
  red[(r * 2) * FIN_CH + lc] = a;
  red[(r * 2 + 1) * FIN_CH + lc] = b;
  __syncthreads();
  if (r == 0 && ch < c) {
    double s = 0.0, q = 0.0;
    for (int k = 0; k < FIN_ROWS; ++k) {
      s += red[(k * 2) * FIN_CH + lc];
      q += red[(k * 2 + 1) * FIN_CH + lc];
    }
    fold[(static_cast<long long>(g) * 2) * c + ch] = s;
    fold[(static_cast<long long>(g) * 2 + 1) * c + ch] = q;
  }
}

// stats [4][c]: mean, rstd, scale = gamma*rstd, shift = beta - mean*scale
template <typename P>
__global__ void __launch_bounds__(FIN_CH * FIN_ROWS) k_bn_finalize(const P* __restrict__ part, int blocks, int c,
                                                                   double m, float eps, const float* __restrict__ gamma,
                                                                   const float* __restrict__ beta,
                                                                   float* __restrict__ stats) {
  __shared__ double red[FIN_ROWS * 2 * FIN_CH];
  double s, q;
  fin_sums(part, blocks, c, red, s, q);
  const int ch = blockIdx.x * FIN_CH + threadIdx.x;
  if (threadIdx.x >= FIN_CH || ch >= c) return;
  const double mean = s / m;
  const double var = fmax(q / m - mean * mean, 0.0);
  const double rstd = 1.0 / sqrt(var + static_cast<double>(eps));
  const double scale = static_cast<double>(gamma[ch]) * rstd;
  stats[ch] = static_cast<float>(mean);
  stats[c + ch] = static_cast<float>(rstd);
  stats[2 * c + ch] = static_cast<float>(scale);
  stats[3 * c + ch] = static_cast<float>(static_cast<double>(beta[ch]) - mean * scale);
}

// dbeta = sum gy, dgamma = sum gy*xhat.  dx = gamma*rstd*(gy - dbeta/M - xhat*dgamma/M) is
// folded to dx = A*gy + K1*x + K0 per channel: coef [3][c] = A, K1, K0.
template <typename P>
__global__ void __launch_bounds__(FIN_CH * FIN_ROWS) k_bn_bwd_finalize(
    const P* __restrict__ part, int blocks, int c, double m, const float* __restrict__ gamma,
    const float* __restrict__ stats, float* __restrict__ dgamma, float* __restrict__ dbeta, int acc,
    float* __restrict__ coef) {
  __shared__ double red[FIN_ROWS * 2 * FIN_CH];
  double s, q;
  fin_sums(part, blocks, c, red, s, q);
  const int ch = blockIdx.x * FIN_CH + threadIdx.x;
  if (threadIdx.x >= FIN_CH || ch >= c) return;
  if (dbeta) dbeta[ch] = static_cast<float>(acc ? dbeta[ch] + s : s);
  if (dgamma) dgamma[ch] = static_cast<float>(acc ? dgamma[ch] + q : q);
  const double mean = stats[ch], rstd = stats[c + ch];
  const double A = static_cast<double>(gamma[ch]) * rstd;
  const double k1 = -A * rstd * q / m;
  coef[ch] = static_cast<float>(A);
  coef[c + ch] = static_cast<float>(k1);
  coef[2 * c + ch] = static_cast<float>(-A * s / m - k1 * mean);
}

// Streams over (pixel, channel group): a thread keeps one channel group and walks pixels, so
// the per-channel coefficients live in registers.  y = relu?(x*scale + shift (+ res)).
template <typename T, int V>
__global__ void __launch_bounds__(BN_THREADS) k_bn_apply(const T* __restrict__ x, int xs,
                                                         const float* __restrict__ stats, const T* __restrict__ res,
                                                         int rs, int relu, T* __restrict__ y, int ys, long long npix,
                                                         int c) {
  const int groups = c / V;
  const int lanes = groups < BN_THREADS ? groups : BN_THREADS;
  const int rows = BN_THREADS / lanes;
  const int row = threadIdx.x / lanes, lane = threadIdx.x - row * lanes;
  if (row >= rows) return;
  for (int g = lane; g < groups; g += lanes) {
    float sc[V], sh[V];
#pragma unroll
    for (int e = 0; e < V; ++e) {
      sc[e] = stats[2 * c + g * V + e];
      sh[e] = stats[3 * c + g * V + e];
    }
    for (long long p = static_cast<long long>(blockIdx.x) * rows + row; p < npix;
         p += static_cast<long long>(gridDim.x) * rows) {
      float v[V];
      Vec<T, V>::load(x + p * xs + g * V, v);
#pragma unroll
      for (int e = 0; e < V; ++e) v[e] = fmaf(v[e], sc[e], sh[e]);
      if (res) {
        float r[V];
        Vec<T, V>::load(res + p * rs + g * V, r);
#pragma unroll
        for (int e = 0; e < V; ++e) v[e] += r[e];
      }
      if (relu) {
#pragma unroll
        for (int e = 0; e < V; ++e) v[e] = fmaxf(v[e], 0.f);
      }
      Vec<T, V>::store(y + p * ys + g * V, v);
    }
  }
}

// dx (+)= A*gy + K1*x + K0
template <typename T, int V>
__global__ void __launch_bounds__(BN_THREADS) k_bn_bwd_apply(const T* __restrict__ x, int xs, const T* __restrict__ gy,
                                                             int gs, const float* __restrict__ coef,
                                                             T* __restrict__ dx, int dxs, int acc, long long npix,
                                                             int c) {
  const int groups = c / V;
  const int lanes = groups < BN_THREADS ? groups : BN_THREADS;
  const int rows = BN_THREADS / lanes;
  const int row = threadIdx.x / lanes, lane = threadIdx.x - row * lanes;
  if (row >= rows) return;
  for (int g = lane; g < groups; g += lanes) {
    float ca[V], c1[V], c0[V];
#pragma unroll
    for (int e = 0; e < V; ++e) {
      ca[e] = coef[g * V + e];
      c1[e] = coef[c + g * V + e];
      c0[e] = coef[2 * c + g * V + e];
    }
    for (long long p = static_cast<long long>(blockIdx.x) * rows + row; p < npix;
         p += static_cast<long long>(gridDim.x) * rows) {
      float xv[V], gv[V], o[V];
      Vec<T, V>::load(x + p * xs + g * V, xv);
      Vec<T, V>::load(gy + p * gs + g * V, gv);
      if (acc) Vec<T, V>::load(dx + p * dxs + g * V, o);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const float d = fmaf(ca[e], gv[e], fmaf(c1[e], xv[e], c0[e]));
        o[e] = acc ? o[e] + d : d;
      }
      Vec<T, V>::store(dx + p * dxs + g * V, o);
    }
  }
}

// ---- bilinear (half-pixel centres, clamp at 0), integer factor f
__device__ __forceinline__ void bl_tap(int o, int n_in, int f, int& i0, int& i1, float& w0, float& w1) {
  // power-of-two factors: multiplying by 1/f is exact, i.e. bit-identical to the division
  float src = ((f & (f - 1)) == 0 ? (o + 0.5f) * __frcp_rn(static_cast<float>(f)) : (o + 0.5f) / f) - 0.5f;
  src = src < 0.f ? 0.f : src;
  i0 = static_cast<int>(src);  // floor (src >= 0)
  i1 = i0 + 1 < n_in ? i0 + 1 : n_in - 1;
  w1 = src - i0;
  w0 = 1.f - w1;
}

// one block per output row (row taps computed once), threads over (column, channel group)
template <typename T, int V>
__global__ void k_bilinear_fwd(const T* __restrict__ x, int xs, T* __restrict__ y, int ys, int n, int h, int w, int c,
                               int f) {
  const int H = h * f, W = w * f, groups = c / V;
  const int Y = blockIdx.x, img = blockIdx.y;
  int y0, y1, x0, x1;
  float wy0, wy1, wx0, wx1;
  bl_tap(Y, h, f, y0, y1, wy0, wy1);
  const T* r0 = x + (static_cast<long long>(img) * h + y0) * w * static_cast<long long>(xs);
  const T* r1 = x + (static_cast<long long>(img) * h + y1) * w * static_cast<long long>(xs);
  T* out = y + (static_cast<long long>(img) * H + Y) * W * static_cast<long long>(ys);
  // when the channel groups divide the block, a thread's group is fixed and its column steps by
  // blockDim / groups (no per-element integer division)
  const bool fixed_g = (blockDim.x % groups) == 0;
  const int g_fixed = threadIdx.x % groups, x_step = blockDim.x / groups;
  for (int i = threadIdx.x, Xs = threadIdx.x / groups; i < W * groups; i += blockDim.x, Xs += x_step) {
    const int X = fixed_g ? Xs : i / groups, g = fixed_g ? g_fixed : i - X * groups;
    bl_tap(X, w, f, x0, x1, wx0, wx1);
    float a[V], b[V], cc[V], d[V], o[V];
    Vec<T, V>::load(r0 + static_cast<long long>(x0) * xs + g * V, a);
    Vec<T, V>::load(r0 + static_cast<long long>(x1) * xs + g * V, b);
    Vec<T, V>::load(r1 + static_cast<long long>(x0) * xs + g * V, cc);
    Vec<T, V>::load(r1 + static_cast<long long>(x1) * xs + g * V, d);
#pragma unroll
    for (int e = 0; e < V; ++e) o[e] = wy0 * (wx0 * a[e] + wx1 * b[e]) + wy1 * (wx0 * cc[e] + wx1 * d[e]);
    Vec<T, V>::store(out + static_cast<long long>(X) * ys + g * V, o);
  }
}

// The VJP is separable: dx[y][x] = sum_Y wy(Y, y) * R[Y][x] with R[Y][x] = sum_X wx(X, x) * dy[Y][X].
// Pass 1 (one block per output row Y) forms R in fp32 at low-res columns, pass 2 (one block per
// input row y) sums the ~2f contributing rows of R -- each dy element is read once, no atomics.
__device__ __forceinline__ void bl_range(int i, int n_in, int f, int n_out, int& lo, int& hi) {
  // outputs whose floor tap is i - 1 or i: src = (o + 0.5) / f - 0.5 in [i - 1, i + 1); the last
  // input also takes the clamped outputs beyond it
  lo = max(0, static_cast<int>(ceilf(f * (i - 1) + 0.5f * f - 0.5f)));
  hi = i == n_in - 1 ? n_out - 1 : min(n_out - 1, static_cast<int>(ceilf(f * (i + 1) + 0.5f * f - 0.5f)) - 1);
}
__device__ __forceinline__ float bl_weight(int o, int i, int n_in, int f) {
  int i0, i1;
  float w0, w1;
  bl_tap(o, n_in, f, i0, i1, w0, w1);
  return (i0 == i ? w0 : 0.f) + (i1 == i ? w1 : 0.f);
}

template <typename T, int V>
__global__ void k_bilinear_bwd_rows(const T* __restrict__ dy, int dys, float* __restrict__ R, int h, int w, int c,
                                    int f) {
  const int H = h * f, W = w * f, groups = c / V;
  const int Y = blockIdx.x, img = blockIdx.y;
  const T* row = dy + (static_cast<long long>(img) * H + Y) * W * static_cast<long long>(dys);
  float* out = R + (static_cast<long long>(img) * H + Y) * w * static_cast<long long>(c);
  const bool fixed_g = (blockDim.x % groups) == 0;
  const int g_fixed = threadIdx.x % groups, x_step = blockDim.x / groups;
  for (int i = threadIdx.x, xs = threadIdx.x / groups; i < w * groups; i += blockDim.x, xs += x_step) {
    const int xx = fixed_g ? xs : i / groups, g = fixed_g ? g_fixed : i - xx * groups;
    int X0, X1;
    bl_range(xx, w, f, W, X0, X1);
    float s[V];
#pragma unroll
    for (int e = 0; e < V; ++e) s[e] = 0.f;
    for (int X = X0; X <= X1; ++X) {
      const float wx = bl_weight(X, xx, w, f);
      if (wx == 0.f) continue;
      float v[V];
      Vec<T, V>::load(row + static_cast<long long>(X) * dys + g * V, v);
#pragma unroll
      for (int e = 0; e < V; ++e) s[e] += wx * v[e];
    }
    float* o = out + static_cast<long long>(xx) * c + g * V;
    if constexpr (V % 4 == 0) {  // 16-byte stores (c % V == 0 and a 256-byte aligned workspace)
#pragma unroll
      for (int e = 0; e < V; e += 4) *reinterpret_cast<float4*>(o + e) = make_float4(s[e], s[e + 1], s[e + 2], s[e + 3]);
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) o[e] = s[e];
    }
  }
}

template <typename T, int V>
__global__ void k_bilinear_bwd_cols(const float* __restrict__ R, T* __restrict__ dx, int dxs,
                                    const T* __restrict__ mask, int ms, int h, int w, int c, int f, int acc) {
  const int H = h * f, groups = c / V;
  const int yy = blockIdx.x, img = blockIdx.y;
  int Y0, Y1;
  bl_range(yy, h, f, H, Y0, Y1);
  const long long q0 = (static_cast<long long>(img) * h + yy) * w;
  // the block's row weights, computed once (same values and order as per element)
  constexpr int BL_MAXY = 64;
  __shared__ float swy[BL_MAXY];
  const bool wy_cached = Y1 - Y0 + 1 <= BL_MAXY;
  if (wy_cached)
    for (int t = threadIdx.x; t <= Y1 - Y0; t += blockDim.x) swy[t] = bl_weight(Y0 + t, yy, h, f);
  __syncthreads();
  const bool fixed_g = (blockDim.x % groups) == 0;
  const int g_fixed = threadIdx.x % groups, x_step = blockDim.x / groups;
  for (int i = threadIdx.x, xs = threadIdx.x / groups; i < w * groups; i += blockDim.x, xs += x_step) {
    const int xx = fixed_g ? xs : i / groups, g = fixed_g ? g_fixed : i - xx * groups;
    float s[V];
#pragma unroll
    for (int e = 0; e < V; ++e) s[e] = 0.f;
    for (int Y = Y0; Y <= Y1; ++Y) {
      const float wy = wy_cached ? swy[Y - Y0] : bl_weight(Y, yy, h, f);
      if (wy == 0.f) continue;
      const float* r = R + ((static_cast<long long>(img) * H + Y) * w + xx) * c + g * V;
      if constexpr (V % 4 == 0) {
#pragma unroll
        for (int e = 0; e < V; e += 4) {
          const float4 r4 = *reinterpret_cast<const float4*>(r + e);
          s[e] += wy * r4.x;
          s[e + 1] += wy * r4.y;
          s[e + 2] += wy * r4.z;
          s[e + 3] += wy * r4.w;
        }
      } else {
#pragma unroll
        for (int e = 0; e < V; ++e) s[e] += wy * r[e];
      }
    }
    const long long q = q0 + xx;
    if (mask) {
      float m[V];
      Vec<T, V>::load(mask + q * ms + g * V, m);
#pragma unroll
      for (int e = 0; e < V; ++e)
        if (!(m[e] > 0.f)) s[e] = 0.f;
    }
    if (acc) {
      float o[V];
      Vec<T, V>::load(dx + q * dxs + g * V, o);
#pragma unroll
      for (int e = 0; e < V; ++e) s[e] += o[e];
    }
    Vec<T, V>::store(dx + q * dxs + g * V, s);
  }
}

static int bn_blocks() { return 2 * num_sms(); }
// blocks for the per-thread-channel-group streams: enough rows of pixels to fill the GPU
static int stream_blocks(long long npix, int groups) {
  const int lanes = groups < BN_THREADS ? groups : BN_THREADS;
  const long long rows = BN_THREADS / lanes;
  return static_cast<int>(std::max<long long>(1, std::min<long long>((npix + rows - 1) / rows, 8LL * num_sms())));
}
static int grid_of(long long total) {
  return static_cast<int>(std::max<long long>(1, std::min<long long>((total + 255) / 256, 16LL * num_sms())));
}
static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
static bool vec_act(const b2dl_act& a, int v) { return !a.ptr || (a.c % v == 0 && a.c_stride % v == 0 && al16(a.ptr)); }
static size_t bn_red_smem(int c, int v) {
  const int groups = c / v;
  const int lanes = groups < BN_THREADS ? groups : BN_THREADS;
  return static_cast<size_t>(BN_THREADS / lanes) * 2 * c * sizeof(double);
}

// dispatch on (fp32?, vector width)
#define B2_TV(F32, VEC, ...)                        \
  do {                                              \
    if (F32) {                                      \
      if (VEC) {                                    \
        using T = float;                            \
        constexpr int V = 4;                        \
        __VA_ARGS__;                                \
      } else {                                      \
        using T = float;                            \
        constexpr int V = 1;                        \
        __VA_ARGS__;                                \
      }                                             \
    } else {                                        \
      if (VEC) {                                    \
        using T = b2h;                    \
        constexpr int V = 8;                        \
        __VA_ARGS__;                                \
      } else {                                      \
        using T = b2h;                    \
        constexpr int V = 1;                        \
        __VA_ARGS__;                                \
      }                                             \
    }                                               \
  } while (0)

}  // namespace b2

using namespace b2;

extern "C" size_t b2dl_bn_workspace_size(int c) {
  return static_cast<size_t>(bn_blocks()) * 2 * c * sizeof(double) + 3 * c * sizeof(float) + 256;
}

extern "C" int b2dl_bn_forward(b2dl_act x, const float* gamma, const float* beta, float eps, b2dl_act residual,
                               int relu, b2dl_act y, float* stats, void* workspace, size_t workspace_bytes, int f32,
                               void* stream) {
  if (!x.ptr || !y.ptr || !gamma || !beta || !stats || x.n != y.n || x.h != y.h || x.w != y.w || x.c != y.c)
    return B2DL_E_VALUE;
  if (!workspace || workspace_bytes < b2dl_bn_workspace_size(x.c)) return B2DL_E_VALUE;
  const int c = x.c;
  const long long npix = static_cast<long long>(x.n) * x.h * x.w;
  const int vw = f32 ? 4 : 8;
  const bool vec = vec_act(x, vw) && vec_act(y, vw) && vec_act(residual, vw);
  const int blocks = bn_blocks();
  double* part = reinterpret_cast<double*>(workspace);
  cudaStream_t st = as_stream(stream);
  const size_t smem = bn_red_smem(c, vec ? vw : 1);
  if (smem > 200 * 1024) return B2DL_E_VALUE;
  B2_TV(f32, vec, {
    auto kern = k_bn_reduce<T, V, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    kern<<<blocks, BN_THREADS, smem, st>>>(reinterpret_cast<const T*>(x.ptr), x.c_stride, nullptr, 0, nullptr,
                                           npix, c, part);
  });
  int rc = check_launch();
  if (rc) return rc;
  k_bn_finalize<double><<<cdiv(c, FIN_CH), FIN_CH * FIN_ROWS, 0, st>>>(part, blocks, c, static_cast<double>(npix),
                                                                        eps, gamma, beta, stats);
  if ((rc = check_launch())) return rc;
  B2_TV(f32, vec, {
    k_bn_apply<T, V><<<stream_blocks(npix, c / V), BN_THREADS, 0, st>>>(
        reinterpret_cast<const T*>(x.ptr), x.c_stride, stats, reinterpret_cast<const T*>(residual.ptr),
        residual.c_stride, relu, reinterpret_cast<T*>(y.ptr), y.c_stride, npix, c);
  });
  return check_launch();
}

extern "C" int b2dl_bn_forward_partials(const float* partials, int tiles, b2dl_act x, const float* gamma,
                                        const float* beta, float eps, b2dl_act residual, int relu, b2dl_act y,
                                        float* stats, void* workspace, size_t workspace_bytes, int f32,
                                        void* stream) {
  if (!partials || tiles < 1 || !x.ptr || !y.ptr || !gamma || !beta || !stats || x.n != y.n || x.h != y.h ||
      x.w != y.w || x.c != y.c)
    return B2DL_E_VALUE;
  if (!workspace || workspace_bytes < b2dl_bn_workspace_size(x.c)) return B2DL_E_VALUE;
  const int c = x.c;
  const long long npix = static_cast<long long>(x.n) * x.h * x.w;
  const int vw = f32 ? 4 : 8;
  const bool vec = vec_act(x, vw) && vec_act(y, vw) && vec_act(residual, vw);
  cudaStream_t st = as_stream(stream);
  int rc;
  if (tiles <= 4 * FIN_ROWS) {   // per-CTA rows (or few tiles): one fixed-order pass
    k_bn_finalize<float><<<cdiv(c, FIN_CH), FIN_CH * FIN_ROWS, 0, st>>>(partials, tiles, c,
                                                                         static_cast<double>(npix), eps, gamma, beta,
                                                                         stats);
  } else {   // per-tile rows: fold contiguous tile ranges first (G rows of fp64), then finalize
    const int G = std::min(bn_blocks(), cdiv(tiles, 4 * FIN_ROWS));
    double* fold = reinterpret_cast<double*>(workspace);
    k_bn_fold_partials<<<dim3(cdiv(c, FIN_CH), G), FIN_CH * FIN_ROWS, 0, st>>>(partials, tiles, c, fold);
    if ((rc = check_launch())) return rc;
    k_bn_finalize<double><<<cdiv(c, FIN_CH), FIN_CH * FIN_ROWS, 0, st>>>(fold, G, c, static_cast<double>(npix), eps,
                                                                          gamma, beta, stats);
  }
  rc = check_launch();
  if (rc) return rc;
  B2_TV(f32, vec, {
    k_bn_apply<T, V><<<stream_blocks(npix, c / V), BN_THREADS, 0, st>>>(
        reinterpret_cast<const T*>(x.ptr), x.c_stride, stats, reinterpret_cast<const T*>(residual.ptr),
        residual.c_stride, relu, reinterpret_cast<T*>(y.ptr), y.c_stride, npix, c);
  });
  return check_launch();
}

extern "C" int b2dl_bn_backward(b2dl_act x, b2dl_act gy, const float* gamma, const float* stats, float* dgamma,
                                float* dbeta, int param_accumulate, b2dl_act dx, int accumulate, void* workspace,
                                size_t workspace_bytes, int f32, void* stream) {
  if (!x.ptr || !gy.ptr || !gamma || !stats || x.n != gy.n || x.h != gy.h || x.w != gy.w || x.c != gy.c)
    return B2DL_E_VALUE;
  if (dx.ptr && (dx.n != x.n || dx.h != x.h || dx.w != x.w || dx.c != x.c)) return B2DL_E_VALUE;
  if (!workspace || workspace_bytes < b2dl_bn_workspace_size(x.c)) return B2DL_E_VALUE;
  const int c = x.c;
  const long long npix = static_cast<long long>(x.n) * x.h * x.w;
  const int vw = f32 ? 4 : 8;
  const bool vec = vec_act(x, vw) && vec_act(gy, vw) && vec_act(dx, vw);
  const int blocks = bn_blocks();
  double* part = reinterpret_cast<double*>(workspace);
  float* coef = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) +
                                         align_up(static_cast<size_t>(blocks) * 2 * c * sizeof(double), 256));
  cudaStream_t st = as_stream(stream);
  const size_t smem = bn_red_smem(c, vec ? vw : 1);
  if (smem > 200 * 1024) return B2DL_E_VALUE;
  B2_TV(f32, vec, {
    auto kern = k_bn_reduce<T, V, true>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    kern<<<blocks, BN_THREADS, smem, st>>>(reinterpret_cast<const T*>(x.ptr), x.c_stride,
                                           reinterpret_cast<const T*>(gy.ptr), gy.c_stride, stats, npix, c, part);
  });
  int rc = check_launch();
  if (rc) return rc;
  k_bn_bwd_finalize<double><<<cdiv(c, FIN_CH), FIN_CH * FIN_ROWS, 0, st>>>(part, blocks, c, static_cast<double>(npix), gamma,
                                                                    stats, dgamma,
                                                   dbeta, param_accumulate, coef);
  if ((rc = check_launch()) || !dx.ptr) return rc;
  B2_TV(f32, vec, {
    k_bn_bwd_apply<T, V><<<stream_blocks(npix, c / V), BN_THREADS, 0, st>>>(
        reinterpret_cast<const T*>(x.ptr), x.c_stride, reinterpret_cast<const T*>(gy.ptr), gy.c_stride, coef,
        reinterpret_cast<T*>(dx.ptr), dx.c_stride, accumulate, npix, c);
  });
  return check_launch();
}

extern "C" int b2dl_bilinear_fwd(b2dl_act x, b2dl_act y, int f, int f32, void* stream) {
  if (!x.ptr || !y.ptr || f < 1 || y.h != x.h * f || y.w != x.w * f || y.c != x.c || y.n != x.n) return B2DL_E_VALUE;
  const int vw = f32 ? 4 : 8;
  const bool vec = vec_act(x, vw) && vec_act(y, vw);
  cudaStream_t st = as_stream(stream);
  B2_TV(f32, vec, {
    k_bilinear_fwd<T, V><<<dim3(y.h, y.n), 256, 0, st>>>(
        reinterpret_cast<const T*>(x.ptr), x.c_stride, reinterpret_cast<T*>(y.ptr), y.c_stride, x.n, x.h, x.w, x.c,
        f);
  });
  return check_launch();
}

extern "C" size_t b2dl_bilinear_workspace_size(b2dl_act dy, int f) {
  if (f < 1) return 0;
  return static_cast<size_t>(dy.n) * dy.h * (dy.w / f) * dy.c * sizeof(float) + 256;
}

extern "C" int b2dl_bilinear_bwd(b2dl_act dy, b2dl_act dx, int f, int accumulate, b2dl_act mask, int f32,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  if (!dy.ptr || !dx.ptr || f < 1 || dy.h != dx.h * f || dy.w != dx.w * f || dy.c != dx.c || dy.n != dx.n)
    return B2DL_E_VALUE;
  if (!workspace || workspace_bytes < b2dl_bilinear_workspace_size(dy, f)) return B2DL_E_VALUE;
  const int vw = f32 ? 4 : 8;
  const bool vec = vec_act(dy, vw) && vec_act(dx, vw) && vec_act(mask, vw);
  float* R = reinterpret_cast<float*>(workspace);
  cudaStream_t st = as_stream(stream);
  B2_TV(f32, vec, {
    k_bilinear_bwd_rows<T, V><<<dim3(dy.h, dy.n), 256, 0, st>>>(reinterpret_cast<const T*>(dy.ptr), dy.c_stride, R,
                                                                dx.h, dx.w, dx.c, f);
  });
  int rc = check_launch();
  if (rc) return rc;
  B2_TV(f32, vec, {
    k_bilinear_bwd_cols<T, V><<<dim3(dx.h, dx.n), 256, 0, st>>>(
        R, reinterpret_cast<T*>(dx.ptr), dx.c_stride, reinterpret_cast<const T*>(mask.ptr), mask.c_stride, dx.h, dx.w,
        dx.c, f, accumulate);
  });
  return check_launch();
}

extern "C" int b2dl_bn_backward_partials(const float* partials, int rows, b2dl_act x, b2dl_act gy,
                                         const float* gamma, const float* stats, float* dgamma, float* dbeta,
                                         int param_accumulate, b2dl_act dx, int accumulate, void* workspace,
                                         size_t workspace_bytes, int f32, void* stream) {
  if (!partials || rows < 1 || !x.ptr || !gy.ptr || !gamma || !stats || x.n != gy.n || x.h != gy.h ||
      x.w != gy.w || x.c != gy.c)
    return B2DL_E_VALUE;
  if (dx.ptr && (dx.n != x.n || dx.h != x.h || dx.w != x.w || dx.c != x.c)) return B2DL_E_VALUE;
  if (!workspace || workspace_bytes < b2dl_bn_workspace_size(x.c)) return B2DL_E_VALUE;
  const int c = x.c;
  const long long npix = static_cast<long long>(x.n) * x.h * x.w;
  cudaStream_t st = as_stream(stream);
  float* coef = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) +
                                         align_up(static_cast<size_t>(bn_blocks()) * 2 * c * sizeof(double), 256));
  int rc;
  if (rows <= 4 * FIN_ROWS) {
    k_bn_bwd_finalize<float><<<cdiv(c, FIN_CH), FIN_CH * FIN_ROWS, 0, st>>>(
        partials, rows, c, static_cast<double>(npix), gamma, stats, dgamma, dbeta, param_accumulate, coef);
  } else {
    const int G = std::min(bn_blocks(), cdiv(rows, 4 * FIN_ROWS));
    double* fold = reinterpret_cast<double*>(workspace);
    k_bn_fold_partials<<<dim3(cdiv(c, FIN_CH), G), FIN_CH * FIN_ROWS, 0, st>>>(partials, rows, c, fold);
    if ((rc = check_launch())) return rc;
    k_bn_bwd_finalize<double><<<cdiv(c, FIN_CH), FIN_CH * FIN_ROWS, 0, st>>>(
        fold, G, c, static_cast<double>(npix), gamma, stats, dgamma, dbeta, param_accumulate, coef);
  }
  if ((rc = check_launch())) return rc;
  if (!dx.ptr) return B2DL_OK;
  const int vw = f32 ? 4 : 8;
  const bool vec = vec_act(x, vw) && vec_act(gy, vw) && vec_act(dx, vw);
  B2_TV(f32, vec, {
    k_bn_bwd_apply<T, V><<<stream_blocks(npix, c / V), BN_THREADS, 0, st>>>(
        reinterpret_cast<const T*>(x.ptr), x.c_stride, reinterpret_cast<const T*>(gy.ptr), gy.c_stride, coef,
        reinterpret_cast<T*>(dx.ptr), dx.c_stride, accumulate, npix, c);
  });
  return check_launch();
}
