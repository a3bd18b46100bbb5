// Standalone lowerings of the reference's remaining op kinds, so any graph built from its op set
// (pkg/src/deskdl/graph.py:16-26) runs through the engine, not only conv-bias-relu chains:
//   elementwise  mul / scale (ops.py:142-148, VJPs :195-202), standalone bias_add (:122-126,
//                :172-175) and relu (:127-128, :176-177) -- one fused stream kernel
//                y (+)= mask? . relu?( alpha . x0 . x1? + bias[c]? )
//   matmul       Y = X @ B over the last (width) axis of an NCHW activation (ops.py:120,166-170):
//                per image row, Y[w2, c] = sum_w B[w, w2] X[w, c] in NHWC; the input gradient is
//                the same product with B transposed; the B gradient sums X[w, c] G[w2, c] over
//                every (n, h, c) in a fixed order (deterministic, no atomics).
// Storage is bf16 (training step) or fp32 (parity mode); arithmetic is fp32, parameters are read
// from the fp32 master.  These are HBM- or latency-bound side ops (no DeepLabV3+ / MiniDenseNet
// layer uses them); the tensor-core convs stay the hot path.
#include <cuda_bf16.h>

#include <algorithm>

#include "internal.h"

namespace b2 {
namespace {

template <typename T>
__device__ __forceinline__ float ldf(const T* p);
template <>
__device__ __forceinline__ float ldf<float>(const float* p) {
  return *p;
}
template <>
__device__ __forceinline__ float ldf<b2h>(const b2h* p) {
  return h_to_f(*p);
}
template <typename T>
__device__ __forceinline__ void stf(T* p, float v);
template <>
__device__ __forceinline__ void stf<float>(float* p, float v) {
  *p = v;
}
template <>
__device__ __forceinline__ void stf<b2h>(b2h* p, float v) {
  *p = f_to_h(v);
}

struct EwiseP {
  const void* x0;
  int s0;
  const void* x1;
  int s1;
  const void* mask;
  int sm;
  void* y;
  int sy;
  const float* bias;
  float alpha;
  int relu, accumulate;
  long long npix;
  int c;
};

template <typename T>
__global__ void k_ewise(const EwiseP p) {
  const long long total = p.npix * p.c;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i % p.c);
    const long long q = i / p.c;
    float v = p.alpha * ldf(static_cast<const T*>(p.x0) + q * p.s0 + ch);
    if (p.x1) v *= ldf(static_cast<const T*>(p.x1) + q * p.s1 + ch);
    if (p.bias) v += p.bias[ch];
    if (p.relu) v = fmaxf(v, 0.f);
    if (p.mask && !(ldf(static_cast<const T*>(p.mask) + q * p.sm + ch) > 0.f)) v = 0.f;
    T* o = static_cast<T*>(p.y) + q * p.sy + ch;
    if (p.accumulate) v += ldf(o);
    stf(o, v);
  }
}

// Y[n, h, j, c] (+)= sum_i X[n, h, i, c] coef(i, j); coef = trans ? B[j * ldb + i] : B[i * ldb + j]
constexpr int MM_TJ = 16, MM_TC = 32;
struct MatmulP {
  const void* x;
  int sx, wi;
  const float* b;
  int ldb, trans;
  void* y;
  int sy, wo;
  const void* mask;
  int sm;
  int rows, c, accumulate;
};

template <typename T>
__global__ void __launch_bounds__(MM_TJ* MM_TC) k_matmul_w(const MatmulP p) {
  // block: one image row (n, h), MM_TJ output columns x MM_TC channels; threads (j, c)
  const int row = blockIdx.x;
  const int j = blockIdx.y * MM_TJ + threadIdx.x / MM_TC;
  const int ch = blockIdx.z * MM_TC + threadIdx.x % MM_TC;
  if (j >= p.wo || ch >= p.c) return;
  const T* xr = static_cast<const T*>(p.x) + static_cast<long long>(row) * p.wi * p.sx;
  float acc = 0.f;
  for (int i = 0; i < p.wi; ++i) {
    const float cf = p.trans ? p.b[static_cast<long long>(j) * p.ldb + i] : p.b[static_cast<long long>(i) * p.ldb + j];
    acc = fmaf(ldf(xr + static_cast<long long>(i) * p.sx + ch), cf, acc);
  }
  const long long q = static_cast<long long>(row) * p.wo + j;
  if (p.mask && !(ldf(static_cast<const T*>(p.mask) + q * p.sm + ch) > 0.f)) acc = 0.f;
  T* o = static_cast<T*>(p.y) + q * p.sy + ch;
  if (p.accumulate) acc += ldf(o);
  stf(o, acc);
}

// gB[i, j] (+)= sum_{rows, c} X[row, i, c] G[row, j, c]: one thread per (i, j), fixed loop order
struct MatmulGradP {
  const void* x;
  int sx, wi;
  const void* g;
  int sg, wo;
  int rows, c;
  float* gb;
  int accumulate;
};

template <typename T>
__global__ void __launch_bounds__(256) k_matmul_w_grad(const MatmulGradP p) {
  const int i = blockIdx.x * 16 + threadIdx.x / 16;
  const int j = blockIdx.y * 16 + threadIdx.x % 16;
  if (i >= p.wi || j >= p.wo) return;
  float acc = 0.f;
  for (int r = 0; r < p.rows; ++r) {
    const T* xr = static_cast<const T*>(p.x) + (static_cast<long long>(r) * p.wi + i) * p.sx;
    const T* gr = static_cast<const T*>(p.g) + (static_cast<long long>(r) * p.wo + j) * p.sg;
    for (int ch = 0; ch < p.c; ++ch) acc = fmaf(ldf(xr + ch), ldf(gr + ch), acc);
  }
  float* o = p.gb + static_cast<long long>(i) * p.wo + j;
  *o = p.accumulate ? *o + acc : acc;
}

// out[c] (+)= sum over pixels of g[p][c] (the bias_add VJP, ops.py:172-175): 8 pixel lanes per
// channel column, summed in a fixed order
template <typename T>
__global__ void __launch_bounds__(256) k_channel_sum(const T* __restrict__ g, int gs, long long npix, int c,
                                                     float* __restrict__ out, int accumulate) {
  __shared__ float part[8][33];
  const int cl = threadIdx.x % 32, row = threadIdx.x / 32;
  const int ch = blockIdx.x * 32 + cl;
  float s = 0.f;
  if (ch < c)
    for (long long q = row; q < npix; q += 8) s += ldf(g + q * gs + ch);
  part[row][cl] = s;
  __syncthreads();
  if (row == 0 && ch < c) {
    float t = 0.f;
#pragma unroll
    for (int r = 0; r < 8; ++r) t += part[r][cl];
    out[ch] = accumulate ? out[ch] + t : t;
  }
}

bool same_px(const b2dl_act& a, const b2dl_act& b) { return a.n == b.n && a.h == b.h && a.w == b.w && a.c == b.c; }

int grid_for(long long total) {
  return static_cast<int>(std::max<long long>(1, std::min<long long>((total + 255) / 256, 16LL * num_sms())));
}

}  // namespace
}  // namespace b2

using namespace b2;

extern "C" int b2dl_ewise(b2dl_act x0, b2dl_act x1, b2dl_act mask, b2dl_act y, const float* bias, float alpha,
                          int relu, int accumulate, int f32, void* stream) {
  if (!x0.ptr || !y.ptr || !same_px(x0, y)) return B2DL_E_VALUE;
  if ((x1.ptr && !same_px(x1, y)) || (mask.ptr && !same_px(mask, y))) return B2DL_E_VALUE;
  EwiseP p{x0.ptr, x0.c_stride, x1.ptr, x1.c_stride, mask.ptr, mask.c_stride, y.ptr, y.c_stride, bias, alpha,
           relu, accumulate, static_cast<long long>(y.n) * y.h * y.w, y.c};
  const int grid = grid_for(p.npix * p.c);
  if (f32)
    k_ewise<float><<<grid, 256, 0, as_stream(stream)>>>(p);
  else
    k_ewise<b2h><<<grid, 256, 0, as_stream(stream)>>>(p);
  return check_launch();
}

extern "C" int b2dl_matmul_w(b2dl_act x, const float* b, int ldb, int trans, b2dl_act y, b2dl_act mask,
                             int accumulate, int f32, void* stream) {
  if (!x.ptr || !b || !y.ptr || x.n != y.n || x.h != y.h || x.c != y.c) return B2DL_E_VALUE;
  if (mask.ptr && !same_px(mask, y)) return B2DL_E_VALUE;
  if (ldb != (trans ? x.w : y.w)) return B2DL_E_VALUE;
  MatmulP p{x.ptr, x.c_stride, x.w, b, ldb, trans, y.ptr, y.c_stride, y.w, mask.ptr, mask.c_stride, x.n * x.h, y.c,
            accumulate};
  if (p.rows == 0 || y.w == 0 || y.c == 0) return B2DL_OK;
  const dim3 grid(p.rows, cdiv(y.w, MM_TJ), cdiv(y.c, MM_TC));
  if (grid.y > 65535 || grid.z > 65535) return B2DL_E_VALUE;
  if (f32)
    k_matmul_w<float><<<grid, MM_TJ * MM_TC, 0, as_stream(stream)>>>(p);
  else
    k_matmul_w<b2h><<<grid, MM_TJ * MM_TC, 0, as_stream(stream)>>>(p);
  return check_launch();
}

extern "C" int b2dl_matmul_w_grad(b2dl_act x, b2dl_act g, float* gb, int accumulate, int f32, void* stream) {
  if (!x.ptr || !g.ptr || !gb || x.n != g.n || x.h != g.h || x.c != g.c) return B2DL_E_VALUE;
  MatmulGradP p{x.ptr, x.c_stride, x.w, g.ptr, g.c_stride, g.w, x.n * x.h, x.c, gb, accumulate};
  if (x.w == 0 || g.w == 0) return B2DL_OK;
  const dim3 grid(cdiv(x.w, 16), cdiv(g.w, 16));
  if (f32)
    k_matmul_w_grad<float><<<grid, 256, 0, as_stream(stream)>>>(p);
  else
    k_matmul_w_grad<b2h><<<grid, 256, 0, as_stream(stream)>>>(p);
  return check_launch();
}

extern "C" int b2dl_channel_sum(b2dl_act g, float* out, int accumulate, int f32, void* stream) {
  if (!g.ptr || !out) return B2DL_E_VALUE;
  const long long npix = static_cast<long long>(g.n) * g.h * g.w;
  if (g.c == 0) return B2DL_OK;
  if (f32)
    k_channel_sum<float><<<cdiv(g.c, 32), 256, 0, as_stream(stream)>>>(static_cast<const float*>(g.ptr), g.c_stride,
                                                                        npix, g.c, out, accumulate);
  else
    k_channel_sum<b2h><<<cdiv(g.c, 32), 256, 0, as_stream(stream)>>>(
        static_cast<const b2h*>(g.ptr), g.c_stride, npix, g.c, out, accumulate);
  return check_launch();
}
