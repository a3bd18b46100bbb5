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

__device__ __forceinline__ float ld_bf(const __nv_bfloat16* p) { return __bfloat162float(*p); }

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
      reinterpret_cast<__nv_bfloat16*>(y)[d] = __float2bfloat16_rn(x[i]);
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
    y[i] = f32 ? reinterpret_cast<const float*>(x)[src] : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(x)[src]);
  }
}

// ------------------------------------------------------------------ pool / upsample
// channel pairs per thread (views have even channel offsets and counts in practice; odd c handled scalar)
__global__ void k_avgpool_fwd(const __nv_bfloat16* __restrict__ x, int xs, __nv_bfloat16* __restrict__ y, int ys,
                              int n, int ho, int wo, int c, int k) {
  const int W = wo * k;
  const long long total = static_cast<long long>(n) * ho * wo * c;
  const float inv = 1.f / (k * k);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int ch = static_cast<int>(i % c);
    long long op = i / c;
    int ox = static_cast<int>(op % wo);
    long long r = op / wo;
    int oy = static_cast<int>(r % ho);
    long long img = r / ho;
    float s = 0.f;
    for (int a = 0; a < k; ++a) {
      const __nv_bfloat16* row = x + ((img * ho * k + oy * k + a) * W + ox * k) * xs + ch;
      for (int b = 0; b < k; ++b) s += ld_bf(row + static_cast<long long>(b) * xs);
    }
    y[op * ys + ch] = __float2bfloat16_rn(s * inv);
  }
}
// dx[p] (+)= mask(dx_fwd)[p] * dy[pool(p)] / k^2
__global__ void k_avgpool_bwd(const __nv_bfloat16* __restrict__ dy, int dys, __nv_bfloat16* __restrict__ dx, int dxs,
                              const __nv_bfloat16* __restrict__ mask, int ms, int n, int h, int w, int c, int k,
                              int acc) {
  const long long total = static_cast<long long>(n) * h * w * c;
  const int wo = w / k, ho = h / k;
  const float inv = 1.f / (k * k);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int ch = static_cast<int>(i % c);
    long long p = i / c;
    int xx = static_cast<int>(p % w);
    long long r = p / w;
    int yy = static_cast<int>(r % h);
    long long img = r / h;
    float v = ld_bf(dy + ((img * ho + yy / k) * wo + xx / k) * dys + ch) * inv;
    if (mask && !(ld_bf(mask + p * ms + ch) > 0.f)) v = 0.f;
    __nv_bfloat16* d = dx + p * dxs + ch;
    if (acc) v += ld_bf(d);
    *d = __float2bfloat16_rn(v);
  }
}
__global__ void k_upsample_fwd(const __nv_bfloat16* __restrict__ x, int xs, __nv_bfloat16* __restrict__ y, int ys,
                               int n, int h, int w, int c, int f) {
  // y is [n, h*f, w*f]; 8 channels (16 B) per thread when aligned
  const int H = h * f, W = w * f;
  const bool vec = (c % 8 == 0) && (xs % 8 == 0) && (ys % 8 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(y) & 15) == 0);
  const int cg = vec ? c / 8 : c;
  const long long total = static_cast<long long>(n) * H * W * cg;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int g = static_cast<int>(i % cg);
    long long p = i / cg;
    int xx = static_cast<int>(p % W);
    long long r = p / W;
    int yy = static_cast<int>(r % H);
    long long img = r / H;
    long long sp = (img * h + yy / f) * w + xx / f;
    if (vec) {
      *reinterpret_cast<uint4*>(y + p * ys + g * 8) = __ldg(reinterpret_cast<const uint4*>(x + sp * xs + g * 8));
    } else {
      y[p * ys + g] = x[sp * xs + g];
    }
  }
}
// dx[q] (+)= sum over the f x f block of mask(dy_fwd) * dy
__global__ void k_upsample_bwd(const __nv_bfloat16* __restrict__ dy, int dys, __nv_bfloat16* __restrict__ dx, int dxs,
                               const __nv_bfloat16* __restrict__ mask, int ms, int n, int h, int w, int c, int f,
                               int acc) {
  const int W = w * f;
  const long long total = static_cast<long long>(n) * h * w * c;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int ch = static_cast<int>(i % c);
    long long q = i / c;
    int xx = static_cast<int>(q % w);
    long long r = q / w;
    int yy = static_cast<int>(r % h);
    long long img = r / h;
    float s = 0.f;
    for (int a = 0; a < f; ++a) {
      long long rowp = (img * h * f + yy * f + a) * W + xx * f;
      for (int b = 0; b < f; ++b) {
        long long pp = rowp + b;
        float v = ld_bf(dy + pp * dys + ch);
        if (mask && !(ld_bf(mask + pp * ms + ch) > 0.f)) v = 0.f;
        s += v;
      }
    }
    __nv_bfloat16* d = dx + q * dxs + ch;
    if (acc) s += ld_bf(d);
    *d = __float2bfloat16_rn(s);
  }
}

// ------------------------------------------------------------------ add / mask
__global__ void k_add(const __nv_bfloat16* __restrict__ x, int xs, __nv_bfloat16* __restrict__ y, int ys,
                      const __nv_bfloat16* __restrict__ mask, int ms, long long npix, int c, int acc) {
  const long long total = npix * c;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int ch = static_cast<int>(i % c);
    long long p = i / c;
    float v = ld_bf(x + p * xs + ch);
    if (mask && !(ld_bf(mask + p * ms + ch) > 0.f)) v = 0.f;
    __nv_bfloat16* d = y + p * ys + ch;
    if (acc) v += ld_bf(d);
    *d = __float2bfloat16_rn(v);
  }
}
__global__ void k_add_vec(const __nv_bfloat16* __restrict__ x, int xs, __nv_bfloat16* __restrict__ y, int ys,
                          const __nv_bfloat16* __restrict__ mask, int ms, long long npix, int c, int acc) {
  const int cg = c / 8;
  const long long total = npix * cg;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int g = static_cast<int>(i % cg);
    long long p = i / cg;
    uint4 xv = __ldg(reinterpret_cast<const uint4*>(x + p * xs + g * 8));
    uint4 mv = mask ? __ldg(reinterpret_cast<const uint4*>(mask + p * ms + g * 8)) : make_uint4(0, 0, 0, 0);
    uint4* dp = reinterpret_cast<uint4*>(y + p * ys + g * 8);
    uint4 yv = acc ? *dp : make_uint4(0, 0, 0, 0);
    const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(&xv);
    const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&mv);
    __nv_bfloat16* yb = reinterpret_cast<__nv_bfloat16*>(&yv);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      float v = __bfloat162float(xb[e]);
      if (mask && !(__bfloat162float(mb[e]) > 0.f)) v = 0.f;
      if (acc) v += __bfloat162float(yb[e]);
      yb[e] = __float2bfloat16_rn(v);
    }
    *dp = yv;
  }
}
__global__ void k_relu_mask(__nv_bfloat16* __restrict__ g, int gs, const __nv_bfloat16* __restrict__ a, int as,
                            long long npix, int c) {
  const long long total = npix * c;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int ch = static_cast<int>(i % c);
    long long p = i / c;
    if (!(ld_bf(a + p * as + ch) > 0.f)) g[p * gs + ch] = __float2bfloat16_rn(0.f);
  }
}

// ------------------------------------------------------------------ bias gradient
// pass 1: partial[b][c] = sum over pixels p = b, b+G, ... ; pass 2: out[c] (+)= sum_b partial[b][c]
__global__ void k_colsum_partial(const __nv_bfloat16* __restrict__ g, int gs, long long npix, int c,
                                 float* __restrict__ part) {
  for (int ch = threadIdx.x; ch < c; ch += blockDim.x) {
    float s = 0.f;
    for (long long p = blockIdx.x; p < npix; p += gridDim.x) s += ld_bf(g + p * gs + ch);
    part[static_cast<long long>(blockIdx.x) * c + ch] = s;
  }
}
__global__ void k_colsum_final(const float* __restrict__ part, int nb, int c, float* __restrict__ out, int acc) {
  int ch = blockIdx.x * blockDim.x + threadIdx.x;
  if (ch >= c) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[static_cast<long long>(b) * c + ch];
  out[ch] = static_cast<float>(acc ? out[ch] + s : s);
}

static int colsum_blocks(long long npix) {
  return static_cast<int>(std::max<long long>(1, std::min<long long>(npix, 4LL * num_sms())));
}

// ------------------------------------------------------------------ weight packing
// master HWIO fp32 [taps][cin][cout] -> fprop [cout][taps][cin_pad] and dgrad [cin][taps'][cout_pad]
__global__ void k_pack_fprop(const float* __restrict__ w, __nv_bfloat16* __restrict__ out, int taps, int cin,
                             int cout, int cin_pad) {
  const long long total = static_cast<long long>(cout) * taps * cin_pad;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int ci = static_cast<int>(i % cin_pad);
    long long r = i / cin_pad;
    int t = static_cast<int>(r % taps);
    int co = static_cast<int>(r / taps);
    out[i] = __float2bfloat16_rn(ci < cin ? w[(static_cast<long long>(t) * cin + ci) * cout + co] : 0.f);
  }
}
__global__ void k_pack_dgrad(const float* __restrict__ w, __nv_bfloat16* __restrict__ out, int taps, int cin,
                             int cout, int cout_pad) {
  const long long total = static_cast<long long>(cin) * taps * cout_pad;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int co = static_cast<int>(i % cout_pad);
    long long r = i / cout_pad;
    int tf = static_cast<int>(r % taps);
    int ci = static_cast<int>(r / taps);
    int t = taps - 1 - tf;
    out[i] = __float2bfloat16_rn(co < cout ? w[(static_cast<long long>(t) * cin + ci) * cout + co] : 0.f);
  }
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace b2

using namespace b2;
#define BF(p) reinterpret_cast<__nv_bfloat16*>(p)
#define CBF(p) reinterpret_cast<const __nv_bfloat16*>(p)

extern "C" int b2dl_nchw_to_nhwc(const float* x, b2dl_act y, int dst_f32, void* stream) {
  if (!x || !y.ptr) return B2DL_E_VALUE;
  long long total = static_cast<long long>(y.n) * y.c * y.h * y.w;
  k_nchw_to_nhwc<<<grid1d(total), 256, 0, as_stream(stream)>>>(x, y.ptr, dst_f32, y.n, y.c, y.h, y.w, y.c_stride);
  return check_launch();
}

extern "C" int b2dl_nhwc_to_nchw(b2dl_act x, int src_f32, float* y, void* stream) {
  if (!y || !x.ptr) return B2DL_E_VALUE;
  long long total = static_cast<long long>(x.n) * x.c * x.h * x.w;
  k_nhwc_to_nchw<<<grid1d(total), 256, 0, as_stream(stream)>>>(x.ptr, src_f32, y, x.n, x.c, x.h, x.w, x.c_stride);
  return check_launch();
}

extern "C" int b2dl_avgpool_fwd(b2dl_act x, b2dl_act y, int k, void* stream) {
  if (k < 1 || x.h % k || x.w % k || y.h != x.h / k || y.w != x.w / k || y.c != x.c || y.n != x.n) return B2DL_E_VALUE;
  long long total = static_cast<long long>(y.n) * y.h * y.w * y.c;
  k_avgpool_fwd<<<grid1d(total), 256, 0, as_stream(stream)>>>(CBF(x.ptr), x.c_stride, BF(y.ptr), y.c_stride, y.n, y.h,
                                                              y.w, y.c, k);
  return check_launch();
}

extern "C" int b2dl_avgpool_bwd(b2dl_act dy, b2dl_act dx, int k, int accumulate, b2dl_act mask, void* stream) {
  if (k < 1 || dx.h != dy.h * k || dx.w != dy.w * k || dx.c != dy.c) return B2DL_E_VALUE;
  long long total = static_cast<long long>(dx.n) * dx.h * dx.w * dx.c;
  k_avgpool_bwd<<<grid1d(total), 256, 0, as_stream(stream)>>>(CBF(dy.ptr), dy.c_stride, BF(dx.ptr), dx.c_stride,
                                                              CBF(mask.ptr), mask.c_stride, dx.n, dx.h, dx.w, dx.c, k,
                                                              accumulate);
  return check_launch();
}

extern "C" int b2dl_upsample_fwd(b2dl_act x, b2dl_act y, int f, void* stream) {
  if (f < 1 || y.h != x.h * f || y.w != x.w * f || y.c != x.c) return B2DL_E_VALUE;
  long long total = static_cast<long long>(y.n) * y.h * y.w * y.c;
  k_upsample_fwd<<<grid1d(total, 8), 256, 0, as_stream(stream)>>>(CBF(x.ptr), x.c_stride, BF(y.ptr), y.c_stride, x.n,
                                                                  x.h, x.w, x.c, f);
  return check_launch();
}

extern "C" int b2dl_upsample_bwd(b2dl_act dy, b2dl_act dx, int f, int accumulate, b2dl_act mask, void* stream) {
  if (f < 1 || dy.h != dx.h * f || dy.w != dx.w * f || dy.c != dx.c) return B2DL_E_VALUE;
  long long total = static_cast<long long>(dx.n) * dx.h * dx.w * dx.c;
  k_upsample_bwd<<<grid1d(total), 256, 0, as_stream(stream)>>>(CBF(dy.ptr), dy.c_stride, BF(dx.ptr), dx.c_stride,
                                                               CBF(mask.ptr), mask.c_stride, dx.n, dx.h, dx.w, dx.c, f,
                                                               accumulate);
  return check_launch();
}

extern "C" int b2dl_add(b2dl_act x, b2dl_act y, int accumulate, b2dl_act mask, void* stream) {
  if (x.c != y.c || x.h != y.h || x.w != y.w || x.n != y.n) return B2DL_E_VALUE;
  long long npix = static_cast<long long>(x.n) * x.h * x.w;
  bool vec = x.c % 8 == 0 && x.c_stride % 8 == 0 && y.c_stride % 8 == 0 && aligned16(x.ptr) && aligned16(y.ptr) &&
             (!mask.ptr || (mask.c_stride % 8 == 0 && aligned16(mask.ptr)));
  if (vec)
    k_add_vec<<<grid1d(npix * x.c, 8), 256, 0, as_stream(stream)>>>(CBF(x.ptr), x.c_stride, BF(y.ptr), y.c_stride,
                                                                     CBF(mask.ptr), mask.c_stride, npix, x.c,
                                                                     accumulate);
  else
    k_add<<<grid1d(npix * x.c), 256, 0, as_stream(stream)>>>(CBF(x.ptr), x.c_stride, BF(y.ptr), y.c_stride,
                                                             CBF(mask.ptr), mask.c_stride, npix, x.c, accumulate);
  return check_launch();
}

extern "C" int b2dl_relu_mask(b2dl_act g, b2dl_act act, void* stream) {
  if (g.c != act.c || g.h != act.h || g.w != act.w || g.n != act.n) return B2DL_E_VALUE;
  long long npix = static_cast<long long>(g.n) * g.h * g.w;
  k_relu_mask<<<grid1d(npix * g.c), 256, 0, as_stream(stream)>>>(BF(g.ptr), g.c_stride, CBF(act.ptr), act.c_stride,
                                                                 npix, g.c);
  return check_launch();
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
  k_colsum_partial<<<nb, 256, 0, as_stream(stream)>>>(CBF(g.ptr), g.c_stride, npix, g.c, part);
  int rc = check_launch();
  if (rc) return rc;
  k_colsum_final<<<(g.c + 127) / 128, 128, 0, as_stream(stream)>>>(part, nb, g.c, out, accumulate);
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
