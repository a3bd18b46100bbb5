// fp32 parity mode (the reference's arithmetic type end to end, north-star "1e-3 in fp32
// mode"): NHWC fp32 activations, fp32 HWIO weights, fp32 FMA accumulation on the CUDA cores.
// Same operations and fusion points as the bf16 tensor-core path -- implicit-GEMM conv with
// the fused bias / residual / relu / relu'-mask / accumulate epilogue, dgrad as a conv over dy
// with tap-flipped weights and "after" pads, split-K wgrad with a fixed-order reduction and the
// bias column sums, and the pool / upsample / add / relu-mask streams -- so the engine can run
// one program in either precision.  Throughput is not the point of this mode (config 1 is a
// 16 x 288 x 192 tile); agreement with the reference's fp32 step is.
#include <algorithm>

#include "internal.h"

namespace b2 {

constexpr int F_BM = 64, F_BN = 64, F_BK = 16, F_THREADS = 256;

struct F32ConvParams {
  const float* in;  // NHWC, pixel pitch in_stride
  int n, h, w, k, in_stride;
  const float* wt;  // HWIO of the forward conv
  int mode;         // 1: W(tap, k, n) = wt[tap][k][n]; 2: W(tap, k, n) = wt[T-1-tap][n][k] (dgrad)
  int kh, kw, dil, pad_top, pad_left, taps, wk, wn;  // wk x wn = HWIO cin x cout of the forward conv
  float* out;
  int nout, out_stride;
  const float* bias;
  const float* res;
  int res_stride;
  const float* mask;
  int mask_stride;
  int relu, accumulate;
};

__global__ void __launch_bounds__(F_THREADS) k_conv_f32(const F32ConvParams p) {
  __shared__ float As[F_BK][F_BM + 4];
  __shared__ float Bs[F_BK][F_BN + 4];
  const int t = threadIdx.x;
  const long long npix = static_cast<long long>(p.n) * p.h * p.w;
  const long long p0 = static_cast<long long>(blockIdx.x) * F_BM;
  const int n0 = blockIdx.y * F_BN;
  // A-load role: one pixel, 4 consecutive k
  const int a_px = t % F_BM, a_k = (t / F_BM) * 4;
  const long long ap = p0 + a_px;
  int ay = 0, ax = 0, aimg = 0;
  if (ap < npix) {
    aimg = static_cast<int>(ap / (static_cast<long long>(p.h) * p.w));
    const int r = static_cast<int>(ap - static_cast<long long>(aimg) * p.h * p.w);
    ay = r / p.w;
    ax = r - ay * p.w;
  }
  // B-load role: one k, 4 consecutive n
  const int b_k = t / 16, b_n = (t % 16) * 4;
  // compute role: 4 pixels x 4 channels
  const int c_px = (t % 16) * 4, c_n = (t / 16) * 4;
  float acc[4][4] = {};
  for (int tap = 0; tap < p.taps; ++tap) {
    const int i = tap / p.kw, j = tap - i * p.kw;
    const int sy = ay + i * p.dil - p.pad_top, sx = ax + j * p.dil - p.pad_left;
    const bool a_ok = ap < npix && sy >= 0 && sy < p.h && sx >= 0 && sx < p.w;
    const float* arow = p.in + ((static_cast<long long>(aimg) * p.h + sy) * p.w + sx) * p.in_stride;
    const int wtap = p.mode == 1 ? tap : p.taps - 1 - tap;
    for (int k0 = 0; k0 < p.k; k0 += F_BK) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kk = k0 + a_k + e;
        As[a_k + e][a_px] = (a_ok && kk < p.k) ? __ldg(arow + kk) : 0.f;
      }
      const int bk = k0 + b_k;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int nn = n0 + b_n + e;
        float v = 0.f;
        if (bk < p.k && nn < p.nout)
          v = p.mode == 1 ? __ldg(p.wt + (static_cast<long long>(wtap) * p.wk + bk) * p.wn + nn)
                          : __ldg(p.wt + (static_cast<long long>(wtap) * p.wk + nn) * p.wn + bk);
        Bs[b_k][b_n + e] = v;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < F_BK; ++kk) {
        float a[4], b[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          a[e] = As[kk][c_px + e];
          b[e] = Bs[kk][c_n + e];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(a[u], b[v], acc[u][v]);
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const long long pp = p0 + c_px + u;
    if (pp >= npix) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int nn = n0 + c_n + v;
      if (nn >= p.nout) continue;
      float x = acc[u][v];
      if (p.bias) x += p.bias[nn];
      if (p.res) x += p.res[pp * p.res_stride + nn];
      if (p.relu) x = fmaxf(x, 0.f);
      if (p.mask && !(p.mask[pp * p.mask_stride + nn] > 0.f)) x = 0.f;
      float* o = p.out + pp * p.out_stride + nn;
      *o = p.accumulate ? *o + x : x;
    }
  }
}

// dW partials: part[s][tap][ci][co] = sum over split s's pixels of x[p + off(tap)][ci] * dy[p][co];
// bias partials bpart[s][co] = sum over split s's pixels of dy[p][co] (from the tap-0, ci-tile-0 blocks)
struct F32WgradParams {
  const float* x;
  int n, h, w, cin, x_stride;
  const float* dy;
  int cout, dy_stride;
  int kw, dil, pad_top, pad_left, taps;
  int splits;
  long long per_split;
  float* part;
  float* bpart;
};

__global__ void __launch_bounds__(F_THREADS) k_wgrad_f32(const F32WgradParams p) {
  __shared__ float Xs[F_BK][F_BM + 4];
  __shared__ float Ds[F_BK][F_BN + 4];
  const int t = threadIdx.x;
  const int ci0 = blockIdx.x * F_BM, co0 = blockIdx.y * F_BN;
  const int tap = blockIdx.z % p.taps, s = blockIdx.z / p.taps;
  const int i = tap / p.kw, j = tap - i * p.kw;
  const long long npix = static_cast<long long>(p.n) * p.h * p.w;
  const long long lo = s * p.per_split, hi = std::min(npix, lo + p.per_split);
  const int l_px = t / 16, l_c = (t % 16) * 4;  // load role: one pixel row, 4 channels
  const int c_ci = (t % 16) * 4, c_co = (t / 16) * 4;
  float acc[4][4] = {};
  float bsum = 0.f;  // threads t < 64: column t of dy (bias) within this block's co tile
  const bool do_bias = p.bpart && tap == 0 && blockIdx.x == 0;
  for (long long q0 = lo; q0 < hi; q0 += F_BK) {
    const long long q = q0 + l_px;
    float xv[4] = {0.f, 0.f, 0.f, 0.f}, dv[4] = {0.f, 0.f, 0.f, 0.f};
    if (q < hi) {
      const int img = static_cast<int>(q / (static_cast<long long>(p.h) * p.w));
      const int r = static_cast<int>(q - static_cast<long long>(img) * p.h * p.w);
      const int y = r / p.w, x = r - y * p.w;
      const int sy = y + i * p.dil - p.pad_top, sx = x + j * p.dil - p.pad_left;
      if (sy >= 0 && sy < p.h && sx >= 0 && sx < p.w) {
        const float* xr = p.x + ((static_cast<long long>(img) * p.h + sy) * p.w + sx) * p.x_stride;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (ci0 + l_c + e < p.cin) xv[e] = __ldg(xr + ci0 + l_c + e);
      }
      const float* dr = p.dy + q * p.dy_stride;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (co0 + l_c + e < p.cout) dv[e] = __ldg(dr + co0 + l_c + e);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      Xs[l_px][l_c + e] = xv[e];
      Ds[l_px][l_c + e] = dv[e];
    }
    __syncthreads();
    if (do_bias && t < F_BN) {
#pragma unroll
      for (int kk = 0; kk < F_BK; ++kk) bsum += Ds[kk][t];
    }
#pragma unroll
    for (int kk = 0; kk < F_BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        a[e] = Xs[kk][c_ci + e];
        b[e] = Ds[kk][c_co + e];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
  float* dst = p.part + static_cast<long long>(s) * p.taps * p.cin * p.cout;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int ci = ci0 + c_ci + u;
    if (ci >= p.cin) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int co = co0 + c_co + v;
      if (co < p.cout) dst[(static_cast<long long>(tap) * p.cin + ci) * p.cout + co] = acc[u][v];
    }
  }
  if (do_bias && t < F_BN && co0 + t < p.cout) p.bpart[static_cast<long long>(s) * p.cout + co0 + t] = bsum;
}

// out[i] (+)= sum_s part[s][i]  (fixed order)
__global__ void k_reduce_f32(const float* __restrict__ part, long long total, int splits, float* __restrict__ out,
                             int accumulate) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float s = accumulate ? out[i] : 0.f;
    for (int k = 0; k < splits; ++k) s += part[k * total + i];
    out[i] = s;
  }
}

// ---- memory-bound streams, fp32 NHWC views (pixel pitch in elements)
__global__ void k_avgpool_fwd_f32(const float* x, int xs, float* y, int ys, int n, int ho, int wo, int c, int k) {
  const long long total = static_cast<long long>(n) * ho * wo * c;
  const float inv = 1.f / (k * k);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i % c);
    const long long q = i / c;
    const int xo = static_cast<int>(q % wo);
    const long long r = q / wo;
    const int yo = static_cast<int>(r % ho);
    const long long img = r / ho;
    float s = 0.f;
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) s += x[((img * ho * k + yo * k + a) * (wo * k) + xo * k + b) * xs + ch];
    y[q * ys + ch] = s * inv;
  }
}
__global__ void k_avgpool_bwd_f32(const float* dy, int dys, float* dx, int dxs, const float* m, int ms, int n, int ho,
                                  int wo, int c, int k, int acc) {
  const int H = ho * k, W = wo * k;
  const long long total = static_cast<long long>(n) * H * W * c;
  const float inv = 1.f / (k * k);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i % c);
    const long long q = i / c;
    const int xx = static_cast<int>(q % W);
    const long long r = q / W;
    const int yy = static_cast<int>(r % H);
    const long long img = r / H;
    float v = dy[((img * ho + yy / k) * wo + xx / k) * dys + ch] * inv;
    if (m && !(m[q * ms + ch] > 0.f)) v = 0.f;
    float* o = dx + q * dxs + ch;
    *o = acc ? *o + v : v;
  }
}
__global__ void k_upsample_fwd_f32(const float* x, int xs, float* y, int ys, int n, int h, int w, int c, int f) {
  const int H = h * f, W = w * f;
  const long long total = static_cast<long long>(n) * H * W * c;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i % c);
    const long long q = i / c;
    const int xx = static_cast<int>(q % W);
    const long long r = q / W;
    const int yy = static_cast<int>(r % H);
    const long long img = r / H;
    y[q * ys + ch] = x[((img * h + yy / f) * w + xx / f) * xs + ch];
  }
}
__global__ void k_upsample_bwd_f32(const float* dy, int dys, float* dx, int dxs, const float* m, int ms, int n, int h,
                                   int w, int c, int f, int acc) {
  const int W = w * f;
  const long long total = static_cast<long long>(n) * h * w * c;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i % c);
    const long long q = i / c;
    const int xo = static_cast<int>(q % w);
    const long long r = q / w;
    const int yo = static_cast<int>(r % h);
    const long long img = r / h;
    float s = 0.f;
    for (int a = 0; a < f; ++a)
      for (int b = 0; b < f; ++b) s += dy[((img * h * f + yo * f + a) * W + xo * f + b) * dys + ch];
    if (m && !(m[q * ms + ch] > 0.f)) s = 0.f;
    float* o = dx + q * dxs + ch;
    *o = acc ? *o + s : s;
  }
}
__global__ void k_add_f32(const float* x, int xs, float* y, int ys, const float* m, int ms, long long npix, int c,
                          int acc) {
  const long long total = npix * c;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int ch = static_cast<int>(i % c);
    const long long q = i / c;
    float v = x[q * xs + ch];
    if (m && !(m[q * ms + ch] > 0.f)) v = 0.f;
    float* o = y + q * ys + ch;
    *o = acc ? *o + v : v;
  }
}

static int grid_f32(long long total) {
  return static_cast<int>(std::max<long long>(1, std::min<long long>((total + 255) / 256, 16LL * num_sms())));
}

}  // namespace b2

using namespace b2;
#define F(p) reinterpret_cast<float*>(p)
#define CF(p) reinterpret_cast<const float*>(p)

extern "C" int b2dl_f32_conv_fprop(const b2dl_conv_args* a, void* stream) {
  if (!a || !a->x.ptr || !a->y.ptr || !a->w_master || (a->w_mode != 1 && a->w_mode != 2)) return B2DL_E_VALUE;
  const b2dl_act& x = a->x;
  const b2dl_act& y = a->y;
  if (x.n != y.n || x.h != y.h || x.w != y.w || y.c != a->cout || a->kh < 1 || a->kw < 1 || a->dilation < 1)
    return B2DL_E_VALUE;
  F32ConvParams p{};
  p.in = CF(x.ptr);
  p.n = x.n;
  p.h = x.h;
  p.w = x.w;
  p.k = x.c;
  p.in_stride = x.c_stride;
  p.wt = CF(a->w_master);
  p.mode = a->w_mode;
  p.kh = a->kh;
  p.kw = a->kw;
  p.dil = a->dilation;
  p.pad_top = a->pad_top;
  p.pad_left = a->pad_left;
  p.taps = a->kh * a->kw;
  // forward conv's HWIO extent: mode 1 [taps][x.c][cout]; mode 2 (dgrad) [taps][cout][x.c]
  p.wk = a->w_mode == 1 ? x.c : a->cout;
  p.wn = a->w_mode == 1 ? a->cout : x.c;
  p.out = F(y.ptr);
  p.nout = a->cout;
  p.out_stride = y.c_stride;
  p.bias = a->bias;
  p.res = CF(a->residual.ptr);
  p.res_stride = a->residual.c_stride;
  p.mask = CF(a->mask.ptr);
  p.mask_stride = a->mask.c_stride;
  p.relu = a->relu;
  p.accumulate = a->accumulate;
  const long long npix = static_cast<long long>(x.n) * x.h * x.w;
  dim3 grid(static_cast<unsigned>((npix + F_BM - 1) / F_BM), static_cast<unsigned>(cdiv(a->cout, F_BN)));
  k_conv_f32<<<grid, F_THREADS, 0, as_stream(stream)>>>(p);
  return check_launch();
}

namespace b2 {
static void f32_wgrad_plan(const b2dl_wgrad_args* a, int* splits, long long* per) {
  const long long npix = static_cast<long long>(a->x.n) * a->x.h * a->x.w;
  const long long tiles = static_cast<long long>(cdiv(a->x.c, F_BM)) * cdiv(a->dy.c, F_BN) * a->kh * a->kw;
  long long s = std::max<long long>(1, (4LL * num_sms() + tiles - 1) / tiles);
  s = std::min<long long>(s, std::max<long long>(1, npix / (4 * F_BK)));
  *per = ((npix + s - 1) / s + F_BK - 1) / F_BK * F_BK;
  *splits = static_cast<int>((npix + *per - 1) / *per);
}
}  // namespace b2

extern "C" size_t b2dl_f32_wgrad_workspace_size(const b2dl_wgrad_args* a) {
  if (!a) return 0;
  int splits;
  long long per;
  f32_wgrad_plan(a, &splits, &per);
  const size_t wbytes = static_cast<size_t>(splits) * a->kh * a->kw * a->x.c * a->dy.c * sizeof(float);
  return align_up(wbytes, 256) + align_up(static_cast<size_t>(splits) * a->dy.c * sizeof(float), 256);
}

extern "C" int b2dl_f32_conv_wgrad(const b2dl_wgrad_args* a, void* stream) {
  if (!a || !a->x.ptr || !a->dy.ptr || !a->dw || a->window) return B2DL_E_VALUE;
  const b2dl_act& x = a->x;
  const b2dl_act& dy = a->dy;
  if (x.n != dy.n || x.h != dy.h || x.w != dy.w) return B2DL_E_VALUE;
  const size_t need = b2dl_f32_wgrad_workspace_size(a);
  if (!a->workspace || a->workspace_bytes < need) return B2DL_E_VALUE;
  F32WgradParams p{};
  p.x = CF(x.ptr);
  p.n = x.n;
  p.h = x.h;
  p.w = x.w;
  p.cin = x.c;
  p.x_stride = x.c_stride;
  p.dy = CF(dy.ptr);
  p.cout = dy.c;
  p.dy_stride = dy.c_stride;
  p.kw = a->kw;
  p.dil = a->dilation;
  p.pad_top = a->pad_top;
  p.pad_left = a->pad_left;
  p.taps = a->kh * a->kw;
  f32_wgrad_plan(a, &p.splits, &p.per_split);
  const size_t wbytes = static_cast<size_t>(p.splits) * p.taps * p.cin * p.cout * sizeof(float);
  p.part = F(a->workspace);
  p.bpart = a->bias_grad ? reinterpret_cast<float*>(reinterpret_cast<char*>(a->workspace) + align_up(wbytes, 256))
                         : nullptr;
  cudaStream_t st = as_stream(stream);
  dim3 grid(cdiv(p.cin, F_BM), cdiv(p.cout, F_BN), p.taps * p.splits);
  k_wgrad_f32<<<grid, F_THREADS, 0, st>>>(p);
  int rc = check_launch();
  if (rc) return rc;
  const long long total = static_cast<long long>(p.taps) * p.cin * p.cout;
  k_reduce_f32<<<grid_f32(total), 256, 0, st>>>(p.part, total, p.splits, a->dw, a->accumulate);
  rc = check_launch();
  if (rc || !a->bias_grad) return rc;
  k_reduce_f32<<<grid_f32(p.cout), 256, 0, st>>>(p.bpart, p.cout, p.splits, a->bias_grad, a->accumulate);
  return check_launch();
}

extern "C" int b2dl_f32_avgpool_fwd(b2dl_act x, b2dl_act y, int k, void* stream) {
  if (k < 1 || x.h % k || x.w % k || y.h != x.h / k || y.w != x.w / k || y.c != x.c || y.n != x.n) return B2DL_E_VALUE;
  const long long total = static_cast<long long>(y.n) * y.h * y.w * y.c;
  k_avgpool_fwd_f32<<<grid_f32(total), 256, 0, as_stream(stream)>>>(CF(x.ptr), x.c_stride, F(y.ptr), y.c_stride, y.n,
                                                                      y.h, y.w, y.c, k);
  return check_launch();
}
extern "C" int b2dl_f32_avgpool_bwd(b2dl_act dy, b2dl_act dx, int k, int accumulate, b2dl_act mask, void* stream) {
  if (k < 1 || dx.h != dy.h * k || dx.w != dy.w * k || dy.c != dx.c) return B2DL_E_VALUE;
  const long long total = static_cast<long long>(dx.n) * dx.h * dx.w * dx.c;
  k_avgpool_bwd_f32<<<grid_f32(total), 256, 0, as_stream(stream)>>>(CF(dy.ptr), dy.c_stride, F(dx.ptr), dx.c_stride,
                                                                      CF(mask.ptr), mask.c_stride, dy.n, dy.h, dy.w,
                                                                      dy.c, k, accumulate);
  return check_launch();
}
extern "C" int b2dl_f32_upsample_fwd(b2dl_act x, b2dl_act y, int f, void* stream) {
  if (f < 1 || y.h != x.h * f || y.w != x.w * f || y.c != x.c) return B2DL_E_VALUE;
  const long long total = static_cast<long long>(y.n) * y.h * y.w * y.c;
  k_upsample_fwd_f32<<<grid_f32(total), 256, 0, as_stream(stream)>>>(CF(x.ptr), x.c_stride, F(y.ptr), y.c_stride,
                                                                       x.n, x.h, x.w, x.c, f);
  return check_launch();
}
extern "C" int b2dl_f32_upsample_bwd(b2dl_act dy, b2dl_act dx, int f, int accumulate, b2dl_act mask, void* stream) {
  if (f < 1 || dy.h != dx.h * f || dy.w != dx.w * f || dy.c != dx.c) return B2DL_E_VALUE;
  const long long total = static_cast<long long>(dx.n) * dx.h * dx.w * dx.c;
  k_upsample_bwd_f32<<<grid_f32(total), 256, 0, as_stream(stream)>>>(CF(dy.ptr), dy.c_stride, F(dx.ptr), dx.c_stride,
                                                                       CF(mask.ptr), mask.c_stride, dx.n, dx.h, dx.w,
                                                                       dx.c, f, accumulate);
  return check_launch();
}
extern "C" int b2dl_f32_add(b2dl_act x, b2dl_act y, int accumulate, b2dl_act mask, void* stream) {
  if (x.n != y.n || x.h != y.h || x.w != y.w || x.c != y.c) return B2DL_E_VALUE;
  const long long npix = static_cast<long long>(x.n) * x.h * x.w;
  k_add_f32<<<grid_f32(npix * x.c), 256, 0, as_stream(stream)>>>(CF(x.ptr), x.c_stride, F(y.ptr), y.c_stride,
                                                                  CF(mask.ptr), mask.c_stride, npix, x.c, accumulate);
  return check_launch();
}
