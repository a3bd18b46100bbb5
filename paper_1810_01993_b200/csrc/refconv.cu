// Reference-precision convolution core: the drop-in for the reference's compiled conv kernels
// (pkg/src/deskdl/model/_convkernels.pyx:16-71 behind _kernels_cy.py:13-44) at the reference's
// own arithmetic type.  The Cython core is a fused-type (float32 / float64) direct loop over
// NCHW tensors; these kernels take the same NCHW tensors in the same two types and compute
// in that type (fp64 DFMA for float64, fp32 FFMA for float32), so the reference's kernel tests
// -- fp64 loop-oracle agreement to 1e-12, finite-difference gradients to 1e-7, fp32 backend
// agreement to 1e-5 (pkg/tests/test_kernels.py:28-82) -- hold for this backend too.  The bf16
// tensor-core variants (host.cu, b2dl_conv2d_forward & co.) are the training-step arithmetic.
//
// One tiled GEMM kernel, three index maps (same "same" padding, TF split, _kernels_py.py:18-21):
//   forward  y[b,co,p]      = sum_{ci,tap} w[co,ci,tap] x[b,ci,p+off(tap)]       M=pixels N=cout K=cin*taps
//   dgrad    dx[b,ci,q]     = sum_{co,tap} w[co,ci,tap] dy[b,co,q-off(tap)]      M=pixels N=cin  K=cout*taps
//   wgrad    dw[co,ci,tap]  = sum_{b,p} dy[b,co,p] x[b,ci,p+off(tap)]           M=cout N=cin*taps K=pixels
// off(i,j) = (i*d - pad_top, j*d - pad_left).  The gather form of dgrad replaces the reference's
// scatter into a padded buffer (pyx:35-51).  wgrad sums its K (all pixels) inside one CTA in a
// fixed order: deterministic, no workspace, no atomics.
#include <algorithm>

#include "internal.h"

namespace b2 {
namespace {

constexpr int R_BM = 64, R_BN = 64, R_BK = 16, R_THREADS = 256;

struct RefConvP {
  const void* x;   // fwd / wgrad input  [n][cin][h][w]
  const void* w;   // fwd / dgrad weight [cout][cin][kh][kw]
  const void* dy;  // dgrad / wgrad      [n][cout][h][w]
  void* out;
  int n, cin, h, wd, cout, kh, kw, dil, pt, pl;
};

template <typename T, int OP>
struct Maps {
  // GEMM extents
  static __device__ long long M(const RefConvP& p) {
    return OP == 2 ? p.cout : static_cast<long long>(p.n) * p.h * p.wd;
  }
  static __device__ long long N(const RefConvP& p) {
    return OP == 0 ? p.cout : OP == 1 ? p.cin : static_cast<long long>(p.cin) * p.kh * p.kw;
  }
  static __device__ long long K(const RefConvP& p) {
    const int taps = p.kh * p.kw;
    return OP == 0 ? static_cast<long long>(p.cin) * taps
                   : OP == 1 ? static_cast<long long>(p.cout) * taps : static_cast<long long>(p.n) * p.h * p.wd;
  }
  // element of the (shifted) activation operand: channel c of image b at (y, x) + tap offset
  static __device__ T act(const T* base, int chans, const RefConvP& p, int b, int c, int y, int x) {
    if (y < 0 || y >= p.h || x < 0 || x >= p.wd) return T(0);
    return base[((static_cast<long long>(b) * chans + c) * p.h + y) * p.wd + x];
  }
  static __device__ T A(const RefConvP& p, long long m, long long k) {
    const int taps = p.kh * p.kw;
    if (OP == 2) {  // dy[b, co=m, pixel k]
      const long long hw = static_cast<long long>(p.h) * p.wd;
      const int b = static_cast<int>(k / hw);
      const long long r = k - b * hw;
      return static_cast<const T*>(p.dy)[(static_cast<long long>(b) * p.cout + m) * hw + r];
    }
    const long long hw = static_cast<long long>(p.h) * p.wd;
    const int b = static_cast<int>(m / hw);
    const int r = static_cast<int>(m - b * hw);
    const int y = r / p.wd, x = r - (r / p.wd) * p.wd;
    const int c = static_cast<int>(k / taps), tap = static_cast<int>(k - static_cast<long long>(c) * taps);
    const int i = tap / p.kw, j = tap - i * p.kw;
    if (OP == 0)
      return act(static_cast<const T*>(p.x), p.cin, p, b, c, y + i * p.dil - p.pt, x + j * p.dil - p.pl);
    return act(static_cast<const T*>(p.dy), p.cout, p, b, c, y - i * p.dil + p.pt, x - j * p.dil + p.pl);
  }
  static __device__ T B(const RefConvP& p, long long k, long long nn) {
    const int taps = p.kh * p.kw;
    const T* w = static_cast<const T*>(p.w);
    if (OP == 0) return w[nn * K(p) + k];  // w[co=nn][k=(ci,tap)]
    if (OP == 1) {                         // k = (co, tap), nn = ci
      const long long co = k / taps, tap = k - co * taps;
      return w[(co * p.cin + nn) * taps + tap];
    }
    // OP 2: k = pixel, nn = (ci, tap)
    const long long hw = static_cast<long long>(p.h) * p.wd;
    const int b = static_cast<int>(k / hw);
    const int r = static_cast<int>(k - b * hw);
    const int y = r / p.wd, x = r - (r / p.wd) * p.wd;
    const int ci = static_cast<int>(nn / taps), tap = static_cast<int>(nn - static_cast<long long>(ci) * taps);
    const int i = tap / p.kw, j = tap - i * p.kw;
    return act(static_cast<const T*>(p.x), p.cin, p, b, ci, y + i * p.dil - p.pt, x + j * p.dil - p.pl);
  }
  static __device__ void store(const RefConvP& p, long long m, long long nn, T v) {
    T* o = static_cast<T*>(p.out);
    if (OP == 2) {  // dw[co=m][(ci,tap)=nn]
      o[m * N(p) + nn] = v;
      return;
    }
    const long long hw = static_cast<long long>(p.h) * p.wd;
    const long long b = m / hw, r = m - b * hw;
    const long long chans = N(p);
    o[(b * chans + nn) * hw + r] = v;
  }
};

template <typename T, int OP>
__global__ void __launch_bounds__(R_THREADS) k_refconv(const RefConvP p) {
  using Mp = Maps<T, OP>;
  __shared__ T As[R_BK][R_BM + 1];
  __shared__ T Bs[R_BK][R_BN + 1];
  const int t = threadIdx.x;
  const long long M = Mp::M(p), N = Mp::N(p), K = Mp::K(p);
  const long long m0 = static_cast<long long>(blockIdx.x) * R_BM;
  const long long n0 = static_cast<long long>(blockIdx.y) * R_BN;
  const int c_m = (t % 16) * 4, c_n = (t / 16) * 4;
  T acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = T(0);
  for (long long k0 = 0; k0 < K; k0 += R_BK) {
    // A tile: m fastest (pixels are contiguous in NCHW); B tile: n fastest
#pragma unroll
    for (int r = 0; r < (R_BK * R_BM) / R_THREADS; ++r) {
      const int e = t + r * R_THREADS;
      const int mm = e % R_BM, kk = e / R_BM;
      const long long m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < K) ? Mp::A(p, m, k) : T(0);
    }
#pragma unroll
    for (int r = 0; r < (R_BK * R_BN) / R_THREADS; ++r) {
      const int e = t + r * R_THREADS;
      const int nn = e % R_BN, kk = e / R_BN;
      const long long n = n0 + nn, k = k0 + kk;
      Bs[kk][nn] = (n < N && k < K) ? Mp::B(p, k, n) : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < R_BK; ++kk) {
      T a[4], b[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        a[e] = As[kk][c_m + e];
        b[e] = Bs[kk][c_n + e];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const long long m = m0 + c_m + u;
    if (m >= M) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const long long n = n0 + c_n + v;
      if (n < N) Mp::store(p, m, n, acc[u][v]);
    }
  }
}

template <typename T, int OP>
int launch(const RefConvP& p, cudaStream_t st) {
  const long long M = OP == 2 ? p.cout : static_cast<long long>(p.n) * p.h * p.wd;
  const long long N = OP == 0 ? p.cout : OP == 1 ? p.cin : static_cast<long long>(p.cin) * p.kh * p.kw;
  if (M == 0 || N == 0) return B2DL_OK;
  const dim3 grid(cdiv(M, R_BM), cdiv(N, R_BN));
  if (grid.y > 65535) return B2DL_E_VALUE;
  k_refconv<T, OP><<<grid, R_THREADS, 0, st>>>(p);
  return check_launch();
}

template <int OP>
int dispatch(int dtype, const RefConvP& p, cudaStream_t st) {
  if (dtype == B2DL_DTYPE_F32) return launch<float, OP>(p, st);
  if (dtype == B2DL_DTYPE_F64) return launch<double, OP>(p, st);
  return B2DL_E_VALUE;
}

RefConvP make(const void* x, const void* w, const void* dy, void* out, int n, int cin, int h, int wd, int cout,
              int kh, int kw, int dil) {
  RefConvP p{};
  p.x = x;
  p.w = w;
  p.dy = dy;
  p.out = out;
  p.n = n;
  p.cin = cin;
  p.h = h;
  p.wd = wd;
  p.cout = cout;
  p.kh = kh;
  p.kw = kw;
  p.dil = dil;
  p.pt = ((kh - 1) * dil) / 2;  // "same", TF split: before = total // 2 (_kernels_py.py:18-21)
  p.pl = ((kw - 1) * dil) / 2;
  return p;
}

bool bad_dims(int n, int cin, int h, int wd, int cout, int kh, int kw, int dil) {
  return n < 0 || cin < 1 || h < 0 || wd < 0 || cout < 1 || kh < 1 || kw < 1 || dil < 1;
}

}  // namespace
}  // namespace b2

using namespace b2;

extern "C" int b2dl_conv2d_forward_typed(int dtype, const void* x, const void* w, void* y, int n, int cin, int h,
                                         int wd, int cout, int kh, int kw, int stride, int dilation, void* stream) {
  if (stride != 1) return B2DL_E_NOT_IMPLEMENTED;
  if (bad_dims(n, cin, h, wd, cout, kh, kw, dilation)) return B2DL_E_VALUE;
  return dispatch<0>(dtype, make(x, w, nullptr, y, n, cin, h, wd, cout, kh, kw, dilation), as_stream(stream));
}

extern "C" int b2dl_conv2d_backward_input_typed(int dtype, const void* dy, const void* w, void* dx, int n, int cin,
                                                int h, int wd, int cout, int kh, int kw, int stride, int dilation,
                                                void* stream) {
  if (stride != 1) return B2DL_E_NOT_IMPLEMENTED;
  if (bad_dims(n, cin, h, wd, cout, kh, kw, dilation)) return B2DL_E_VALUE;
  return dispatch<1>(dtype, make(nullptr, w, dy, dx, n, cin, h, wd, cout, kh, kw, dilation), as_stream(stream));
}

extern "C" int b2dl_conv2d_backward_weights_typed(int dtype, const void* x, const void* dy, void* dw, int n, int cin,
                                                  int h, int wd, int cout, int kh, int kw, int dilation,
                                                  void* stream) {
  if (bad_dims(n, cin, h, wd, cout, kh, kw, dilation)) return B2DL_E_VALUE;
  return dispatch<2>(dtype, make(x, nullptr, dy, dw, n, cin, h, wd, cout, kh, kw, dilation), as_stream(stream));
}
