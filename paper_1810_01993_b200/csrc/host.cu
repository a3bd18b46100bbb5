// Host helpers (device query, TMA descriptor encoding) and the reference-shaped
// NCHW fp32 entry points of include/b2dl.h group (1).
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "internal.h"

namespace b2 {

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int encode_tiled(CUtensorMap* m, CUtensorMapDataType dt, int rank, void* ptr, const uint64_t* dims,
                 const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle sw,
                 const uint32_t* elem_strides) {
  auto fn = encode_fn();
  if (!fn) return B2DL_E_CUDA;
  cuuint64_t d[5];
  cuuint64_t s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = elem_strides ? elem_strides[i] : 1;
    if (i + 1 < rank) s[i] = strides_bytes[i];
  }
  CUresult r = fn(m, dt, rank, ptr, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? B2DL_OK : B2DL_E_ALIGN;
}

int act_map(CUtensorMap* m, const b2dl_act& a, int box_c, int box_w, int box_h, CUtensorMapSwizzle sw) {
  const uint64_t cs = static_cast<uint64_t>(a.c_stride) * 2;
  const uint64_t dims[4] = {static_cast<uint64_t>(a.c), static_cast<uint64_t>(a.w), static_cast<uint64_t>(a.h),
                            static_cast<uint64_t>(a.n)};
  const uint64_t strides[3] = {cs, cs * a.w, cs * a.w * a.h};
  const uint32_t box[4] = {static_cast<uint32_t>(box_c), static_cast<uint32_t>(box_w), static_cast<uint32_t>(box_h),
                           1u};
  return encode_tiled(m, B2H_TMA, 4, a.ptr, dims, strides, box, sw);
}

// Strided traversal: a box of bw x bh pixels taken every `stride` pixels in W and H (the TMA
// box spans bw*stride x bh*stride input pixels; elementStrides select every stride-th one).
int act_map_strided(CUtensorMap* m, const b2dl_act& a, int box_c, int box_w, int box_h, int stride,
                    CUtensorMapSwizzle sw) {
  const uint64_t cs = static_cast<uint64_t>(a.c_stride) * 2;
  const uint64_t dims[4] = {static_cast<uint64_t>(a.c), static_cast<uint64_t>(a.w), static_cast<uint64_t>(a.h),
                            static_cast<uint64_t>(a.n)};
  const uint64_t strides[3] = {cs, cs * a.w, cs * a.w * a.h};
  const uint32_t box[4] = {static_cast<uint32_t>(box_c), static_cast<uint32_t>(box_w * stride),
                           static_cast<uint32_t>(box_h * stride), 1u};
  const uint32_t es[4] = {1u, static_cast<uint32_t>(stride), static_cast<uint32_t>(stride), 1u};
  return encode_tiled(m, B2H_TMA, 4, a.ptr, dims, strides, box, sw, es);
}

// Phase view of a full-resolution NHWC tensor: pixel (i, j) of the (h/f, w/f) view is pixel
// (f*i + ph, f*j + pw) -- plain strides of f pixels / f rows from a shifted base.
int act_map_phase(CUtensorMap* m, const b2dl_act& a, int f, int ph, int pw, int box_c, int box_w, int box_h,
                  CUtensorMapSwizzle sw) {
  const uint64_t cs = static_cast<uint64_t>(a.c_stride) * 2;
  const uint64_t dims[4] = {static_cast<uint64_t>(a.c), static_cast<uint64_t>(a.w / f),
                            static_cast<uint64_t>(a.h / f), static_cast<uint64_t>(a.n)};
  const uint64_t strides[3] = {cs * f, cs * a.w * f, cs * a.w * a.h};
  const uint32_t box[4] = {static_cast<uint32_t>(box_c), static_cast<uint32_t>(box_w), static_cast<uint32_t>(box_h),
                           1u};
  char* base = static_cast<char*>(a.ptr) + (static_cast<uint64_t>(ph) * a.w + pw) * cs;
  return encode_tiled(m, B2H_TMA, 4, base, dims, strides, box, sw);
}

// Row-window view of a haloed NHWC image (conv window mode): virtual pixel (y, xx) holds the
// c_v contiguous values x[y][xx..][..] starting at pixel xx, so neighbouring virtual pixels
// overlap in memory (pixel stride < inner extent); TMA zero-fills virtual channels >= c_v.
int window_map(CUtensorMap* m, const b2dl_act& x, int c_v, int w_v, int box_c, int box_w, int box_h,
               CUtensorMapSwizzle sw) {
  const uint64_t ps = static_cast<uint64_t>(x.c_stride) * 2;
  const uint64_t dims[4] = {static_cast<uint64_t>(c_v), static_cast<uint64_t>(w_v), static_cast<uint64_t>(x.h),
                            static_cast<uint64_t>(x.n)};
  const uint64_t strides[3] = {ps, ps * x.w, ps * x.w * x.h};
  const uint32_t box[4] = {static_cast<uint32_t>(box_c), static_cast<uint32_t>(box_w), static_cast<uint32_t>(box_h),
                           1u};
  return encode_tiled(m, B2H_TMA, 4, x.ptr, dims, strides, box, sw);
}

// 5-D map (64-channel inner, W, H, N, channel block): one box = g chunks of [pixels][64 ch],
// stored chunk-major in shared memory (the MN-major operand's LBO-separated chunks)
int act_map5(CUtensorMap* m, const b2dl_act& a, int box_w, int box_h, int g) {
  const uint64_t cs = static_cast<uint64_t>(a.c_stride) * 2;
  const uint64_t dims[5] = {64u, static_cast<uint64_t>(a.w), static_cast<uint64_t>(a.h), static_cast<uint64_t>(a.n),
                            static_cast<uint64_t>(a.c / 64)};
  const uint64_t strides[4] = {cs, cs * a.w, cs * a.w * a.h, 128u};
  const uint32_t box[5] = {64u, static_cast<uint32_t>(box_w), static_cast<uint32_t>(box_h), 1u,
                           static_cast<uint32_t>(g)};
  return encode_tiled(m, B2H_TMA, 5, a.ptr, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

// -------------------------------------------------------------- layout kernels
// OIHW fp32 -> fprop packed bf16 [cout][taps][cin_pad]  (zero padded)
__global__ void pack_oihw_fprop(const float* __restrict__ w, b2h* __restrict__ out, int cout, int cin,
                                int taps, int cin_pad) {
  long long total = static_cast<long long>(cout) * taps * cin_pad;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int ci = static_cast<int>(i % cin_pad);
    long long r = i / cin_pad;
    int t = static_cast<int>(r % taps);
    int co = static_cast<int>(r / taps);
    float v = ci < cin ? w[(static_cast<long long>(co) * cin + ci) * taps + t] : 0.f;
    out[i] = f_to_h(v);
  }
}
// OIHW fp32 -> dgrad packed bf16 [cin][taps flipped][cout_pad]
__global__ void pack_oihw_dgrad(const float* __restrict__ w, b2h* __restrict__ out, int cout, int cin,
                                int taps, int cout_pad) {
  long long total = static_cast<long long>(cin) * taps * cout_pad;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int co = static_cast<int>(i % cout_pad);
    long long r = i / cout_pad;
    int tf = static_cast<int>(r % taps);
    int ci = static_cast<int>(r / taps);
    int t = taps - 1 - tf;  // 180-degree rotation of the kernel window
    float v = co < cout ? w[(static_cast<long long>(co) * cin + ci) * taps + t] : 0.f;
    out[i] = f_to_h(v);
  }
}
// HWIO fp32 -> OIHW fp32
__global__ void hwio_to_oihw(const float* __restrict__ w, float* __restrict__ out, int cout, int cin, int taps) {
  long long total = static_cast<long long>(cout) * cin * taps;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int t = static_cast<int>(i % taps);
    long long r = i / taps;
    int ci = static_cast<int>(r % cin);
    int co = static_cast<int>(r / cin);
    out[i] = w[(static_cast<long long>(t) * cin + ci) * cout + co];
  }
}

static int grid_for(long long total) {
  return static_cast<int>(std::max<long long>(1, std::min<long long>((total + 255) / 256, 8LL * num_sms())));
}

}  // namespace b2

using namespace b2;

namespace {
struct RefWs {
  char* base;
  size_t off = 0;
  size_t cap;
  void* take(size_t bytes) {
    off = align_up(off, 256);
    if (off + bytes > cap) return nullptr;
    void* p = base + off;
    off += bytes;
    return p;
  }
};
int same_pad_before(int k, int d) { return ((k - 1) * d) / 2; }
int same_pad_after(int k, int d) { return (k - 1) * d - same_pad_before(k, d); }
b2dl_act nhwc(void* p, int n, int h, int w, int c) {
  b2dl_act a;
  a.ptr = p;
  a.n = n;
  a.h = h;
  a.w = w;
  a.c = c;
  a.c_stride = round_up(c, 8);
  return a;
}
size_t act_bytes(int n, int h, int w, int c, int eb) {
  return static_cast<size_t>(n) * h * w * round_up(c, 8) * eb;
}
}  // namespace

extern "C" size_t b2dl_conv2d_workspace_size(int n, int cin, int h, int w, int cout, int kh, int kw) {
  const int taps = kh * kw;
  size_t s = 0;
  s += act_bytes(n, h, w, cin, 2) + 256;                                              // x nhwc bf16
  s += act_bytes(n, h, w, cout, 2) + 256;                                             // dy nhwc bf16
  s += act_bytes(n, h, w, std::max(cin, cout), 4) + 256;                              // fp32 nhwc result
  s += static_cast<size_t>(cout) * taps * b2dl_cin_pad(cin) * 2 + 256;                // fprop packed
  s += static_cast<size_t>(cin) * taps * b2dl_cin_pad(cout) * 2 + 256;                // dgrad packed
  s += static_cast<size_t>(cout) * taps * cin * 4 + 256;                              // hwio dw
  // wgrad split-K partials: exactly what the wgrad planner will ask for
  b2dl_wgrad_args wa{};
  wa.x = nhwc(nullptr, n, h, w, cin);
  wa.dy = nhwc(nullptr, n, h, w, cout);
  wa.kh = kh;
  wa.kw = kw;
  wa.dilation = 1;
  s += b2dl_wgrad_workspace_size(&wa) + 4096;
  return s;
}

extern "C" int b2dl_conv2d_forward(const float* x, const float* w, float* y, int n, int cin, int h, int wd,
                                   int cout, int kh, int kw, int stride, int dilation, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  if (stride != 1) return B2DL_E_NOT_IMPLEMENTED;
  if (n < 1 || cin < 1 || h < 1 || wd < 1 || cout < 1 || kh < 1 || kw < 1 || dilation < 1) return B2DL_E_VALUE;
  cudaStream_t st = as_stream(stream);
  RefWs ws{reinterpret_cast<char*>(workspace), 0, workspace_bytes};
  const int taps = kh * kw;
  void* xb = ws.take(act_bytes(n, h, wd, cin, 2));
  void* yf = ws.take(act_bytes(n, h, wd, cout, 4));
  void* wp = ws.take(static_cast<size_t>(cout) * taps * b2dl_cin_pad(cin) * 2);
  if (!xb || !yf || !wp) return B2DL_E_VALUE;
  b2dl_act xa = nhwc(xb, n, h, wd, cin);
  int rc = b2dl_nchw_to_nhwc(x, xa, 0, stream);
  if (rc) return rc;
  long long tot = static_cast<long long>(cout) * taps * b2dl_cin_pad(cin);
  pack_oihw_fprop<<<grid_for(tot), 256, 0, st>>>(w, reinterpret_cast<b2h*>(wp), cout, cin, taps,
                                                 b2dl_cin_pad(cin));
  if ((rc = check_launch())) return rc;
  b2dl_conv_args a{};
  a.x = xa;
  a.w_packed = wp;
  a.cout = cout;
  a.kh = kh;
  a.kw = kw;
  a.dilation = dilation;
  a.pad_top = same_pad_before(kh, dilation);
  a.pad_left = same_pad_before(kw, dilation);
  a.y = nhwc(yf, n, h, wd, cout);
  a.y_f32 = 1;
  if ((rc = b2dl_conv_fprop(&a, stream))) return rc;
  return b2dl_nhwc_to_nchw(a.y, 1, y, stream);
}

extern "C" int b2dl_conv2d_backward_input(const float* dy, const float* w, float* dx, int n, int cin, int h, int wd,
                                          int cout, int kh, int kw, int stride, int dilation, void* workspace,
                                          size_t workspace_bytes, void* stream) {
  if (stride != 1) return B2DL_E_NOT_IMPLEMENTED;
  if (n < 1 || cin < 1 || h < 1 || wd < 1 || cout < 1 || kh < 1 || kw < 1 || dilation < 1) return B2DL_E_VALUE;
  cudaStream_t st = as_stream(stream);
  RefWs ws{reinterpret_cast<char*>(workspace), 0, workspace_bytes};
  const int taps = kh * kw;
  void* dyb = ws.take(act_bytes(n, h, wd, cout, 2));
  void* dxf = ws.take(act_bytes(n, h, wd, cin, 4));
  void* wp = ws.take(static_cast<size_t>(cin) * taps * b2dl_cin_pad(cout) * 2);
  if (!dyb || !dxf || !wp) return B2DL_E_VALUE;
  b2dl_act dya = nhwc(dyb, n, h, wd, cout);
  int rc = b2dl_nchw_to_nhwc(dy, dya, 0, stream);
  if (rc) return rc;
  long long tot = static_cast<long long>(cin) * taps * b2dl_cin_pad(cout);
  pack_oihw_dgrad<<<grid_for(tot), 256, 0, st>>>(w, reinterpret_cast<b2h*>(wp), cout, cin, taps,
                                                 b2dl_cin_pad(cout));
  if ((rc = check_launch())) return rc;
  b2dl_conv_args a{};
  a.x = dya;
  a.w_packed = wp;
  a.cout = cin;
  a.kh = kh;
  a.kw = kw;
  a.dilation = dilation;
  // gather form of the reference's scatter (pyx:35-51): flipped taps, "after" pads lead
  a.pad_top = same_pad_after(kh, dilation);
  a.pad_left = same_pad_after(kw, dilation);
  a.y = nhwc(dxf, n, h, wd, cin);
  a.y_f32 = 1;
  if ((rc = b2dl_conv_fprop(&a, stream))) return rc;
  return b2dl_nhwc_to_nchw(a.y, 1, dx, stream);
}

extern "C" int b2dl_conv2d_backward_weights(const float* x, const float* dy, float* dw, int n, int cin, int h,
                                            int wd, int cout, int kh, int kw, int dilation, void* workspace,
                                            size_t workspace_bytes, void* stream) {
  if (n < 1 || cin < 1 || h < 1 || wd < 1 || cout < 1 || kh < 1 || kw < 1 || dilation < 1) return B2DL_E_VALUE;
  cudaStream_t st = as_stream(stream);
  RefWs ws{reinterpret_cast<char*>(workspace), 0, workspace_bytes};
  const int taps = kh * kw;
  void* xb = ws.take(act_bytes(n, h, wd, cin, 2));
  void* dyb = ws.take(act_bytes(n, h, wd, cout, 2));
  float* hw = reinterpret_cast<float*>(ws.take(static_cast<size_t>(cout) * taps * cin * 4));
  if (!xb || !dyb || !hw) return B2DL_E_VALUE;
  b2dl_act xa = nhwc(xb, n, h, wd, cin);
  b2dl_act dya = nhwc(dyb, n, h, wd, cout);
  int rc = b2dl_nchw_to_nhwc(x, xa, 0, stream);
  if (rc) return rc;
  if ((rc = b2dl_nchw_to_nhwc(dy, dya, 0, stream))) return rc;
  b2dl_wgrad_args a{};
  a.x = xa;
  a.dy = dya;
  a.kh = kh;
  a.kw = kw;
  a.dilation = dilation;
  a.pad_top = same_pad_before(kh, dilation);
  a.pad_left = same_pad_before(kw, dilation);
  a.dw = hw;
  ws.off = align_up(ws.off, 256);
  a.workspace = reinterpret_cast<char*>(workspace) + ws.off;
  a.workspace_bytes = workspace_bytes - ws.off;
  if ((rc = b2dl_conv_wgrad(&a, stream))) return rc;
  long long tot = static_cast<long long>(cout) * cin * taps;
  hwio_to_oihw<<<grid_for(tot), 256, 0, st>>>(hw, dw, cout, cin, taps);
  return check_launch();
}

extern "C" const char* b2dl_version(void) { return "b2dl 0.1 sm_100a tcgen05"; }
