// Fused class-weighted softmax cross-entropy (pkg/src/deskdl/model/loss.py:47-93).
//
// Per sample n:  L_n = sum_p w[y_p] * (-log softmax(z_p)[y_p]) / sum_p w[y_p]
// loss = mean_n L_n,   dlogits_p = (softmax(z_p) - onehot(y_p)) * w[y_p] / (sum_p w[y_p] * N)
//
// The per-sample weight total only depends on the labels, so it comes from an
// exact integer class histogram (pass 1).  Pass 2 is one read of the logits and
// one write of dlogits / argmax per pixel; pass 3 folds the per-block partial
// sums in a fixed order (deterministic).
#include <cuda_bf16.h>

#include <algorithm>

#include "internal.h"

namespace b2 {

constexpr int WCE_MAX_CLASSES = 16;
constexpr int WCE_BLOCKS_PER_IMG = 64;

__global__ void k_wce_hist(const uint8_t* __restrict__ labels, long long hw, int classes, int* __restrict__ counts,
                           int* __restrict__ err) {
  __shared__ int h[WCE_MAX_CLASSES];
  const int img = blockIdx.y;
  if (threadIdx.x < WCE_MAX_CLASSES) h[threadIdx.x] = 0;
  __syncthreads();
  const uint8_t* lab = labels + img * hw;
  for (long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; p < hw;
       p += static_cast<long long>(gridDim.x) * blockDim.x) {
    int y = lab[p];
    if (y < classes)
      atomicAdd(&h[y], 1);
    else
      atomicExch(err, 1);
  }
  __syncthreads();
  if (threadIdx.x < classes && h[threadIdx.x]) atomicAdd(&counts[img * classes + threadIdx.x], h[threadIdx.x]);
}

__global__ void k_wce_main(const float* __restrict__ logits, int ls, const uint8_t* __restrict__ labels,
                           const float* __restrict__ cw, const int* __restrict__ counts, long long hw, int classes,
                           int nimg, void* __restrict__ dl, int ds, int dl_f32, uint8_t* __restrict__ pred,
                           double* __restrict__ part) {
  const int img = blockIdx.y;
  __shared__ float s_w[WCE_MAX_CLASSES];
  __shared__ float s_scale;
  __shared__ double red[32];
  if (threadIdx.x < classes) s_w[threadIdx.x] = cw[threadIdx.x];
  if (threadIdx.x == 0) {
    double ws = 0.0;
    for (int c = 0; c < classes; ++c) ws += static_cast<double>(counts[img * classes + c]) * cw[c];
    s_scale = static_cast<float>(1.0 / (ws * nimg));
  }
  __syncthreads();
  const float scale = s_scale;
  double acc = 0.0;
  const int zero_to = ds <= WCE_MAX_CLASSES ? ds : classes;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < hw;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long p = img * hw + q;
    const float* z = logits + p * ls;
    float zv[WCE_MAX_CLASSES];
    float mx = -INFINITY;
    int am = 0;
    for (int c = 0; c < classes; ++c) {
      zv[c] = z[c];
      if (zv[c] > mx) {  // strict: ties keep the lowest class index (np.argmax)
        mx = zv[c];
        am = c;
      }
    }
    float se = 0.f;
    for (int c = 0; c < classes; ++c) se += __expf(zv[c] - mx);
    const float lse = __logf(se);
    int y = labels[p];
    if (y >= classes) y = 0;  // flagged by the histogram pass
    const float wy = s_w[y];
    const float nll = lse - (zv[y] - mx);
    acc += static_cast<double>(wy) * nll;
    const float gs = wy * scale;
    for (int c = 0; c < zero_to; ++c) {
      float g = 0.f;
      if (c < classes) g = (__expf(zv[c] - mx - lse) - (c == y ? 1.f : 0.f)) * gs;
      if (dl_f32)
        reinterpret_cast<float*>(dl)[p * ds + c] = g;
      else
        reinterpret_cast<__nv_bfloat16*>(dl)[p * ds + c] = __float2bfloat16_rn(g);
    }
    if (pred) pred[p] = static_cast<uint8_t>(am);
  }
  // block reduction of the weighted nll (fp64, fixed order)
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += red[w];
    part[img * gridDim.x + blockIdx.x] = s;
  }
}

__global__ void k_wce_final(const double* __restrict__ part, int nb, const int* __restrict__ counts,
                            const float* __restrict__ cw, int classes, int nimg, float* __restrict__ loss) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double total = 0.0;
  for (int n = 0; n < nimg; ++n) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[n * nb + b];
    double ws = 0.0;
    for (int c = 0; c < classes; ++c) ws += static_cast<double>(counts[n * classes + c]) * cw[c];
    total += s / ws;
  }
  loss[0] = static_cast<float>(total / nimg);
}

}  // namespace b2

using namespace b2;

extern "C" size_t b2dl_wce_workspace_size(int n, int h, int w, int classes) {
  (void)h;
  (void)w;
  (void)classes;
  return static_cast<size_t>(n) * WCE_BLOCKS_PER_IMG * sizeof(double) + 256 + 64;
}

extern "C" int b2dl_wce(b2dl_act logits, const uint8_t* labels, const float* class_weights, int classes,
                        float* loss_out, int* counts, b2dl_act dlogits, int dlogits_f32, uint8_t* pred,
                        void* workspace, size_t workspace_bytes, void* stream) {
  if (classes < 2 || classes > WCE_MAX_CLASSES || logits.c != classes || dlogits.c != classes) return B2DL_E_VALUE;
  if (!logits.ptr || !labels || !class_weights || !loss_out || !counts || !dlogits.ptr) return B2DL_E_VALUE;
  if (workspace_bytes < b2dl_wce_workspace_size(logits.n, logits.h, logits.w, classes)) return B2DL_E_VALUE;
  cudaStream_t st = as_stream(stream);
  const long long hw = static_cast<long long>(logits.h) * logits.w;
  double* part = reinterpret_cast<double*>(workspace);
  int* err = reinterpret_cast<int*>(reinterpret_cast<char*>(workspace) +
                                    align_up(static_cast<size_t>(logits.n) * WCE_BLOCKS_PER_IMG * sizeof(double), 256));
  cudaMemsetAsync(counts, 0, sizeof(int) * logits.n * classes, st);
  cudaMemsetAsync(err, 0, sizeof(int), st);
  dim3 grid(WCE_BLOCKS_PER_IMG, logits.n);
  k_wce_hist<<<grid, 256, 0, st>>>(labels, hw, classes, counts, err);
  k_wce_main<<<grid, 256, 0, st>>>(reinterpret_cast<const float*>(logits.ptr), logits.c_stride, labels, class_weights,
                                   counts, hw, classes, logits.n, dlogits.ptr, dlogits.c_stride, dlogits_f32,
                                   pred, part);
  k_wce_final<<<1, 32, 0, st>>>(part, WCE_BLOCKS_PER_IMG, counts, class_weights, classes, logits.n, loss_out);
  return check_launch();
}
