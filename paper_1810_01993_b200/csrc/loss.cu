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
constexpr int WCE_THREADS = 256;
constexpr int WCE_TARGET_BLOCKS = 148 * 4;  // 4 resident 8-warp CTAs on each of the 148 SMs

// Blocks per sample: fill the GPU (the step has n = 2 samples of 0.88 M pixels; 64 blocks per
// sample left 20 SMs idle and 8 warps per busy SM, latency-bound at 8 % of HBM).
static inline int wce_blocks_per_img(int n, long long hw) {
  const long long want = (WCE_TARGET_BLOCKS + n - 1) / n;
  const long long cap = (hw + WCE_THREADS - 1) / WCE_THREADS;
  return static_cast<int>(std::max(1LL, std::min(want, cap)));
}

__global__ void k_wce_hist(const uint8_t* __restrict__ labels, long long hw, int classes, int* __restrict__ counts,
                           int* __restrict__ err) {
  __shared__ int h[WCE_MAX_CLASSES];
  const int img = blockIdx.y;
  if (threadIdx.x < WCE_MAX_CLASSES) h[threadIdx.x] = 0;
  __syncthreads();
  const uint8_t* lab = labels + img * hw;
  // per-warp class counts from ballots (no shared-memory atomics in the loop: 3 classes made
  // every pixel a same-address atomic); the trip count is warp-uniform so all lanes vote.
  int cnt[WCE_MAX_CLASSES];
#pragma unroll
  for (int c = 0; c < WCE_MAX_CLASSES; ++c) cnt[c] = 0;
  bool bad = false;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long base = blockIdx.x * static_cast<long long>(blockDim.x) + (threadIdx.x & ~31);
  for (long long p0 = base; p0 < hw; p0 += stride) {
    const long long p = p0 + (threadIdx.x & 31);
    const int y = p < hw ? lab[p] : -1;
    bad |= y >= classes;
#pragma unroll
    for (int c = 0; c < WCE_MAX_CLASSES; ++c)
      if (c < classes) cnt[c] += __popc(__ballot_sync(0xffffffffu, y == c));
  }
  if (bad) atomicExch(err, 1);
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int c = 0; c < WCE_MAX_CLASSES; ++c)
      if (c < classes && cnt[c]) atomicAdd(&h[c], cnt[c]);
  }
  __syncthreads();
  if (threadIdx.x < classes && h[threadIdx.x]) atomicAdd(&counts[img * classes + threadIdx.x], h[threadIdx.x]);
}

__global__ void k_wce_main(const float* __restrict__ logits, int ls, const uint8_t* __restrict__ labels,
                           const float* __restrict__ cw, const int* __restrict__ counts, long long hw, int classes,
                           int nimg, void* __restrict__ dl, int ds, int dl_f32, float dl_scale,
                           uint8_t* __restrict__ pred, double* __restrict__ part) {
  const int img = blockIdx.y;
  __shared__ float s_w[WCE_MAX_CLASSES];
  __shared__ float s_scale;
  __shared__ double red[32];
  if (threadIdx.x < classes) s_w[threadIdx.x] = cw[threadIdx.x];
  if (threadIdx.x == 0) {
    double ws = 0.0;
    for (int c = 0; c < classes; ++c) ws += static_cast<double>(counts[img * classes + c]) * cw[c];
    s_scale = static_cast<float>(dl_scale / (ws * nimg));   // dl_scale: the fp16 build's loss scale
  }
  __syncthreads();
  const float scale = s_scale;
  double acc = 0.0;
  const int zero_to = ds <= WCE_MAX_CLASSES ? ds : classes;
  const bool vec8 = !dl_f32 && ds == 8 && classes <= 8 && (reinterpret_cast<uintptr_t>(dl) & 15) == 0;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < hw;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long p = img * hw + q;
    const float* z = logits + p * ls;
    // fully unrolled, class-guarded loops keep zv in registers (no dynamic indexing)
    float zv[WCE_MAX_CLASSES];
    float mx = -INFINITY;
    int am = 0;
#pragma unroll
    for (int c = 0; c < WCE_MAX_CLASSES; ++c) {
      zv[c] = c < classes ? z[c] : -INFINITY;
      if (zv[c] > mx) {  // strict: ties keep the lowest class index (np.argmax)
        mx = zv[c];
        am = c;
      }
    }
    float se = 0.f;
#pragma unroll
    for (int c = 0; c < WCE_MAX_CLASSES; ++c)
      if (c < classes) se += __expf(zv[c] - mx);
    const float lse = __logf(se);
    int y = labels[p];
    if (y >= classes) y = 0;  // flagged by the histogram pass
    const float wy = s_w[y];
    float zy = 0.f;
#pragma unroll
    for (int c = 0; c < WCE_MAX_CLASSES; ++c)
      if (c == y) zy = zv[c];
    const float nll = lse - (zy - mx);
    acc += static_cast<double>(wy) * nll;
    const float gs = wy * scale;
    if (vec8) {  // bf16 dlogits padded to 8 channels: one 16-byte store per pixel
      __align__(16) b2h g8[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float g = 0.f;
        if (c < classes) g = (__expf(zv[c] - mx - lse) - (c == y ? 1.f : 0.f)) * gs;
        g8[c] = f_to_h(g);
      }
      reinterpret_cast<uint4*>(dl)[p] = *reinterpret_cast<const uint4*>(g8);
    } else {
#pragma unroll
      for (int c = 0; c < WCE_MAX_CLASSES; ++c) {
        if (c >= zero_to) break;
        float g = 0.f;
        if (c < classes) g = (__expf(zv[c] - mx - lse) - (c == y ? 1.f : 0.f)) * gs;
        if (dl_f32)
          reinterpret_cast<float*>(dl)[p * ds + c] = g;
        else
          reinterpret_cast<b2h*>(dl)[p * ds + c] = f_to_h(g);
      }
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
                            const float* __restrict__ cw, int classes, int nimg, float* __restrict__ loss,
                            const int* __restrict__ err, int* __restrict__ status) {
  // one warp: lane-strided partial sums, then a fixed xor tree (deterministic order)
  if (blockIdx.x != 0) return;
  const int lane = threadIdx.x & 31;
  double total = 0.0;
  for (int n = 0; n < nimg; ++n) {
    double s = 0.0;
    for (int b = lane; b < nb; b += 32) s += part[n * nb + b];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    double ws = 0.0;
    for (int c = 0; c < classes; ++c) ws += static_cast<double>(counts[n * classes + c]) * cw[c];
    total += s / ws;
  }
  if (lane == 0) {
    // a label outside [0, classes) (the reference raises ValueError, loss.py:72-74): the loss is
    // NaN, so it cannot pass for a real value, and the status word says why
    const bool bad = *err != 0;
    loss[0] = bad ? __int_as_float(0x7fc00000) : static_cast<float>(total / nimg);
    if (status) *status = bad ? 1 : 0;
  }
}

}  // namespace b2

using namespace b2;

extern "C" size_t b2dl_wce_workspace_size(int n, int h, int w, int classes) {
  (void)classes;
  const int nb = wce_blocks_per_img(n, static_cast<long long>(h) * w);
  return align_up(static_cast<size_t>(n) * nb * sizeof(double), 256) + 64;
}

extern "C" int b2dl_wce(b2dl_act logits, const uint8_t* labels, const float* class_weights, int classes,
                        float* loss_out, int* counts, b2dl_act dlogits, int dlogits_f32, float dlogits_scale,
                        uint8_t* pred,
                        int* status, void* workspace, size_t workspace_bytes, void* stream) {
  if (classes < 2 || classes > WCE_MAX_CLASSES || logits.c != classes || dlogits.c != classes) return B2DL_E_VALUE;
  if (!logits.ptr || !labels || !class_weights || !loss_out || !counts || !dlogits.ptr) return B2DL_E_VALUE;
  if (workspace_bytes < b2dl_wce_workspace_size(logits.n, logits.h, logits.w, classes)) return B2DL_E_VALUE;
  cudaStream_t st = as_stream(stream);
  const long long hw = static_cast<long long>(logits.h) * logits.w;
  const int nb = wce_blocks_per_img(logits.n, hw);
  double* part = reinterpret_cast<double*>(workspace);
  int* err = reinterpret_cast<int*>(reinterpret_cast<char*>(workspace) +
                                    align_up(static_cast<size_t>(logits.n) * nb * sizeof(double), 256));
  cudaMemsetAsync(counts, 0, sizeof(int) * logits.n * classes, st);
  cudaMemsetAsync(err, 0, sizeof(int), st);
  dim3 grid(nb, logits.n);
  k_wce_hist<<<grid, WCE_THREADS, 0, st>>>(labels, hw, classes, counts, err);
  k_wce_main<<<grid, WCE_THREADS, 0, st>>>(reinterpret_cast<const float*>(logits.ptr), logits.c_stride, labels, class_weights,
                                   counts, hw, classes, logits.n, dlogits.ptr, dlogits.c_stride, dlogits_f32,
                                   dlogits_scale,
                                   pred, part);
  k_wce_final<<<1, 32, 0, st>>>(part, nb, counts, class_weights, classes, logits.n, loss_out, err, status);
  return check_launch();
}
