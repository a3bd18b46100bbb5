// LARC layer-wise rate control + SGD momentum over all parameter tensors
// (pkg/src/deskdl/optimizer.py:48-83, applied per tensor by trainer.py:364-367).
//
// Launch 1: per-(tensor, slice) partial sums of w^2 and g^2 (fp64 accumulation).
// Launch 2: one warp per tensor folds its partials in a fixed order, applies the
//           zero-norm / eps rules and the trust-ratio clip, writes lr_t.
// Launch 3: m = beta*m + s*g + wd*w ; w -= lr_t * m   (s = grad_scale = 1/P)
// The reference raises FloatingPointError on a non-finite norm; here a device
// status word is set and launch 3 leaves every tensor untouched.
#include <cuda_bf16.h>

#include <algorithm>

#include "internal.h"

namespace b2 {

constexpr int LARC_SLICES = 32;

__global__ void k_larc_norms(const float* __restrict__ w, const float* __restrict__ g,
                             const int64_t* __restrict__ off, double* __restrict__ part) {
  const int t = blockIdx.y;
  const int64_t lo = off[t], hi = off[t + 1];
  double sw = 0.0, sg = 0.0;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
  // 16-byte loads over the 4-aligned interior (segments start 64-aligned), each float4's four
  // squares summed in fp32 and then folded into fp64 (fixed order; a quarter of the f32 -> f64
  // conversions), two float4 of each tensor in flight; head / tail (or a short segment) element-wise
  const int64_t a0 = (lo + 3) & ~int64_t(3), a1 = hi & ~int64_t(3);
  auto one = [&](int64_t i) {
    const double a = w[i], b = g[i];
    sw += a * a;
    sg += b * b;
  };
  if (a0 >= a1) {
    for (int64_t i = lo + tid; i < hi; i += nth) one(i);
  } else {
    for (int64_t i = lo + tid; i < a0; i += nth) one(i);
    const float4* w4 = reinterpret_cast<const float4*>(w);
    const float4* g4 = reinterpret_cast<const float4*>(g);
    auto sq4 = [](float4 q) { return fmaf(q.w, q.w, fmaf(q.z, q.z, fmaf(q.y, q.y, q.x * q.x))); };
    int64_t v = a0 / 4 + tid;
    for (; v + nth < a1 / 4; v += 2 * nth) {
      const float4 wa = w4[v], wb = w4[v + nth], ga = g4[v], gb = g4[v + nth];
      sw += sq4(wa);
      sw += sq4(wb);
      sg += sq4(ga);
      sg += sq4(gb);
    }
    for (; v < a1 / 4; v += nth) {
      sw += sq4(w4[v]);
      sg += sq4(g4[v]);
    }
    for (int64_t i = a1 + tid; i < hi; i += nth) one(i);
  }
  __shared__ double rw[32], rg[32];
  for (int o = 16; o > 0; o >>= 1) {
    sw += __shfl_xor_sync(0xffffffffu, sw, o);
    sg += __shfl_xor_sync(0xffffffffu, sg, o);
  }
  if ((threadIdx.x & 31) == 0) {
    rw[threadIdx.x >> 5] = sw;
    rg[threadIdx.x >> 5] = sg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) {
      a += rw[k];
      b += rg[k];
    }
    part[(static_cast<int64_t>(t) * gridDim.x + blockIdx.x) * 2 + 0] = a;
    part[(static_cast<int64_t>(t) * gridDim.x + blockIdx.x) * 2 + 1] = b;
  }
}

__global__ void k_larc_rates(const double* __restrict__ part, int ntensors, int slices, float lr, float trust,
                             float wd, float eps, float grad_scale, float* __restrict__ lr_out,
                             int* __restrict__ status) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= ntensors) return;
  double a = 0.0, b = 0.0;
  if (lane == 0) {
    for (int k = 0; k < slices; ++k) {
      a += part[(static_cast<int64_t>(t) * slices + k) * 2 + 0];
      b += part[(static_cast<int64_t>(t) * slices + k) * 2 + 1];
    }
    // norms rounded to fp32 like np.linalg.norm on float32 arrays (optimizer.py:54-55)
    const float wn = static_cast<float>(sqrt(a));
    const float gn = static_cast<float>(sqrt(b) * static_cast<double>(grad_scale));
    float r;
    if (!isfinite(wn) || !isfinite(gn)) {
      atomicExch(status, 1);
      r = 0.f;
    } else if (wn == 0.f) {
      r = lr;
    } else {
      // python-float (fp64) scalar arithmetic as in optimizer.py:58-63
      const double denom = static_cast<double>(gn) + static_cast<double>(wd) * wn;
      if (denom < static_cast<double>(eps))
        r = lr;
      else
        r = static_cast<float>(fmin(static_cast<double>(trust) * wn / denom, static_cast<double>(lr)));
    }
    lr_out[t] = r;
  }
}

// w, m, g segment update, 4 elements per thread on aligned interiors; optionally also
// writes the bf16 mirror of w that the conv kernels read as their weight operand.
__device__ __forceinline__ void larc_one(float* w, float* m, const float* g, b2h* wb, int64_t i, float r,
                                         float beta, float wd, float gs) {
  float mv = m[i] * beta;
  mv += g[i] * gs;
  const float wv = w[i];
  if (wd != 0.f) mv += wd * wv;
  m[i] = mv;
  const float nw = wv - r * mv;
  w[i] = nw;
  if (wb) wb[i] = f_to_h(nw);
}

__global__ void k_larc_apply(float* __restrict__ w, float* __restrict__ m, const float* __restrict__ g,
                             b2h* __restrict__ wb, const int64_t* __restrict__ off,
                             const float* __restrict__ lr_t, float beta, float wd, float grad_scale,
                             const int* __restrict__ status, int cast_only) {
  if (*status) return;
  const int t = blockIdx.y;
  const int64_t lo = off[t], hi = off[t + 1];
  const float r = cast_only ? 0.f : lr_t[t];
  const int64_t a0 = (lo + 3) & ~int64_t(3), a1 = hi & ~int64_t(3);
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
  if (a0 >= a1) {
    for (int64_t i = lo + tid; i < hi; i += nth) {
      if (cast_only)
        wb[i] = f_to_h(w[i]);
      else
        larc_one(w, m, g, wb, i, r, beta, wd, grad_scale);
    }
    return;
  }
  for (int64_t i = lo + tid; i < a0; i += nth) {
    if (cast_only)
      wb[i] = f_to_h(w[i]);
    else
      larc_one(w, m, g, wb, i, r, beta, wd, grad_scale);
  }
  for (int64_t i = a1 + tid; i < hi; i += nth) {
    if (cast_only)
      wb[i] = f_to_h(w[i]);
    else
      larc_one(w, m, g, wb, i, r, beta, wd, grad_scale);
  }
  // two float4 groups per thread in flight (the loop body is independent per group)
#pragma unroll 2
  for (int64_t v = a0 / 4 + tid; v < a1 / 4; v += nth) {
    float4 wv = reinterpret_cast<float4*>(w)[v];
    if (!cast_only) {
      float4 mv = reinterpret_cast<float4*>(m)[v];
      const float4 gv = reinterpret_cast<const float4*>(g)[v];
      float* mm = &mv.x;
      float* ww = &wv.x;
      const float* gg = &gv.x;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float x = mm[e] * beta;        // m *= beta
        x += gg[e] * grad_scale;       // m += g
        if (wd != 0.f) x += wd * ww[e];  // m += wd * w
        mm[e] = x;
        ww[e] = ww[e] - r * x;         // w -= f32(lr_eff) * m
      }
      reinterpret_cast<float4*>(m)[v] = mv;
      reinterpret_cast<float4*>(w)[v] = wv;
    }
    if (wb) {
      b2h2 lo2 = h2_from(wv.x, wv.y), hi2 = h2_from(wv.z, wv.w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&lo2);
      u.y = *reinterpret_cast<uint32_t*>(&hi2);
      reinterpret_cast<uint2*>(wb)[v] = u;
    }
  }
}

}  // namespace b2

using namespace b2;

extern "C" size_t b2dl_larc_workspace_size(int64_t total_elems, int ntensors) {
  (void)total_elems;
  return static_cast<size_t>(ntensors) * LARC_SLICES * 2 * sizeof(double) + 256;
}

extern "C" int b2dl_larc_update(const b2dl_larc_args* a, void* stream) {
  if (!a || !a->w || !a->m || !a->g || !a->offsets || a->ntensors < 1 || !a->lr_out || !a->status)
    return B2DL_E_VALUE;
  if (a->workspace_bytes < b2dl_larc_workspace_size(0, a->ntensors)) return B2DL_E_VALUE;
  cudaStream_t st = as_stream(stream);
  double* part = reinterpret_cast<double*>(a->workspace);
  if (a->mode < 0 || a->mode > 3) return B2DL_E_VALUE;
  if (a->mode == 3 && !a->w_bf16) return B2DL_E_VALUE;
  cudaMemsetAsync(a->status, 0, sizeof(int), st);
  dim3 grid(LARC_SLICES, a->ntensors);
  if (a->mode == 0 || a->mode == 1) {
    k_larc_norms<<<grid, 256, 0, st>>>(a->w, a->g, a->offsets, part);
    const int warps_per_block = 8;
    k_larc_rates<<<(a->ntensors + warps_per_block - 1) / warps_per_block, 32 * warps_per_block, 0, st>>>(
        part, a->ntensors, LARC_SLICES, a->lr, a->trust, a->weight_decay, a->eps, a->grad_scale, a->lr_out,
        a->status);
  }
  if (a->mode == 1) return check_launch();
  k_larc_apply<<<grid, 256, 0, st>>>(a->w, a->m, a->g, reinterpret_cast<b2h*>(a->w_bf16), a->offsets,
                                     a->lr_out, a->momentum, a->weight_decay, a->grad_scale, a->status,
                                     a->mode == 3);
  return check_launch();
}
