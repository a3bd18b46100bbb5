// Host-side helpers shared by the .cu translation units of libb2dl.so.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <cstdio>

#include "../../include/b2dl.h"
#include "half.cuh"

namespace b2 {

int num_sms();
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda needed).
int encode_tiled(CUtensorMap* m, CUtensorMapDataType dt, int rank, void* ptr, const uint64_t* dims,
                 const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle sw,
                 const uint32_t* elem_strides = nullptr);
// 4-D NHWC bf16 activation map: dims (c, w, h, n), box (box_c, box_w, box_h, 1).
int act_map(CUtensorMap* m, const b2dl_act& a, int box_c, int box_w, int box_h, CUtensorMapSwizzle sw);
int window_map(CUtensorMap* m, const b2dl_act& x, int c_v, int w_v, int box_c, int box_w, int box_h,
               CUtensorMapSwizzle sw);
int act_map_phase(CUtensorMap* m, const b2dl_act& a, int f, int ph, int pw, int box_c, int box_w, int box_h,
                  CUtensorMapSwizzle sw);
int act_map_strided(CUtensorMap* m, const b2dl_act& a, int box_c, int box_w, int box_h, int stride,
                    CUtensorMapSwizzle sw);
int act_map5(CUtensorMap* m, const b2dl_act& a, int box_w, int box_h, int g);

inline int check_launch() {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return B2DL_OK;
  fprintf(stderr, "b2dl: CUDA error %s\n", cudaGetErrorString(e));
  return B2DL_E_CUDA;
}
inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline int round_up(int a, int b) { return (a + b - 1) / b * b; }
inline int cdiv(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }
inline size_t align_up(size_t a, size_t b) { return (a + b - 1) / b * b; }

// largest power of two (<= cap) dividing w
inline int pow2_divisor(int w, int cap) {
  int b = 1;
  while (b * 2 <= cap && w % (b * 2) == 0) b *= 2;
  return b;
}

}  // namespace b2
