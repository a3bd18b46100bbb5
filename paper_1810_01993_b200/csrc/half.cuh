// The 16-bit storage type of activations, gradients and the weight mirror.  One source, two
// builds: libb2dl.so (bf16, the training step) and libb2dl_f16.so (-DB2DL_F16: IEEE fp16, the
// paper's FP16 arithmetic for config 4 -- kind::f16 MMAs with f16 A/B operands, fp32
// accumulation).  Everything that packs, unpacks or describes a 16-bit value goes through here.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

#ifdef B2DL_F16
typedef __half b2h;
typedef __half2 b2h2;
#define B2H_TMA CU_TENSOR_MAP_DATA_TYPE_FLOAT16
constexpr uint32_t B2H_MMA_FMT = 0;  // tcgen05 kind::f16 operand format: F16
__device__ __forceinline__ float h_lo(uint32_t v) {
  return __half2float(__ushort_as_half(static_cast<unsigned short>(v & 0xFFFFu)));
}
__device__ __forceinline__ float h_hi(uint32_t v) {
  return __half2float(__ushort_as_half(static_cast<unsigned short>(v >> 16)));
}
__device__ __forceinline__ uint32_t pack_h2(float a, float b) {  // a -> low half
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ b2h f_to_h(float x) { return __float2half_rn(x); }
__device__ __forceinline__ float h_to_f(b2h x) { return __half2float(x); }
__device__ __forceinline__ b2h2 h2_from(float a, float b) { return __floats2half2_rn(a, b); }
#else
typedef __nv_bfloat16 b2h;
typedef __nv_bfloat162 b2h2;
#define B2H_TMA CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
constexpr uint32_t B2H_MMA_FMT = 1;  // tcgen05 kind::f16 operand format: BF16
__device__ __forceinline__ float h_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float h_hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pack_h2(float a, float b) {  // a -> low half
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ b2h f_to_h(float x) { return __float2bfloat16_rn(x); }
__device__ __forceinline__ float h_to_f(b2h x) { return __bfloat162float(x); }
__device__ __forceinline__ b2h2 h2_from(float a, float b) { return __floats2bfloat162_rn(a, b); }
#endif

// 0xFFFF in each 16-bit half of w whose value is > 0, else 0 (an IEEE compare: -0, negatives and
// NaN give 0) -- the relu-VJP mask of a packed pair, applied to a packed result with one AND
__device__ __forceinline__ uint32_t pos_mask_h2(uint32_t w) {
  return __hgt2_mask(*reinterpret_cast<const b2h2*>(&w), h2_from(0.f, 0.f));
}
