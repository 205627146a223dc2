// vec2.cuh -- the arithmetic the generated stencil (ku_gen.cuh) is written in.
//
// For a scalar TA (float, double) these are the plain operations. For float2
// they are sm_100's paired f32 instructions (FFMA2 / FADD2 / FMUL2): one
// instruction applies the same operation to two independent lanes -- here two
// vertices of the same colour handled by one thread -- so a level-0 kernel
// issues half the floating-point instructions. Each lane rounds exactly like
// the scalar instruction (round-to-nearest, no contraction changes), so a
// paired kernel is bit-identical to its scalar twin.
#pragma once
#include <cuda_runtime.h>

namespace ihomgpu {

template <typename T>
__device__ __forceinline__ T vzero() {
  return T(0);
}
template <>
__device__ __forceinline__ float2 vzero<float2>() {
  return make_float2(0.f, 0.f);
}

template <typename T, typename S>
__device__ __forceinline__ T vbc(S s) {
  return T(s);
}
template <>
__device__ __forceinline__ float2 vbc<float2, float>(float s) {
  return make_float2(s, s);
}

template <typename T>
__device__ __forceinline__ T vadd(T a, T b) {
  return a + b;
}
template <typename T>
__device__ __forceinline__ T vsub(T a, T b) {
  return a - b;
}
template <typename T>
__device__ __forceinline__ T vneg(T a) {
  return -a;
}
template <typename T>
__device__ __forceinline__ T vmul(T a, T b) {
  return a * b;
}
template <typename T>
__device__ __forceinline__ T vfma(T a, T b, T c) {
  return fma(a, b, c);
}

__device__ __forceinline__ float2 vneg(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float2 vadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 vsub(float2 a, float2 b) { return __fadd2_rn(a, vneg(b)); }
__device__ __forceinline__ float2 vmul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 vfma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

}  // namespace ihomgpu
