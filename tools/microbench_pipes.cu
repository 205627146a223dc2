// Pipe-throughput probe: DFMA, FFMA, F2F.F64.F32, F2F.F32.F64 per SM per clock.
#include <cstdio>
#include <cuda_runtime.h>
#define N_ITER 4096
__global__ void k_dfma(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < N_ITER; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_ffma(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < N_ITER; ++i) {
    x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
    x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
// all-register FFMA (per-thread multiplier/addend) and the sm_100 paired FFMA2 (2 lanes of f32 per instruction)
__global__ void k_ffma_reg(float* out, const float* in) {
  const float a = in[threadIdx.x], b = in[threadIdx.x + 1];
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < N_ITER; ++i) {
    x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
    x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_ffma2(float* out, const float* in) {
  const float2 a = make_float2(in[threadIdx.x], in[threadIdx.x + 2]), b = make_float2(in[threadIdx.x + 1], in[threadIdx.x + 3]);
  float2 x0 = make_float2(threadIdx.x, 1), x1 = make_float2(2, 3), x2 = make_float2(4, 5), x3 = make_float2(6, 7);
  float2 x4 = make_float2(8, threadIdx.x), x5 = make_float2(9, 1), x6 = make_float2(10, 2), x7 = make_float2(11, 3);
  for (int i = 0; i < N_ITER; ++i) {
    x0 = __ffma2_rn(x0, a, b); x1 = __ffma2_rn(x1, a, b); x2 = __ffma2_rn(x2, a, b); x3 = __ffma2_rn(x3, a, b);
    x4 = __ffma2_rn(x4, a, b); x5 = __ffma2_rn(x5, a, b); x6 = __ffma2_rn(x6, a, b); x7 = __ffma2_rn(x7, a, b);
  }
  const float2 s = __fadd2_rn(__fadd2_rn(__fadd2_rn(x0, x1), __fadd2_rn(x2, x3)), __fadd2_rn(__fadd2_rn(x4, x5), __fadd2_rn(x6, x7)));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s.x + s.y;
}
// pure f32 -> f64 conversion throughput (integer adds keep the inputs distinct; DADD-free accumulation
// through the bit pattern) vs the same conversion done with integer ops on the ALU pipe
__global__ void k_f2d_pure(unsigned long long* out, float a) {
  float f0 = threadIdx.x * 1e-3f + 1.0f, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3;
  unsigned long long acc = 0;
  for (int i = 0; i < N_ITER; ++i) {
    acc ^= __double_as_longlong((double)f0) ^ __double_as_longlong((double)f1) ^ __double_as_longlong((double)f2) ^
           __double_as_longlong((double)f3);
    f0 = __int_as_float(__float_as_int(f0) + 1); f1 = __int_as_float(__float_as_int(f1) + 1);
    f2 = __int_as_float(__float_as_int(f2) + 1); f3 = __int_as_float(__float_as_int(f3) + 1);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__device__ __forceinline__ unsigned long long f2d_bits(float x) {  // normal, non-zero finite x only
  const unsigned b = __float_as_uint(x);
  const unsigned hi = (b & 0x80000000u) | (((b >> 3) & 0x0fffffffu) + (896u << 20));
  return ((unsigned long long)hi << 32) | (unsigned long long)(b << 29);
}
__global__ void k_f2d_int(unsigned long long* out, float a) {
  float f0 = threadIdx.x * 1e-3f + 1.0f, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3;
  unsigned long long acc = 0;
  for (int i = 0; i < N_ITER; ++i) {
    acc ^= f2d_bits(f0) ^ f2d_bits(f1) ^ f2d_bits(f2) ^ f2d_bits(f3);
    f0 = __int_as_float(__float_as_int(f0) + 1); f1 = __int_as_float(__float_as_int(f1) + 1);
    f2 = __int_as_float(__float_as_int(f2) + 1); f3 = __int_as_float(__float_as_int(f3) + 1);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
// f32 -> f64 conversions feeding DFMA (the mixed-precision stencil apply pattern)
__global__ void k_f2d(double* out, float a) {
  float f0 = threadIdx.x * 1e-3f, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3, f4=f0+4,f5=f0+5,f6=f0+6,f7=f0+7;
  double acc = 0;
  for (int i = 0; i < N_ITER; ++i) {
    f0 += a; f1 += a; f2 += a; f3 += a; f4 += a; f5 += a; f6 += a; f7 += a;
    acc += (double)f0 + (double)f1 + (double)f2 + (double)f3 + (double)f4 + (double)f5 + (double)f6 + (double)f7;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_d2f(float* out, double a) {
  double d0 = threadIdx.x * 1e-3, d1 = d0 + 1, d2 = d0 + 2, d3 = d0 + 3, d4=d0+4,d5=d0+5,d6=d0+6,d7=d0+7;
  float acc = 0;
  for (int i = 0; i < N_ITER; ++i) {
    d0 += a; d1 += a; d2 += a; d3 += a; d4 += a; d5 += a; d6 += a; d7 += a;
    acc += (float)d0 + (float)d1 + (float)d2 + (float)d3 + (float)d4 + (float)d5 + (float)d6 + (float)d7;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int blocks = p.multiProcessorCount * 8, threads = 256;
  double* d; float* f; cudaMalloc(&d, blocks * threads * 8); cudaMalloc(&f, blocks * threads * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch, double ops_per_iter) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(a); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = 5.0 * blocks * threads * (double)N_ITER * ops_per_iter;
    double per_clk_sm = ops / (ms * 1e-3) / (p.multiProcessorCount * clk * 1e3);
    printf("%-34s %10.3f Gop/s  %7.2f op/clk/SM (at nominal %d MHz)\n", name, ops / (ms * 1e-3) / 1e9, per_clk_sm, clk / 1000);
  };
  run("DFMA", [&] { k_dfma<<<blocks, threads>>>(d, 0.999, 1e-3); }, 8);
  run("FFMA", [&] { k_ffma<<<blocks, threads>>>(f, 0.999f, 1e-3f); }, 8);
  float* in; cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0, 4096 * 4);
  run("FFMA all-register", [&] { k_ffma_reg<<<blocks, threads>>>(f, in); }, 8);
  run("FFMA2 all-register (f32 lanes)", [&] { k_ffma2<<<blocks, threads>>>(f, in); }, 16);
  unsigned long long* ul; cudaMalloc(&ul, blocks * threads * 8);
  run("F2F.F64.F32 pure (+4 IADD, XOR)", [&] { k_f2d_pure<<<blocks, threads>>>(ul, 1e-3f); }, 4);
  run("f32->f64 by integer ops (+4 IADD, XOR)", [&] { k_f2d_int<<<blocks, threads>>>(ul, 1e-3f); }, 4);
  run("F2F.F64.F32 (+8 FADD +8 DADD)", [&] { k_f2d<<<blocks, threads>>>(d, 1e-3f); }, 8);
  run("F2F.F32.F64 (+8 DADD +8 FADD)", [&] { k_d2f<<<blocks, threads>>>(f, 1e-3); }, 8);
  printf("SMs %d\n", p.multiProcessorCount);
  return 0;
}
