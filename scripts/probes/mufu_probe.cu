// MUFU ex2 / FFMA throughput probe (B200): ops per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int KIND>
__global__ void k(float* out, int iters, long long* cyc) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      else if (KIND == 1) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f3A000000;" : "+f"(a[i]));
      else { unsigned short h; asm volatile("{.reg .b32 t; mov.b32 t, %0; ex2.approx.ftz.bf16x2 t, t; mov.b32 %0, t;}" : "+f"(a[i])); }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; long long* cyc; cudaMalloc(&out, sms * 1024 * 4); cudaMalloc(&cyc, sms * 8);
  const int iters = 4096;
  for (int kind = 0; kind < 3; ++kind)
    for (int threads = 128; threads <= 1024; threads *= 2) {
      auto f = kind == 0 ? k<0> : kind == 1 ? k<1> : k<2>;
      f<<<sms, threads>>>(out, iters, cyc);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double ops = (double)threads * iters * 8 * (kind == 2 ? 2 : 1);
      printf("%s threads %4d: %.2f results/clk/SM\n", kind == 0 ? "ex2.f32  " : kind == 1 ? "ffma     " : "ex2.bf16x2",
             threads, ops / c);
    }
  return 0;
}
