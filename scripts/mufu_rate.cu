// MUFU.EX2 throughput per SM: nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/mufu scripts/mufu_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP, int FMA>
__global__ void k(float* out, int n, float a) {
  float x[ILP];
  for (int i = 0; i < ILP; ++i) x[i] = a * (threadIdx.x + i) * 1e-3f;
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
      float z = y;
#pragma unroll
      for (int f = 0; f < FMA; ++f) z = fmaf(z, 0.999f, -0.5f);
      x[i] = z;
    }
  }
  float s = 0;
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == 1234.5f) out[0] = s;
}
template <int ILP, int FMA>
void run(int warps) {
  int dev; cudaGetDevice(&dev); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* o; cudaMalloc(&o, 4);
  int n = 4096;
  k<ILP, FMA><<<sms, warps * 32>>>(o, 16, 1.f);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<ILP, FMA><<<sms, warps * 32>>>(o, n, 1.f);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ex = (double)sms * warps * 32 * n * ILP;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("warps/SM %2d ILP %2d FMA/ex2 %d: %.2f ex2/clk/SM (at %d MHz)\n", warps, ILP, FMA,
         ex / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  cudaFree(o);
}
int main() {
  run<8, 0>(4); run<8, 0>(8); run<8, 0>(16); run<16, 0>(8); run<32, 0>(8);
  run<8, 1>(8); run<8, 2>(8); run<16, 2>(8); run<16, 4>(16);
  return 0;
}
