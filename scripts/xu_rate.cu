// Pipe-sharing probe: MUFU.EX2 vs F2FP (fp32 -> bf16x2 pack) throughput per SM, alone and mixed.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/_exp/xu_rate scripts/xu_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
template <int MODE>
__global__ void k(unsigned* out, int n) {
  float x[32];
  unsigned acc = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = (threadIdx.x + i) * -1e-3f;
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      float a = x[i], b = x[i + 1];
      if (MODE == 0 || MODE == 2 || MODE == 3) {  // exp2
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
      }
      unsigned p = 0;
      if (MODE == 1 || MODE == 2) {  // F2FP pack
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(a), "f"(b));
      } else if (MODE == 3) {  // PRMT (truncating) pack
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(p) : "r"(__float_as_uint(b)), "r"(__float_as_uint(a)));
      }
      if (MODE == 4 || MODE == 6) {  // FMNMX3 chain work (2 per pair of elements)
        float m;
        asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(m) : "f"(a), "f"(b), "f"(x[(i + 2) & 31]));
        asm volatile("max.f32 %0, %1, %2, %3;" : "+f"(a) : "f"(m), "f"(b), "f"(x[(i + 5) & 31]));
      }
      if (MODE == 5 || MODE == 7) {  // FMNMX (2-input) x2
        asm volatile("max.f32 %0, %0, %1;" : "+f"(a) : "f"(b));
        asm volatile("max.f32 %0, %0, %1;" : "+f"(b) : "f"(a));
      }
      if (MODE == 6 || MODE == 7) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
      }
      acc += p;
      x[i] = a - 1e-3f; x[i + 1] = b - 2e-3f;
    }
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) acc += __float_as_uint(x[i]);
  if (acc == 12345u) out[0] = acc;
}
template <int MODE>
void run(const char* name, int warps) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned* o; cudaMalloc(&o, 4);
  k<MODE><<<sms, warps * 32>>>(o, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int n = 2048;
  cudaEventRecord(a);
  k<MODE><<<sms, warps * 32>>>(o, n);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double elems = (double)sms * warps * 32 * n * 32;
  printf("%-28s warps/SM %2d: %.2f elements/clk/SM\n", name, warps, elems / (ms * 1e-3) / sms / (clk * 1e3));
  cudaFree(o);
}
int main() {
  for (int w : {4, 8, 16}) {
    run<0>("ex2 only", w); run<1>("F2FP pack only (per 2 el)", w); run<2>("ex2 + F2FP pack", w);
    run<3>("ex2 + PRMT pack", w);
    run<4>("FMNMX3 x2 per 2 el", w); run<5>("FMNMX x2 per 2 el", w); run<6>("ex2 + FMNMX3 x1/el", w);
    run<7>("ex2 + FMNMX x1/el", w);
  }
  return 0;
}
