// L2 reduction throughput probe for the msa_row bias gradient: every (b, h, key tile, query tile)
// adds a 128 x 128 fp32 tile into dbias[h][key][query] (2 MB) with red.global.add(.v4).f32, i.e. the
// batch sum done by L2 atomics instead of a bf16 workspace + reduction pass.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/_exp/red_rate scripts/red_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int V4>
__global__ void k(float* dbias, int B, int H, int L) {
  // unit = (b, h, kt, qt); a CTA of 256 threads adds one 128 x 128 tile
  const int nt = L / 128;
  for (int u = blockIdx.x; u < B * H * nt * nt; u += gridDim.x) {
    const int qt = u % nt, kt = (u / nt) % nt, h = (u / (nt * nt)) % H;
    float* tile = dbias + ((size_t)h * L + kt * 128) * L + qt * 128;
    for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) {  // 32 float4 per key row
      const int r = i / 32, c4 = i % 32;
      float* p = tile + (size_t)r * L + c4 * 4;
      const float v = 1e-3f * (u & 7);
      if (V4) {
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
      } else {
        atomicAdd(p, v); atomicAdd(p + 1, v); atomicAdd(p + 2, v); atomicAdd(p + 3, v);
      }
    }
  }
}
int main() {
  const int B = 128, H = 8, L = 256;
  float* d; cudaMalloc(&d, (size_t)H * L * L * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int v4 = 0; v4 < 2; ++v4)
    for (int grid : {sms, 2 * sms, 4 * sms}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(d, 0, (size_t)H * L * L * 4);
        cudaEventRecord(a);
        if (v4) k<1><<<grid, 256>>>(d, B, H, L); else k<0><<<grid, 256>>>(d, B, H, L);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("%s grid %4d: %.1f us for %d M fp32 adds (%.2f T adds/s)\n", v4 ? "red.v4" : "atomicAdd", grid,
                        ms * 1e3, B * H * L * L / 1000000, (double)B * H * L * L / (ms * 1e-3) / 1e12);
      }
    }
  return 0;
}
