// Probe: tcgen05.mma SS-mode issue rate (M=128, N = 64/128/256, K=16 bf16) from fixed smem tiles,
// and tcgen05.ld 32x32b.x32 drain rate.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../include
// -I../paper_2203_00854_b200/csrc mma_probe.cu -o mma_probe && ./mma_probe
#include <cstdio>
#include "common.cuh"
using namespace evo;

template <int N, int SW>
__global__ void probe(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tsh;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&tsh, 256);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tsh, sA = smem_u32(smem), sB = sA + 16384;
  constexpr uint32_t ID = make_idesc_bf16(128, N, 0, 0);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t ad, bd;
        if (SW == 128) {
          ad = (uint64_t)(((sA + kk * 32) >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
          bd = (uint64_t)(((sB + kk * 32) >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
        } else {
          ad = make_sdesc(sA + kk * 2 * 16 * 128, 16 * 128, 128);
          bd = make_sdesc(sB + kk * 2 * (N / 8) * 128, (N / 8) * 128, 128);
        }
        mma_bf16(tm, ad, bd, ID, (it | kk) != 0);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 256);
}

__global__ void ldprobe(long long* out, int iters) {
  __shared__ uint32_t tsh;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&tsh, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tsh + ((uint32_t)((warp & 3) * 32) << 16);
  float acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int c = 0; c < 128; c += 32) {
      float v[32];
      tmem_ld32(tm + c + (warp >> 2) * 128, v);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += v[j];
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345.f) out[1] = 0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tsh, 256);
}


__global__ void contend(long long* out, int iters, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tsh;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&tsh, 512);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); stop = 0; }
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tsh, sA = smem_u32(smem), sB = sA + 16384;
  constexpr uint32_t ID = make_idesc_bf16(128, 128, 0, 0);
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t ad = (uint64_t)(((sA + kk * 32) >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
        uint64_t bd = (uint64_t)(((sB + kk * 32) >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
        mma_bf16(tm, ad, bd, ID, (it | kk) != 0);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[0] = clock64() - t0;
    stop = 1;
  } else if (warp >= 4) {
    const uint32_t tl = tm + ((uint32_t)((warp & 3) * 32) << 16) + 128 + ((warp - 4) >> 2) * 128;
    const uint32_t sdst = sA + 65536 + (warp - 4) * 4096 + (threadIdx.x & 31) * 16;
    float acc = 0;
    long long n = 0;
    while (!stop) {
      if (mode == 1) {
        float v[32];
        tmem_ld32(tl, v);
        tmem_ld_wait();
        for (int j = 0; j < 32; ++j) acc += v[j];
      } else if (mode == 2) {
        for (int r = 0; r < 8; ++r) st_shared_v4(sdst + (r & 7) * 512, n, r, 0, 0);
      }
      ++n;
    }
    if ((threadIdx.x & 31) == 0) out[1 + warp] = n;
    if (acc == 1234.f) out[100] = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

// A K-major SW128, B MN-major SW128 (atoms of 64 n x 8 k rows; LBO = atom stride, SBO = 1 KB)
template <int N, bool BMN, bool AMN>
__global__ void probe_mn(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tsh;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&tsh, 256);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tsh, sA = smem_u32(smem), sB = sA + 16384;
  constexpr uint32_t ID = make_idesc_bf16(128, N, AMN, BMN);
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t ad = AMN ? ((uint64_t)(((sA + kk * 2048) >> 4) & 0x3FFF) | ((uint64_t)(8192 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61))
                          : ((uint64_t)(((sA + kk * 32) >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61));
        uint64_t bd = BMN ? ((uint64_t)(((sB + kk * 2048) >> 4) & 0x3FFF) | ((uint64_t)(8192 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61))
                          : ((uint64_t)(((sB + kk * 32) >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61));
        mma_bf16(tm, ad, bd, ID, (it | kk) != 0);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[0] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 256);
}
template <int N, bool BMN, bool AMN>
void run_mn(long long* d) {
  cudaFuncSetAttribute(probe_mn<N, BMN, AMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  probe_mn<N, BMN, AMN><<<1, 128, 65536>>>(d, 2000);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("SS mma N=%d A %s B %s (sw128): %.1f clk per K=16 MMA\n", N, AMN ? "MN" : "K", BMN ? "MN" : "K", (double)h / 8000);
}

template <int N, int SW>
void run(long long* d, int grid) {
  cudaFuncSetAttribute(probe<N, SW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int iters = 2000;
  probe<N, SW><<<grid, 128, 65536>>>(d, iters);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("SS mma M=128 N=%d sw=%d grid=%d: %.1f clk per K=16 MMA (floor %d)\n", N, SW, grid, (double)h / (iters * 4), 128 * N / 256);
}

int main() {
  long long* d;
  cudaMalloc(&d, 4096 * 8);
  run<64, 128>(d, 1); run<128, 128>(d, 1); run<256, 128>(d, 1);
  run<64, 0>(d, 1); run<128, 0>(d, 1); run<256, 0>(d, 1);
  run<128, 128>(d, 148); run<256, 128>(d, 148);
  for (int w : {4, 8}) {
    ldprobe<<<1, 32 * w>>>(d, 1000);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("tcgen05.ld 32x32b.x32 + wait, %d warps: %.1f clk per load per warp -> %.1f B/clk per SM\n", w, (double)h / (1000 * 4),
           4096.0 * w / ((double)h / (1000 * 4)));
  }
  run_mn<128, true, false>(d); run_mn<128, false, true>(d); run_mn<128, true, true>(d); run_mn<256, true, false>(d);
  cudaFuncSetAttribute(contend, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  for (int mode : {0, 1, 2}) {
    contend<<<148, 384, 131072>>>(d, 2000, mode);
    cudaDeviceSynchronize();
    long long h[16];
    cudaMemcpy(h, d, 16 * 8, cudaMemcpyDeviceToHost);
    printf("contention mode %d (0 none, 1 tmem loads x8 warps, 2 st.shared x8 warps): %.1f clk per N=128 MMA; side iters/warp %lld\n",
           mode, (double)h[0] / 8000, h[5]);
  }
  return 0;
}
