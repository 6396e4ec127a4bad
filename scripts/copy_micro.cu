// Streaming-load microbenchmark: how fast can one persistent CTA per SM pull bytes from
// HBM into a 4-stage shared-memory ring with (a) 128 threads of 16-byte cp.async +
// cp.async.mbarrier.arrive.noinc, (b) one thread of cp.async.bulk (1-D TMA) + expect_tx.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/copy_micro scripts/copy_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D_%=;\nbra W_%=;\nD_%=:\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

constexpr int STAGES = 4;
constexpr int STAGE_BYTES = 32768;

template <int MODE>
__global__ void __launch_bounds__(160, 1) stream_kernel(const char* __restrict__ src, int64_t chunks, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], MODE == 0 ? 128 : 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp < 4) {
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
      mbar_wait(&empty[stage], phase ^ 1);
      const char* g = src + c * STAGE_BYTES;
      uint32_t s = smem_u32(smem + stage * STAGE_BYTES);
      if (MODE == 0) {
#pragma unroll
        for (int i = 0; i < STAGE_BYTES / 16 / 128; ++i) {
          int off = (threadIdx.x + i * 128) * 16;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s + off), "l"(g + off) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[stage])) : "memory");
      } else if (threadIdx.x == 0) {
        mbar_expect_tx(&full[stage], STAGE_BYTES);
        constexpr int PIECE = MODE == 1 ? STAGE_BYTES : 64;  // MODE 2: 64-byte pieces
        for (int off = 0; off < STAGE_BYTES; off += PIECE)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s + off),
              "l"(g + off), "r"(PIECE), "r"(smem_u32(&full[stage]))
              : "memory");
      }
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    if (MODE == 0) asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (threadIdx.x == 128) {
    int stage = 0;
    uint32_t phase = 0;
    float acc = 0.f;
    for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
      mbar_wait(&full[stage], phase);
      acc += *reinterpret_cast<const float*>(smem + stage * STAGE_BYTES + (c & 255) * 4);
      mbar_arrive(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    out[blockIdx.x] = acc;
  }
}

int main() {
  const int64_t bytes = 1ll << 30;
  char* src;
  float* out;
  cudaMalloc(&src, bytes);
  cudaMalloc(&out, 4096);
  cudaMemset(src, 0, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t chunks = bytes / STAGE_BYTES;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * STAGE_BYTES);
    for (int w = 0; w < 3; ++w) kern<<<sms, 160, STAGES * STAGE_BYTES>>>(src, chunks, out);
    cudaEventRecord(e0);
    for (int w = 0; w < 10; ++w) kern<<<sms, 160, STAGES * STAGE_BYTES>>>(src, chunks, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-34s %8.1f GB/s  (%s)\n", name, 10.0 * bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  run(stream_kernel<0>, "cp.async 16B x128 thr, 4x32KB");
  run(stream_kernel<1>, "cp.async.bulk 32KB, 4x32KB");
  run(stream_kernel<2>, "cp.async.bulk 64B pieces, 4x32KB");
  return 0;
}
