// LayerNorm forward/backward (engine.layernorm_raw, engine.py:206-217):
//   y = (x - mean) / sqrt(var + eps) * gamma + beta,  var = population variance.
// HBM-bound: one warp per row with 16/8/4/2-byte vector loads for contiguous
// rows (x_cs == 1, cols % 32 == 0, cols <= 1024); one thread per row for the
// channel-major input of the triangle LN2 (x_cs != 1, coalesced across rows).
// Statistics and the gamma/beta reductions are fp32; dgamma/dbeta use a
// per-CTA shared-memory partial and one atomicAdd per column per CTA.
#include "common.cuh"

namespace evo {

template <typename T, int VPT>
__device__ __forceinline__ void load_row(const T* p, float* v) {
  // VPT consecutive elements starting at p (aligned to VPT*sizeof(T))
  if constexpr (sizeof(T) == 2 && VPT % 8 == 0) {
#pragma unroll
    for (int i = 0; i < VPT; i += 8) {
      uint4 u = *reinterpret_cast<const uint4*>(p + i);
      unpack_bf16x2(u.x, v[i], v[i + 1]);
      unpack_bf16x2(u.y, v[i + 2], v[i + 3]);
      unpack_bf16x2(u.z, v[i + 4], v[i + 5]);
      unpack_bf16x2(u.w, v[i + 6], v[i + 7]);
    }
  } else if constexpr (sizeof(T) == 2 && VPT % 4 == 0) {
#pragma unroll
    for (int i = 0; i < VPT; i += 4) {
      uint2 u = *reinterpret_cast<const uint2*>(p + i);
      unpack_bf16x2(u.x, v[i], v[i + 1]);
      unpack_bf16x2(u.y, v[i + 2], v[i + 3]);
    }
  } else if constexpr (sizeof(T) == 4 && VPT % 4 == 0) {
#pragma unroll
    for (int i = 0; i < VPT; i += 4) {
      float4 u = *reinterpret_cast<const float4*>(p + i);
      v[i] = u.x; v[i + 1] = u.y; v[i + 2] = u.z; v[i + 3] = u.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < VPT; ++i) v[i] = ldf<T>(p + i);
  }
}

template <typename T, int VPT>
__device__ __forceinline__ void store_row(T* p, const float* v) {
  if constexpr (sizeof(T) == 2 && VPT % 8 == 0) {
#pragma unroll
    for (int i = 0; i < VPT; i += 8) {
      uint4 u;
      u.x = pack_bf16x2(v[i], v[i + 1]);
      u.y = pack_bf16x2(v[i + 2], v[i + 3]);
      u.z = pack_bf16x2(v[i + 4], v[i + 5]);
      u.w = pack_bf16x2(v[i + 6], v[i + 7]);
      *reinterpret_cast<uint4*>(p + i) = u;
    }
  } else if constexpr (sizeof(T) == 2 && VPT % 4 == 0) {
#pragma unroll
    for (int i = 0; i < VPT; i += 4) {
      uint2 u;
      u.x = pack_bf16x2(v[i], v[i + 1]);
      u.y = pack_bf16x2(v[i + 2], v[i + 3]);
      *reinterpret_cast<uint2*>(p + i) = u;
    }
  } else if constexpr (sizeof(T) == 4 && VPT % 4 == 0) {
#pragma unroll
    for (int i = 0; i < VPT; i += 4)
      *reinterpret_cast<float4*>(p + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
  } else {
#pragma unroll
    for (int i = 0; i < VPT; ++i) stf<T>(p + i, v[i]);
  }
}

// ------------------------------------------------------------- contiguous rows, warp per row
// lane l owns columns [l*VPT, (l+1)*VPT)
template <typename TX, typename TY, int VPT, int K>
__global__ void __launch_bounds__(256) ln_fwd_warp(const TX* __restrict__ x, int64_t x_rs,
                                                   const float* __restrict__ gamma, const float* __restrict__ beta,
                                                   TY* __restrict__ y, float* __restrict__ mean_out,
                                                   float* __restrict__ rstd_out, int64_t rows, float eps,
                                                   const float* __restrict__ w, TY* __restrict__ dot_out,
                                                   int64_t dot_hs) {
  constexpr int COLS = VPT * 32;
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  float v[VPT];
  load_row<TX, VPT>(x + row * x_rs + lane * VPT, v);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) s += v[i];
  const float mu = warp_sum(s) * (1.0f / COLS);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    v[i] -= mu;
    q += v[i] * v[i];
  }
  const float rstd = rsqrtf(warp_sum(q) * (1.0f / COLS) + eps);
  float g[VPT], b[VPT];
  load_row<float, VPT>(gamma + lane * VPT, g);
  load_row<float, VPT>(beta + lane * VPT, b);
#pragma unroll
  for (int i = 0; i < VPT; ++i) v[i] = v[i] * rstd * g[i] + b[i];
  if (y) store_row<TY, VPT>(y + row * COLS + lane * VPT, v);
  if (lane == 0) {
    if (mean_out) mean_out[row] = mu;
    if (rstd_out) rstd_out[row] = rstd;
  }
  if constexpr (K > 0) {
    // fused per-row dot products with w[COLS, k] (msa_row_bias, evoformer.py:204-206)
#pragma unroll
    for (int h = 0; h < K; ++h) {
      float d = 0.f;
#pragma unroll
      for (int i = 0; i < VPT; ++i) d += v[i] * w[(lane * VPT + i) * K + h];
      d = warp_sum(d);
      if (lane == h) stf<TY>(dot_out + h * dot_hs + row, d);
    }
  }
}

// ------------------------------------------------------------- strided rows, thread per row
template <typename TX, typename TY, int MAXC>
__global__ void __launch_bounds__(256) ln_fwd_thread(const TX* __restrict__ x, int64_t x_rs, int64_t x_cs,
                                                     const float* __restrict__ gamma, const float* __restrict__ beta,
                                                     TY* __restrict__ y, float* __restrict__ mean_out,
                                                     float* __restrict__ rstd_out, int64_t rows, int cols,
                                                     float eps) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  float v[MAXC];
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < MAXC; ++c)
    if (c < cols) {
      v[c] = ldf<TX>(x + row * x_rs + c * x_cs);
      s += v[c];
    }
  const float mu = s / cols;
  float q = 0.f;
#pragma unroll
  for (int c = 0; c < MAXC; ++c)
    if (c < cols) {
      v[c] -= mu;
      q += v[c] * v[c];
    }
  const float rstd = rsqrtf(q / cols + eps);
#pragma unroll
  for (int c = 0; c < MAXC; ++c)
    if (c < cols) stf<TY>(y + row * cols + c, v[c] * rstd * gamma[c] + beta[c]);
  if (mean_out) mean_out[row] = mu;
  if (rstd_out) rstd_out[row] = rstd;
}

// ------------------------------------------------------------- backward
// dx = rstd * (g*dy - mean(g*dy) - xhat * mean(g*dy*xhat));  dgamma += dy*xhat; dbeta += dy
template <typename TD, typename TX, typename TO, int VPT>
__global__ void __launch_bounds__(256) ln_bwd_warp(const TD* __restrict__ dy, const TX* __restrict__ x, int64_t x_rs,
                                                   const float* __restrict__ gamma, const float* __restrict__ mean,
                                                   const float* __restrict__ rstd, TO* __restrict__ dx, int acc,
                                                   float* __restrict__ dgamma, float* __restrict__ dbeta,
                                                   int64_t rows) {
  constexpr int COLS = VPT * 32;
  extern __shared__ float red[];  // [2][COLS]
  for (int i = threadIdx.x; i < 2 * COLS; i += blockDim.x) red[i] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  float g[VPT];
  load_row<float, VPT>(gamma + lane * VPT, g);
  float dg[VPT], db[VPT];
#pragma unroll
  for (int i = 0; i < VPT; ++i) dg[i] = db[i] = 0.f;
  for (int64_t row = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); row < rows; row += (int64_t)gridDim.x * wpb) {
    float xv[VPT], d[VPT];
    load_row<TX, VPT>(x + row * x_rs + lane * VPT, xv);
    load_row<TD, VPT>(dy + row * COLS + lane * VPT, d);
    const float mu = mean[row], rs = rstd[row];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      xv[i] = (xv[i] - mu) * rs;  // xhat
      float gd = g[i] * d[i];
      s1 += gd;
      s2 += gd * xv[i];
      dg[i] += d[i] * xv[i];
      db[i] += d[i];
    }
    s1 = warp_sum(s1) * (1.0f / COLS);
    s2 = warp_sum(s2) * (1.0f / COLS);
    float o[VPT];
#pragma unroll
    for (int i = 0; i < VPT; ++i) o[i] = rs * (g[i] * d[i] - s1 - xv[i] * s2);
    TO* dp = dx + row * x_rs + lane * VPT;
    if (acc) {
      float prev[VPT];
      load_row<TO, VPT>(dp, prev);
#pragma unroll
      for (int i = 0; i < VPT; ++i) o[i] += prev[i];
    }
    store_row<TO, VPT>(dp, o);
  }
  if (dgamma || dbeta) {
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      atomicAdd(&red[lane * VPT + i], dg[i]);
      atomicAdd(&red[COLS + lane * VPT + i], db[i]);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < COLS; i += blockDim.x) {
      if (dgamma) atomicAdd(dgamma + i, red[i]);
      if (dbeta) atomicAdd(dbeta + i, red[COLS + i]);
    }
  }
}

template <typename TD, typename TX, typename TO, int MAXC>
__global__ void __launch_bounds__(256) ln_bwd_thread(const TD* __restrict__ dy, const TX* __restrict__ x, int64_t x_rs,
                                                     int64_t x_cs, const float* __restrict__ gamma,
                                                     const float* __restrict__ mean, const float* __restrict__ rstd,
                                                     TO* __restrict__ dx, int acc, float* __restrict__ dgamma,
                                                     float* __restrict__ dbeta, int64_t rows, int cols) {
  __shared__ float red[2 * MAXC];
  for (int i = threadIdx.x; i < 2 * MAXC; i += blockDim.x) red[i] = 0.f;
  __syncthreads();
  float dg[MAXC], db[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) dg[c] = db[c] = 0.f;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < rows;
       row += (int64_t)gridDim.x * blockDim.x) {
    float xh[MAXC], d[MAXC];
    const float mu = mean[row], rs = rstd[row];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
      if (c < cols) {
        xh[c] = (ldf<TX>(x + row * x_rs + c * x_cs) - mu) * rs;
        d[c] = ldf<TD>(dy + row * cols + c);
        float gd = gamma[c] * d[c];
        s1 += gd;
        s2 += gd * xh[c];
        dg[c] += d[c] * xh[c];
        db[c] += d[c];
      }
    s1 /= cols;
    s2 /= cols;
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
      if (c < cols) {
        TO* p = dx + row * x_rs + c * x_cs;
        float o = rs * (gamma[c] * d[c] - s1 - xh[c] * s2);
        if (acc) o += ldf<TO>(p);
        stf<TO>(p, o);
      }
  }
  if (dgamma || dbeta) {
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
      if (c < cols) {
        float a = warp_sum(dg[c]), b = warp_sum(db[c]);
        if ((threadIdx.x & 31) == 0) {
          atomicAdd(&red[c], a);
          atomicAdd(&red[MAXC + c], b);
        }
      }
    __syncthreads();
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {
      if (dgamma) atomicAdd(dgamma + c, red[c]);
      if (dbeta) atomicAdd(dbeta + c, red[MAXC + c]);
    }
  }
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}
int sm_count() { return num_sms(); }

template <typename TX, typename TY, int K>
static int ln_fwd_dispatch_warp(const void* x, int64_t x_rs, const float* g, const float* b, void* y, float* mean,
                                float* rstd, int64_t rows, int64_t cols, float eps, const float* w, void* dot,
                                int64_t dot_hs, cudaStream_t st) {
  const int wpb = 8;
  dim3 grid((unsigned)((rows + wpb - 1) / wpb));
#define LNF(VPT)                                                                                             \
  ln_fwd_warp<TX, TY, VPT, K><<<grid, wpb * 32, 0, st>>>((const TX*)x, x_rs, g, b, (TY*)y, mean, rstd, rows, \
                                                         eps, w, (TY*)dot, dot_hs)
  switch (cols) {
    case 32: LNF(1); break;
    case 64: LNF(2); break;
    case 128: LNF(4); break;
    case 256: LNF(8); break;
    case 384: LNF(12); break;
    case 512: LNF(16); break;
    case 768: LNF(24); break;
    case 1024: LNF(32); break;
    default: set_error("layernorm: unsupported contiguous width %lld", (long long)cols); return EVO_ERR_SHAPE;
  }
#undef LNF
  EVO_LAUNCH_CHECK("layernorm fwd");
  return EVO_OK;
}

}  // namespace evo

using namespace evo;

#define DT2(xd, yd, F, ...)                                                  \
  ((xd) == EVO_BF16 ? ((yd) == EVO_BF16 ? F<bf16, bf16>(__VA_ARGS__) : F<bf16, float>(__VA_ARGS__)) \
                    : ((yd) == EVO_BF16 ? F<float, bf16>(__VA_ARGS__) : F<float, float>(__VA_ARGS__)))

template <typename TX, typename TY>
static int ln_fwd_impl(const void* x, int64_t x_rs, int64_t x_cs, const float* g, const float* b, void* y,
                       float* mean, float* rstd, int64_t rows, int64_t cols, float eps, cudaStream_t st) {
  if (x_cs == 1 && cols % 32 == 0 && cols <= 1024) {
    EVO_CHECK_ARG(((uintptr_t)x & 15) == 0 && (x_rs % 8) == 0, EVO_ERR_ALIGN, "layernorm: x must be 16B aligned");
    return ln_fwd_dispatch_warp<TX, TY, 0>(x, x_rs, g, b, y, mean, rstd, rows, cols, eps, nullptr, nullptr, 0, st);
  }
  EVO_CHECK_ARG(cols <= 64, EVO_ERR_SHAPE, "layernorm: strided rows support cols <= 64 (got %lld)", (long long)cols);
  dim3 grid((unsigned)((rows + 255) / 256));
  ln_fwd_thread<TX, TY, 64><<<grid, 256, 0, st>>>((const TX*)x, x_rs, x_cs, g, b, (TY*)y, mean, rstd, rows,
                                                  (int)cols, eps);
  EVO_LAUNCH_CHECK("layernorm fwd strided");
  return EVO_OK;
}

extern "C" int evo_layernorm_fwd(const void* x, int x_dtype, int64_t x_rs, int64_t x_cs, const float* gamma,
                                 const float* beta, void* y, int y_dtype, float* mean, float* rstd, int64_t rows,
                                 int64_t cols, float eps, void* stream) {
  EVO_CHECK_ARG(x && gamma && beta && y, EVO_ERR_ARG, "layernorm: null pointer");
  EVO_CHECK_ARG(rows >= 0 && cols >= 1, EVO_ERR_SHAPE, "layernorm: bad extents");
  if (rows == 0) return EVO_OK;
  return DT2(x_dtype, y_dtype, ln_fwd_impl, x, x_rs, x_cs, gamma, beta, y, mean, rstd, rows, cols, eps,
             (cudaStream_t)stream);
}

extern "C" int evo_layernorm_rowdot_fwd(const void* x, int x_dtype, const float* gamma, const float* beta,
                                        const float* w, int k, void* out, int out_dtype, int64_t out_hs,
                                        void* ln_out, float* mean, float* rstd, int64_t rows, int64_t cols, float eps,
                                        void* stream) {
  EVO_CHECK_ARG(x && gamma && beta && w && out, EVO_ERR_ARG, "layernorm_rowdot: null pointer");
  EVO_CHECK_ARG(k >= 1 && k <= 16 && cols % 32 == 0 && cols <= 1024, EVO_ERR_SHAPE,
                "layernorm_rowdot: need 1<=k<=16 and cols %% 32 == 0, <= 1024");
  EVO_CHECK_ARG(x_dtype == out_dtype, EVO_ERR_DTYPE, "layernorm_rowdot: x and out dtype must match");
  EVO_CHECK_ARG(((uintptr_t)x & 15) == 0, EVO_ERR_ALIGN, "layernorm_rowdot: x must be 16B aligned");
  cudaStream_t st = (cudaStream_t)stream;
  if (rows == 0) return EVO_OK;
#define RD(KK)                                                                                                   \
  (x_dtype == EVO_BF16 ? ln_fwd_dispatch_warp<bf16, bf16, KK>(x, cols, gamma, beta, ln_out, mean, rstd, rows,   \
                                                               cols, eps, w, out, out_hs, st)                   \
                       : ln_fwd_dispatch_warp<float, float, KK>(x, cols, gamma, beta, ln_out, mean, rstd, rows, \
                                                                cols, eps, w, out, out_hs, st))
  switch (k) {
    case 1: return RD(1);
    case 2: return RD(2);
    case 4: return RD(4);
    case 8: return RD(8);
    case 16: return RD(16);
    default: break;
  }
#undef RD
  set_error("layernorm_rowdot: k must be 1, 2, 4, 8 or 16 (got %d)", k);
  return EVO_ERR_SHAPE;
}

template <typename TD, typename TX, typename TO>
static int ln_bwd_impl(const void* dy, const void* x, int64_t x_rs, int64_t x_cs, const float* g, const float* mean,
                       const float* rstd, void* dx, int acc, float* dg, float* db, int64_t rows, int64_t cols,
                       cudaStream_t st) {
  const int grid_max = sm_count() * 8;
  if (x_cs == 1 && cols % 32 == 0 && cols <= 1024) {
    const int wpb = 8;
    int64_t need = (rows + wpb - 1) / wpb;
    dim3 grid((unsigned)(need < grid_max ? need : grid_max));
    size_t sm = 2 * cols * sizeof(float);
#define LNB(VPT)                                                                                            \
  ln_bwd_warp<TD, TX, TO, VPT><<<grid, wpb * 32, sm, st>>>((const TD*)dy, (const TX*)x, x_rs, g, mean, rstd, \
                                                           (TO*)dx, acc, dg, db, rows)
    switch (cols) {
      case 32: LNB(1); break;
      case 64: LNB(2); break;
      case 128: LNB(4); break;
      case 256: LNB(8); break;
      case 384: LNB(12); break;
      case 512: LNB(16); break;
      case 768: LNB(24); break;
      case 1024: LNB(32); break;
      default: return EVO_ERR_SHAPE;
    }
#undef LNB
    EVO_LAUNCH_CHECK("layernorm bwd");
    return EVO_OK;
  }
  EVO_CHECK_ARG(cols <= 64, EVO_ERR_SHAPE, "layernorm bwd: strided rows support cols <= 64");
  int64_t need = (rows + 255) / 256;
  dim3 grid((unsigned)(need < grid_max ? need : grid_max));
  ln_bwd_thread<TD, TX, TO, 64><<<grid, 256, 0, st>>>((const TD*)dy, (const TX*)x, x_rs, x_cs, g, mean, rstd,
                                                      (TO*)dx, acc, dg, db, rows, (int)cols);
  EVO_LAUNCH_CHECK("layernorm bwd strided");
  return EVO_OK;
}

extern "C" int evo_layernorm_bwd(const void* dy, int dy_dtype, const void* x, int x_dtype, int64_t x_rs, int64_t x_cs,
                                 const float* gamma, const float* mean, const float* rstd, void* dx, int dx_dtype,
                                 int accumulate_dx, float* dgamma, float* dbeta, int64_t rows, int64_t cols,
                                 void* stream) {
  EVO_CHECK_ARG(dy && x && gamma && mean && rstd && dx, EVO_ERR_ARG, "layernorm bwd: null pointer");
  if (rows == 0) return EVO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  EVO_CHECK_ARG(x_dtype == dx_dtype, EVO_ERR_DTYPE, "layernorm bwd: x and dx dtypes must match");
  if (dy_dtype == EVO_BF16) {
    if (x_dtype == EVO_BF16)
      return ln_bwd_impl<bf16, bf16, bf16>(dy, x, x_rs, x_cs, gamma, mean, rstd, dx, accumulate_dx, dgamma, dbeta,
                                           rows, cols, st);
    return ln_bwd_impl<bf16, float, float>(dy, x, x_rs, x_cs, gamma, mean, rstd, dx, accumulate_dx, dgamma, dbeta,
                                           rows, cols, st);
  }
  if (x_dtype == EVO_BF16)
    return ln_bwd_impl<float, bf16, bf16>(dy, x, x_rs, x_cs, gamma, mean, rstd, dx, accumulate_dx, dgamma, dbeta,
                                          rows, cols, st);
  return ln_bwd_impl<float, float, float>(dy, x, x_rs, x_cs, gamma, mean, rstd, dx, accumulate_dx, dgamma, dbeta,
                                          rows, cols, st);
}
