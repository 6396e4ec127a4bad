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
  pdl_wait();
  static_assert(K == 0, "fused row dots live in ln_rowdot_fwd");
  constexpr int COLS = VPT * 32;
  constexpr int U = VPT <= 8 ? 2 : 1;  // rows in flight per warp
  const int lane = threadIdx.x & 31;
  float g[VPT], b[VPT];
  load_row<float, VPT>(gamma + lane * VPT, g);
  load_row<float, VPT>(beta + lane * VPT, b);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t rb = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * U; rb < rows; rb += nw * U) {
    float v[U][VPT];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (rb + u < rows) load_row<TX, VPT>(x + (rb + u) * x_rs + lane * VPT, v[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = rb + u;
      if (row >= rows) break;
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < VPT; ++i) s += v[u][i];
      const float mu = warp_sum(s) * (1.0f / COLS);
      float q = 0.f;
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        v[u][i] -= mu;
        q += v[u][i] * v[u][i];
      }
      const float rstd = rsqrtf(warp_sum(q) * (1.0f / COLS) + eps);
#pragma unroll
      for (int i = 0; i < VPT; ++i) v[u][i] = v[u][i] * rstd * g[i] + b[i];
      if (y) store_row<TY, VPT>(y + row * COLS + lane * VPT, v[u]);
      if (lane == 0) {
        if (mean_out) mean_out[row] = mu;
        if (rstd_out) rstd_out[row] = rstd;
      }
    }
  }
}

// ------------------------------------------------------------- LN + k row dots (msa_row_bias)
// Sum of K per-lane partials across the 32 lanes with a transposing butterfly:
// after the xor-16/8/4 steps each lane holds 1 of the K=8 sums (K/8 per lane for
// larger K), 9 shuffles instead of 5*K.  Returns the sum for head  (lane >> 2) & 7.
template <int K>
__device__ __forceinline__ float butterfly_sum8(float* v, int lane) {
  static_assert(K == 8, "butterfly for 8 heads");
  // step 16: keep heads [0,4) on lanes < 16, [4,8) on lanes >= 16
  const bool up16 = lane & 16;
  float a[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = up16 ? v[i] : v[4 + i];
    const float recv = __shfl_xor_sync(0xffffffffu, send, 16);
    a[i] = (up16 ? v[4 + i] : v[i]) + recv;
  }
  const bool up8 = lane & 8;
  float b2[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = up8 ? a[i] : a[2 + i];
    const float recv = __shfl_xor_sync(0xffffffffu, send, 8);
    b2[i] = (up8 ? a[2 + i] : a[i]) + recv;
  }
  const bool up4 = lane & 4;
  const float send = up4 ? b2[0] : b2[1];
  float c = (up4 ? b2[1] : b2[0]) + __shfl_xor_sync(0xffffffffu, send, 4);
  c += __shfl_xor_sync(0xffffffffu, c, 2);
  c += __shfl_xor_sync(0xffffffffu, c, 1);
  return c;  // head = ((lane>>4)&1)*4 + ((lane>>3)&1)*2 + ((lane>>2)&1)
}

// one warp per row, persistent over rows (w cached in registers); K <= 8 heads
// (padded), output out[h * out_hs + row]
template <typename TX, int VPT>
__global__ void __launch_bounds__(256) ln_rowdot_fwd(const TX* __restrict__ x, const float* __restrict__ gamma,
                                                     const float* __restrict__ beta, const float* __restrict__ w,
                                                     TX* __restrict__ out, int64_t out_hs, TX* __restrict__ ln_out,
                                                     float* __restrict__ mean_out, float* __restrict__ rstd_out,
                                                     int64_t rows, float eps) {
  pdl_wait();
  constexpr int COLS = VPT * 32, K = 8;
  const int lane = threadIdx.x & 31;
  float g[VPT], bt[VPT], wr[VPT][K];
  load_row<float, VPT>(gamma + lane * VPT, g);
  load_row<float, VPT>(beta + lane * VPT, bt);
#pragma unroll
  for (int i = 0; i < VPT; ++i)
#pragma unroll
    for (int h = 0; h < K; ++h) wr[i][h] = w[(lane * VPT + i) * K + h];
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows; row += wstride) {
    float v[VPT];
    load_row<TX, VPT>(x + row * COLS + lane * VPT, v);
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
    const float rs = rsqrtf(warp_sum(q) * (1.0f / COLS) + eps);
#pragma unroll
    for (int i = 0; i < VPT; ++i) v[i] = v[i] * rs * g[i] + bt[i];
    if (ln_out) store_row<TX, VPT>(ln_out + row * COLS + lane * VPT, v);
    if (lane == 0 && mean_out) {
      mean_out[row] = mu;
      rstd_out[row] = rs;
    }
    float d[K];
#pragma unroll
    for (int h = 0; h < K; ++h) {
      d[h] = 0.f;
#pragma unroll
      for (int i = 0; i < VPT; ++i) d[h] += v[i] * wr[i][h];
    }
    const float r = butterfly_sum8<K>(d, lane);
    if ((lane & 3) == 0) {
      const int h = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
      stf<TX>(out + h * out_hs + row, r);
    }
  }
}

// backward of LN + row dots, fused: dy = w . dout_row; dW += LN(x) dout^T; LN backward
// into dx (dx = res + dLN, res may alias dx); dgamma/dbeta/dW: CTA partials + one
// atomic per element per CTA.
template <typename TX, int VPT>
__global__ void __launch_bounds__(256) ln_rowdot_bwd(const TX* __restrict__ x, const float* __restrict__ gamma,
                                                     const float* __restrict__ beta, const float* __restrict__ w,
                                                     const float* __restrict__ dout, int64_t out_hs,
                                                     const float* __restrict__ mean, const float* __restrict__ rstd,
                                                     const TX* res, TX* dx, float* __restrict__ dgamma,
                                                     float* __restrict__ dbeta, float* __restrict__ dw,
                                                     int64_t rows) {
  pdl_wait();
  constexpr int COLS = VPT * 32, K = 8;
  __shared__ float red[8][COLS * (2 + K) / 8 + 1];  // per-warp partials, flushed in column slices
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float g[VPT], bt[VPT], wr[VPT][K];
  load_row<float, VPT>(gamma + lane * VPT, g);
  load_row<float, VPT>(beta + lane * VPT, bt);
#pragma unroll
  for (int i = 0; i < VPT; ++i)
#pragma unroll
    for (int h = 0; h < K; ++h) wr[i][h] = w[(lane * VPT + i) * K + h];
  float dg[VPT], db[VPT], dwa[VPT][K];
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    dg[i] = db[i] = 0.f;
#pragma unroll
    for (int h = 0; h < K; ++h) dwa[i][h] = 0.f;
  }
  const int64_t slab = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * slab, r1 = r0 + slab < rows ? r0 + slab : rows;
  for (int64_t row = r0 + wid; row < r1; row += 8) {
    float xv[VPT];
    load_row<TX, VPT>(x + row * COLS + lane * VPT, xv);
    const float mu = mean[row], rs = rstd[row];
    float dh[K];
#pragma unroll
    for (int h = 0; h < K; ++h) dh[h] = dout[h * out_hs + row];
    float d[VPT], s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      xv[i] = (xv[i] - mu) * rs;  // xhat
      const float lnv = xv[i] * g[i] + bt[i];
      d[i] = 0.f;
#pragma unroll
      for (int h = 0; h < K; ++h) {
        d[i] += dh[h] * wr[i][h];
        dwa[i][h] += lnv * dh[h];
      }
      const float gd = g[i] * d[i];
      s1 += gd;
      s2 += gd * xv[i];
      dg[i] += d[i] * xv[i];
      db[i] += d[i];
    }
    s1 = warp_sum(s1) * (1.0f / COLS);
    s2 = warp_sum(s2) * (1.0f / COLS);
    float o[VPT];
    if (res) load_row<TX, VPT>(res + row * COLS + lane * VPT, o);
#pragma unroll
    for (int i = 0; i < VPT; ++i) o[i] = (res ? o[i] : 0.f) + rs * (g[i] * d[i] - s1 - xv[i] * s2);
    store_row<TX, VPT>(dx + row * COLS + lane * VPT, o);
  }
  // CTA reduction: dgamma, dbeta, dW (COLS * (2 + K) values), 8 warps
  constexpr int NV = COLS * (2 + K);
  float* flat = &red[0][0];
  constexpr int PITCH = COLS * (2 + K) / 8 + 1;
  for (int base = 0; base < NV; base += NV / 8) {
    // each warp deposits its values of slice [base, base + NV/8)
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int c = lane * VPT + i;
      const int idx[2] = {c, COLS + c};
      const float val[2] = {dg[i], db[i]};
#pragma unroll
      for (int t = 0; t < 2; ++t)
        if (idx[t] >= base && idx[t] < base + NV / 8) flat[wid * PITCH + idx[t] - base] = val[t];
#pragma unroll
      for (int h = 0; h < K; ++h) {
        const int id = 2 * COLS + c * K + h;
        if (id >= base && id < base + NV / 8) flat[wid * PITCH + id - base] = dwa[i][h];
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < NV / 8; t += blockDim.x) {
      float acc = 0.f;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) acc += flat[ww * PITCH + t];
      const int id = base + t;
      if (id < COLS) atomicAdd(dgamma + id, acc);
      else if (id < 2 * COLS) atomicAdd(dbeta + id - COLS, acc);
      else atomicAdd(dw + (id - 2 * COLS), acc);
    }
    __syncthreads();
  }
}


// ------------------------------------------------------------- lane-group rows (16-byte lanes)
// Every lane owns 8 consecutive channels (one 16-byte bf16 vector); a row is handled by
// LPR = COLS/8 lanes (4..32), so a warp covers 32/LPR rows per step and every load moves
// 16 bytes per lane.  Reductions are xor-shuffles within the lane group.
template <int LPR>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename TX, typename TY, int COLS, int U>
__global__ void __launch_bounds__(256) ln_fwd_grp(const TX* __restrict__ x, int64_t x_rs,
                                                  const float* __restrict__ gamma, const float* __restrict__ beta,
                                                  TY* __restrict__ y, float* __restrict__ mean_out,
                                                  float* __restrict__ rstd_out, int64_t rows, float eps) {
  pdl_wait();
  constexpr int LPR = COLS / 8, RPW = 32 / LPR;  // lanes per row, rows per warp step
  const int lane = threadIdx.x & 31, sub = lane / LPR, cl = (lane % LPR) * 8;
  float g[8], b[8];
  load_row<float, 8>(gamma + cl, g);
  load_row<float, 8>(beta + cl, b);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t rb = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * RPW * U; rb < rows;
       rb += nw * RPW * U) {
    float v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = rb + u * RPW + sub;
      if (row < rows) load_row<TX, 8>(x + row * x_rs + cl, v[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = rb + u * RPW + sub;
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) s += v[u][i];
      const float mu = group_sum<LPR>(s) * (1.0f / COLS);
      float q = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v[u][i] -= mu;
        q += v[u][i] * v[u][i];
      }
      const float rs = rsqrtf(group_sum<LPR>(q) * (1.0f / COLS) + eps);
      if (row < rows) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[u][i] = v[u][i] * rs * g[i] + b[i];
        if (y) store_row<TY, 8>(y + row * COLS + cl, v[u]);
        if (cl == 0 && mean_out) {
          mean_out[row] = mu;
          rstd_out[row] = rs;
        }
      }
    }
  }
}

// 8 consecutive elements kept as raw bits until used (bf16: one 16-byte register quad), so
// U row-groups of x, dy and res can be in flight without spilling the unpacked floats.
template <typename T> struct Raw8;
template <> struct Raw8<bf16> {
  uint4 u;
  __device__ __forceinline__ void load(const bf16* p) { u = *reinterpret_cast<const uint4*>(p); }
  __device__ __forceinline__ void zero() { u = make_uint4(0, 0, 0, 0); }
  __device__ __forceinline__ void get(float* v) const {
    unpack_bf16x2(u.x, v[0], v[1]); unpack_bf16x2(u.y, v[2], v[3]);
    unpack_bf16x2(u.z, v[4], v[5]); unpack_bf16x2(u.w, v[6], v[7]);
  }
};
template <> struct Raw8<float> {
  float4 a, b;
  __device__ __forceinline__ void load(const float* p) {
    a = *reinterpret_cast<const float4*>(p);
    b = *reinterpret_cast<const float4*>(p + 4);
  }
  __device__ __forceinline__ void zero() { a = b = make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ __forceinline__ void get(float* v) const {
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
};

#ifndef LNF_PIPE
#define LNF_PIPE 1
#endif
// ln_fwd_grp with a software pipeline: the raw 16-byte loads of the lane's next U row groups are issued
// before this step's statistics and stores, so the loads of consecutive steps overlap
template <typename TX, typename TY, int COLS, int U>
__global__ void __launch_bounds__(256) ln_fwd_grp_pipe(const TX* __restrict__ x, int64_t x_rs,
                                                       const float* __restrict__ gamma, const float* __restrict__ beta,
                                                       TY* __restrict__ y, float* __restrict__ mean_out,
                                                       float* __restrict__ rstd_out, int64_t rows, float eps) {
  pdl_wait();
  constexpr int LPR = COLS / 8, RPW = 32 / LPR;
  const int lane = threadIdx.x & 31, sub = lane / LPR, cl = (lane % LPR) * 8;
  float g[8], b[8];
  load_row<float, 8>(gamma + cl, g);
  load_row<float, 8>(beta + cl, b);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5), step = nw * RPW * U;
  Raw8<TX> nx[U];
  auto load = [&](int64_t rb_) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = rb_ + u * RPW + sub;
      if (row < rows) nx[u].load(x + row * x_rs + cl); else nx[u].zero();
    }
  };
  int64_t rb = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * RPW * U;
  if (rb < rows) load(rb);
  for (; rb < rows; rb += step) {
    float v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) nx[u].get(v[u]);
    if (rb + step < rows) load(rb + step);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = rb + u * RPW + sub;
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) s += v[u][i];
      const float mu = group_sum<LPR>(s) * (1.0f / COLS);
      float q = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v[u][i] -= mu;
        q += v[u][i] * v[u][i];
      }
      const float rs = rsqrtf(group_sum<LPR>(q) * (1.0f / COLS) + eps);
      if (row < rows) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[u][i] = v[u][i] * rs * g[i] + b[i];
        if (y) store_row<TY, 8>(y + row * COLS + cl, v[u]);
        if (cl == 0 && mean_out) {
          mean_out[row] = mu;
          rstd_out[row] = rs;
        }
      }
    }
  }
}


// LPR = COLS/8 lanes per row, each owning 8 channels; a CTA walks one contiguous slab of
// rows, U row-groups per warp step with every load of the step issued before any math.
// <= 128 registers (2 CTAs = 16 warps per SM) keep ~100 KB of loads in flight per SM.
// dsum (optional): column sums of the written dx, i.e. the bias gradient of the module that
// consumes this residual-stream gradient (fused here instead of a separate colsum pass).
template <typename TD, typename TX, typename TO, int COLS, int U>
__global__ void __launch_bounds__(256, 2) ln_bwd_grp(const TD* __restrict__ dy, const TX* __restrict__ x, int64_t x_rs,
                                                     const float* __restrict__ gamma, const float* __restrict__ mean,
                                                     const float* __restrict__ rstd, TO* dx, const TO* res,
                                                     float* __restrict__ dgamma, float* __restrict__ dbeta,
                                                     float* __restrict__ dsum, int64_t rows) {
  pdl_wait();
  constexpr int LPR = COLS / 8, RPW = 32 / LPR;
  __shared__ float red[8][3][COLS];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, sub = lane / LPR, cl = (lane % LPR) * 8;
  float g[8], dg[8], db[8], ds[8];
  load_row<float, 8>(gamma + cl, g);
#pragma unroll
  for (int i = 0; i < 8; ++i) dg[i] = db[i] = ds[i] = 0.f;
  const int64_t slab = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * slab, r1 = r0 + slab < rows ? r0 + slab : rows;
  for (int64_t rb = r0 + wid * RPW * U; rb < r1; rb += 8 * RPW * U) {
    Raw8<TX> rx[U];
    Raw8<TD> rd[U];
    Raw8<TO> rr[U];
    float mu[U], rs[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = rb + u * RPW + sub;
      if (row < r1) {
        rx[u].load(x + row * x_rs + cl);
        rd[u].load(dy + row * COLS + cl);
        if (res) rr[u].load(res + row * x_rs + cl);
        mu[u] = mean[row];
        rs[u] = rstd[row];
      } else {
        rx[u].zero();
        rd[u].zero();
        mu[u] = rs[u] = 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = rb + u * RPW + sub;
      float xv[8], d[8];
      rx[u].get(xv);
      rd[u].get(d);
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        xv[i] = (xv[i] - mu[u]) * rs[u];  // xhat
        const float gd = g[i] * d[i];
        s1 += gd;
        s2 += gd * xv[i];
        dg[i] += d[i] * xv[i];
        db[i] += d[i];
      }
      s1 = group_sum<LPR>(s1) * (1.0f / COLS);
      s2 = group_sum<LPR>(s2) * (1.0f / COLS);
      if (row < r1) {
        float o[8];
        if (res) rr[u].get(o);
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = (res ? o[i] : 0.f) + rs[u] * (g[i] * d[i] - s1 - xv[i] * s2);
        store_row<TO, 8>(dx + row * x_rs + cl, o);
        if (dsum) {
#pragma unroll
          for (int i = 0; i < 8; ++i) ds[i] += o[i];
        }
      }
    }
  }
  if (dgamma || dbeta || dsum) {
    // lanes of different row-groups hold partials of the same channels: fold them first
#pragma unroll
    for (int i = 0; i < 8; ++i) {
#pragma unroll
      for (int o = LPR; o < 32; o <<= 1) {
        dg[i] += __shfl_xor_sync(0xffffffffu, dg[i], o);
        db[i] += __shfl_xor_sync(0xffffffffu, db[i], o);
        ds[i] += __shfl_xor_sync(0xffffffffu, ds[i], o);
      }
    }
    if (sub == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        red[wid][0][cl + i] = dg[i];
        red[wid][1][cl + i] = db[i];
        red[wid][2][cl + i] = ds[i];
      }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < COLS; c += blockDim.x) {
      float a = 0.f, b = 0.f, e = 0.f;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) {
        a += red[ww][0][c];
        b += red[ww][1][c];
        e += red[ww][2][c];
      }
      if (dgamma) atomicAdd(dgamma + c, a);
      if (dbeta) atomicAdd(dbeta + c, b);
      if (dsum) atomicAdd(dsum + c, e);
    }
  }
}

// ------------------------------------------------------------- channel-major rows, tiled
// x channel-major (element (r, c) at x[c * x_cs + r], the triangle update's t[p][i][j]): a CTA stages
// a [C][128-row] tile with 16-byte loads (every byte of the tile in flight at once, unlike a
// thread-per-row kernel's 2-byte strided loads), one thread per row computes from shared memory,
// and the row-major output tile leaves as contiguous 16-byte chunks.
constexpr int CM_RT = 128;  // rows per CTA (one per thread)

template <int C>
__device__ __forceinline__ void cm_load_tile(bf16 (*xs)[CM_RT + 8], const bf16* __restrict__ x, int64_t x_cs,
                                             int64_t r0, int nr) {
  for (int i = threadIdx.x; i < C * CM_RT / 8; i += CM_RT) {
    const int c = i / (CM_RT / 8), r8 = (i % (CM_RT / 8)) * 8;
    const bf16* src = x + c * x_cs + r0 + r8;
    if (r8 + 8 <= nr) {
      *reinterpret_cast<uint4*>(&xs[c][r8]) = *reinterpret_cast<const uint4*>(src);
    } else {
      for (int e = 0; e < 8; ++e) xs[c][r8 + e] = r8 + e < nr ? src[e] : __float2bfloat16(0.f);
    }
  }
}

template <int C>
__global__ void __launch_bounds__(CM_RT) ln_fwd_cm(const bf16* __restrict__ x, int64_t x_cs,
                                                   const float* __restrict__ gamma, const float* __restrict__ beta,
                                                   bf16* __restrict__ y, float* __restrict__ mean_out,
                                                   float* __restrict__ rstd_out, int64_t rows, float eps) {
  pdl_wait();
  __shared__ __align__(16) bf16 xs[C][CM_RT + 8];
  __shared__ __align__(16) bf16 ys[CM_RT][C + 8];
  const int t = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * CM_RT;
  const int nr = rows - r0 < CM_RT ? (int)(rows - r0) : CM_RT;
  cm_load_tile<C>(xs, x, x_cs, r0, nr);
  __syncthreads();
  if (t < nr) {
    float v[C];
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      v[c] = __bfloat162float(xs[c][t]);
      s += v[c];
    }
    const float mu = s * (1.0f / C);
    float q = 0.f;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      v[c] -= mu;
      q += v[c] * v[c];
    }
    const float rs = rsqrtf(q * (1.0f / C) + eps);
#pragma unroll
    for (int c = 0; c < C; c += 8) {
      float o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = v[c + e] * rs * gamma[c + e] + beta[c + e];
      uint4 u;
      u.x = pack_bf16x2(o[0], o[1]); u.y = pack_bf16x2(o[2], o[3]);
      u.z = pack_bf16x2(o[4], o[5]); u.w = pack_bf16x2(o[6], o[7]);
      *reinterpret_cast<uint4*>(&ys[t][c]) = u;
    }
    if (mean_out) mean_out[r0 + t] = mu;
    if (rstd_out) rstd_out[r0 + t] = rs;
  }
  __syncthreads();
  for (int i = t; i < nr * (C / 8); i += CM_RT) {
    const int r = i / (C / 8), c8 = (i % (C / 8)) * 8;
    *reinterpret_cast<uint4*>(y + (r0 + r) * C + c8) = *reinterpret_cast<const uint4*>(&ys[r][c8]);
  }
}

// backward: dy row-major [rows][C], x / dx / res channel-major; dgamma / dbeta per CTA + atomics
template <int C>
__global__ void __launch_bounds__(CM_RT) ln_bwd_cm(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                                                   int64_t x_cs, const float* __restrict__ gamma,
                                                   const float* __restrict__ mean, const float* __restrict__ rstd,
                                                   bf16* dx, const bf16* res, float* __restrict__ dgamma,
                                                   float* __restrict__ dbeta, int64_t rows) {
  pdl_wait();
  __shared__ __align__(16) bf16 xs[C][CM_RT + 8];   // x, then dx (channel-major)
  __shared__ __align__(16) bf16 ds[CM_RT][C + 8];   // dy (row-major)
  __shared__ float red[C][CM_RT + 1];                // per-row dgamma / dbeta terms, summed per channel
  const int t = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * CM_RT;
  const int nr = rows - r0 < CM_RT ? (int)(rows - r0) : CM_RT;
  cm_load_tile<C>(xs, x, x_cs, r0, nr);
  for (int i = t; i < nr * (C / 8); i += CM_RT) {
    const int r = i / (C / 8), c8 = (i % (C / 8)) * 8;
    *reinterpret_cast<uint4*>(&ds[r][c8]) = *reinterpret_cast<const uint4*>(dy + (r0 + r) * C + c8);
  }
  __syncthreads();
  float dg[C], db[C];
#pragma unroll
  for (int c = 0; c < C; ++c) dg[c] = db[c] = 0.f;
  if (t < nr) {
    const float mu = mean[r0 + t], rs = rstd[r0 + t];
    float xh[C], d[C], s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int c = 0; c < C; c += 8) {
      const uint4 u = *reinterpret_cast<const uint4*>(&ds[t][c]);
      unpack_bf16x2(u.x, d[c], d[c + 1]); unpack_bf16x2(u.y, d[c + 2], d[c + 3]);
      unpack_bf16x2(u.z, d[c + 4], d[c + 5]); unpack_bf16x2(u.w, d[c + 6], d[c + 7]);
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
      xh[c] = (__bfloat162float(xs[c][t]) - mu) * rs;
      const float gd = gamma[c] * d[c];
      s1 += gd;
      s2 += gd * xh[c];
      dg[c] = d[c] * xh[c];
      db[c] = d[c];
    }
    s1 *= 1.0f / C;
    s2 *= 1.0f / C;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      float o = rs * (gamma[c] * d[c] - s1 - xh[c] * s2);
      if (res) o += __bfloat162float(res[c * x_cs + r0 + t]);
      xs[c][t] = __float2bfloat16(o);  // own column of the tile: no barrier needed before the write
    }
  }
  // (dgamma / dbeta: one smem transpose per term instead of 2 C warp reductions per warp)
  if (dgamma) {
#pragma unroll
    for (int c = 0; c < C; ++c) red[c][t] = dg[c];
  }
  __syncthreads();
  float sum_g = 0.f;
  if (dgamma && t < C) {
    for (int k = 0; k < nr; ++k) sum_g += red[t][k];
  }
  __syncthreads();
  if (dbeta) {
#pragma unroll
    for (int c = 0; c < C; ++c) red[c][t] = db[c];
  }
  __syncthreads();
  for (int i = t; i < C * CM_RT / 8; i += CM_RT) {
    const int c = i / (CM_RT / 8), r8 = (i % (CM_RT / 8)) * 8;
    bf16* dst = dx + c * x_cs + r0 + r8;
    if (r8 + 8 <= nr) {
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(&xs[c][r8]);
    } else {
      for (int e = 0; r8 + e < nr; ++e) dst[e] = xs[c][r8 + e];
    }
  }
  if (t < C) {
    if (dgamma) atomicAdd(dgamma + t, sum_g);
    if (dbeta) {
      float b = 0.f;
      for (int k = 0; k < nr; ++k) b += red[t][k];
      atomicAdd(dbeta + t, b);
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
  pdl_wait();
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
  if (sizeof(TY) == 2 && MAXC % 8 == 0 && cols == MAXC) {
    // the row-major output row (MAXC bf16) as 16-byte stores instead of MAXC 2-byte ones
#pragma unroll
    for (int c = 0; c < MAXC; c += 8) {
      float o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = v[c + e] * rstd * gamma[c + e] + beta[c + e];
      store_row<TY, 8>(y + row * cols + c, o);
    }
  } else {
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
      if (c < cols) stf<TY>(y + row * cols + c, v[c] * rstd * gamma[c] + beta[c]);
  }
  if (mean_out) mean_out[row] = mu;
  if (rstd_out) rstd_out[row] = rstd;
}

// ------------------------------------------------------------- backward
// dx = rstd * (g*dy - mean(g*dy) - xhat * mean(g*dy*xhat));  dgamma += dy*xhat; dbeta += dy
template <typename TD, typename TX, typename TO, int VPT>
__global__ void __launch_bounds__(256) ln_bwd_warp(const TD* __restrict__ dy, const TX* __restrict__ x, int64_t x_rs,
                                                   const float* __restrict__ gamma, const float* __restrict__ mean,
                                                   const float* __restrict__ rstd, TO* dx, const TO* res,
                                                   float* __restrict__ dgamma, float* __restrict__ dbeta,
                                                   int64_t rows) {
  pdl_wait();
  constexpr int COLS = VPT * 32;
  extern __shared__ float red[];  // [8 warps][2][COLS]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float g[VPT];
  load_row<float, VPT>(gamma + lane * VPT, g);
  float dg[VPT], db[VPT];
#pragma unroll
  for (int i = 0; i < VPT; ++i) dg[i] = db[i] = 0.f;
  const int64_t slab = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * slab, r1 = r0 + slab < rows ? r0 + slab : rows;
  constexpr int U = VPT <= 4 ? 4 : (VPT <= 8 ? 2 : 1);  // rows in flight per warp (memory-level parallelism)
  for (int64_t rb = r0 + wid * U; rb < r1; rb += 8 * U) {
    float xv[U][VPT], d[U][VPT], o[U][VPT];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (rb + u < r1) {
        load_row<TX, VPT>(x + (rb + u) * x_rs + lane * VPT, xv[u]);
        load_row<TD, VPT>(dy + (rb + u) * COLS + lane * VPT, d[u]);
        if (res) load_row<TO, VPT>(res + (rb + u) * x_rs + lane * VPT, o[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = rb + u;
      if (row >= r1) break;
      const float mu = mean[row], rs = rstd[row];
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        xv[u][i] = (xv[u][i] - mu) * rs;  // xhat
        float gd = g[i] * d[u][i];
        s1 += gd;
        s2 += gd * xv[u][i];
        dg[i] += d[u][i] * xv[u][i];
        db[i] += d[u][i];
      }
      s1 = warp_sum(s1) * (1.0f / COLS);
      s2 = warp_sum(s2) * (1.0f / COLS);
#pragma unroll
      for (int i = 0; i < VPT; ++i)
        o[u][i] = (res ? o[u][i] : 0.f) + rs * (g[i] * d[u][i] - s1 - xv[u][i] * s2);
      store_row<TO, VPT>(dx + row * x_rs + lane * VPT, o[u]);
    }
  }
  if (dgamma || dbeta) {
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      red[(wid * 2) * COLS + lane * VPT + i] = dg[i];
      red[(wid * 2 + 1) * COLS + lane * VPT + i] = db[i];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < COLS; c += blockDim.x) {
      float a = 0.f, b = 0.f;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) {
        a += red[(ww * 2) * COLS + c];
        b += red[(ww * 2 + 1) * COLS + c];
      }
      if (dgamma) atomicAdd(dgamma + c, a);
      if (dbeta) atomicAdd(dbeta + c, b);
    }
  }
}

// strided (channel-major) rows, one thread per row, exact width C
template <typename TD, typename TX, typename TO, int C>
__global__ void __launch_bounds__(256) ln_bwd_thread(const TD* __restrict__ dy, const TX* __restrict__ x, int64_t x_rs,
                                                     int64_t x_cs, const float* __restrict__ gamma,
                                                     const float* __restrict__ mean, const float* __restrict__ rstd,
                                                     TO* dx, const TO* res, float* __restrict__ dgamma,
                                                     float* __restrict__ dbeta, int64_t rows) {
  pdl_wait();
  __shared__ float red[2][8][C];
  float dg[C], db[C];
#pragma unroll
  for (int c = 0; c < C; ++c) dg[c] = db[c] = 0.f;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < rows;
       row += (int64_t)gridDim.x * blockDim.x) {
    float xh[C], d[C];
    const float mu = mean[row], rs = rstd[row];
    float s1 = 0.f, s2 = 0.f;
    if (sizeof(TD) == 2 && C % 8 == 0) {  // the row-major dy row as 16-byte loads
#pragma unroll
      for (int c = 0; c < C; c += 8) load_row<TD, 8>(dy + row * C + c, d + c);
    } else {
#pragma unroll
      for (int c = 0; c < C; ++c) d[c] = ldf<TD>(dy + row * C + c);
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
      xh[c] = (ldf<TX>(x + row * x_rs + c * x_cs) - mu) * rs;
      const float gd = gamma[c] * d[c];
      s1 += gd;
      s2 += gd * xh[c];
      dg[c] += d[c] * xh[c];
      db[c] += d[c];
    }
    s1 *= 1.0f / C;
    s2 *= 1.0f / C;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      float o = rs * (gamma[c] * d[c] - s1 - xh[c] * s2);
      if (res) o += ldf<TO>(res + row * x_rs + c * x_cs);
      stf<TO>(dx + row * x_rs + c * x_cs, o);
    }
  }
  if (dgamma || dbeta) {
    const int wid = threadIdx.x >> 5;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const float a = warp_sum(dg[c]), b = warp_sum(db[c]);
      if ((threadIdx.x & 31) == 0) {
        red[0][wid][c] = a;
        red[1][wid][c] = b;
      }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
      float a = 0.f, b = 0.f;
      for (int ww = 0; ww < 8; ++ww) {
        a += red[0][ww][c];
        b += red[1][ww][c];
      }
      if (dgamma) atomicAdd(dgamma + c, a);
      if (dbeta) atomicAdd(dbeta + c, b);
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
  if (cols == 32 || cols == 64 || cols == 128 || cols == 256) {
    const int64_t rpw = 32 / (cols / 8);
    int64_t need = (rows + 8 * rpw * 2 - 1) / (8 * rpw * 2), cap = (int64_t)sm_count() * 8;
    dim3 g2((unsigned)(need < cap ? need : cap));
#if LNF_PIPE  // pipelined for >= 64 columns (kernel_microbench: [65536,128] 8.4 -> 7.8 us, [32768,256] 8.8 -> 7.9,
               // [1M,128] 97 -> 86 us = 96 % of HBM); 32 columns measured slower pipelined (2.45 -> 2.8 us)
#define LNG(CC)                                                                                                    \
  ((CC) >= 64 ? ::evo::pdl_launch(ln_fwd_grp_pipe<TX, TY, CC, 2>, g2, 256, 0, st, (const TX*)x, x_rs, g, b, (TY*)y, \
                                  mean, rstd, rows, eps)                                                           \
              : ::evo::pdl_launch(ln_fwd_grp<TX, TY, CC, 2>, g2, 256, 0, st, (const TX*)x, x_rs, g, b, (TY*)y, mean,  \
                                  rstd, rows, eps))
#else
#define LNG(CC) ::evo::pdl_launch(ln_fwd_grp<TX, TY, CC, 2>, g2, 256, 0, st, (const TX*)x, x_rs, g, b, (TY*)y, mean, rstd, rows, eps)
#endif
    switch (cols) {
      case 32: LNG(32); break;
      case 64: LNG(64); break;
      case 128: LNG(128); break;
      default: LNG(256); break;
    }
#undef LNG
    EVO_LAUNCH_CHECK("layernorm fwd");
    return EVO_OK;
  }
  const int wpb = 8;
  int64_t need = (rows + 2 * wpb - 1) / (2 * wpb), cap = (int64_t)sm_count() * 8;
  dim3 grid((unsigned)(need < cap ? need : cap));
#define LNF(VPT)                                                                                             \
  ::evo::pdl_launch(ln_fwd_warp<TX, TY, VPT, K>, grid, wpb * 32, 0, st, (const TX*)x, x_rs, g, b, (TY*)y, mean, rstd, rows, \
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
  if (sizeof(TX) == 2 && sizeof(TY) == 2 && x_rs == 1 && x_cs % 8 == 0 && ((uintptr_t)x & 15) == 0 &&
      ((uintptr_t)y & 15) == 0 && (cols == 16 || cols == 32 || cols == 64)) {
    dim3 gc((unsigned)((rows + CM_RT - 1) / CM_RT));
    if (cols == 16) ::evo::pdl_launch(ln_fwd_cm<16>, gc, CM_RT, 0, st, (const bf16*)x, x_cs, g, b, (bf16*)y, mean, rstd, rows, eps);
    else if (cols == 32) ::evo::pdl_launch(ln_fwd_cm<32>, gc, CM_RT, 0, st, (const bf16*)x, x_cs, g, b, (bf16*)y, mean, rstd, rows, eps);
    else ::evo::pdl_launch(ln_fwd_cm<64>, gc, CM_RT, 0, st, (const bf16*)x, x_cs, g, b, (bf16*)y, mean, rstd, rows, eps);
    EVO_LAUNCH_CHECK("layernorm fwd channel-major");
    return EVO_OK;
  }
  dim3 grid((unsigned)((rows + 255) / 256));
  // exact widths get the 16-byte row stores (cols == MAXC)
#define LFT(MC) ::evo::pdl_launch(ln_fwd_thread<TX, TY, MC>, grid, 256, 0, st, (const TX*)x, x_rs, x_cs, g, b, (TY*)y, mean, rstd, \
                                                                rows, (int)cols, eps)
  if (cols == 32) LFT(32);
  else if (cols == 16) LFT(16);
  else if (cols == 8) LFT(8);
  else LFT(64);
#undef LFT
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
  EVO_CHECK_ARG(k == 8, EVO_ERR_SHAPE, "layernorm_rowdot: w must be padded to 8 heads (got %d)", k);
  EVO_CHECK_ARG(x_dtype == out_dtype && x_dtype == EVO_BF16, EVO_ERR_DTYPE, "layernorm_rowdot: bf16 only");
  EVO_CHECK_ARG(((uintptr_t)x & 15) == 0, EVO_ERR_ALIGN, "layernorm_rowdot: x must be 16B aligned");
  if (rows == 0) return EVO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t need = (rows + 7) / 8, cap = (int64_t)sm_count() * 8;
  dim3 grid((unsigned)(need < cap ? need : cap));
#define RDF(VPT)                                                                                               \
  ::evo::pdl_launch(ln_rowdot_fwd<bf16, VPT>, grid, 256, 0, st, (const bf16*)x, gamma, beta, w, (bf16*)out, out_hs, (bf16*)ln_out, \
                                                 mean, rstd, rows, eps)
  switch (cols) {
    case 32: RDF(1); break;
    case 64: RDF(2); break;
    case 128: RDF(4); break;
    case 256: RDF(8); break;
    default: set_error("layernorm_rowdot: unsupported width %lld", (long long)cols); return EVO_ERR_SHAPE;
  }
#undef RDF
  EVO_LAUNCH_CHECK("layernorm_rowdot fwd");
  return EVO_OK;
}

extern "C" int evo_layernorm_rowdot_bwd(const void* x, int x_dtype, const float* gamma, const float* beta,
                                        const float* w, int k, const float* dout, int64_t out_hs, const float* mean,
                                        const float* rstd, const void* res, void* dx, float* dgamma, float* dbeta,
                                        float* dw, int64_t rows, int64_t cols, void* stream) {
  EVO_CHECK_ARG(x && gamma && beta && w && dout && mean && rstd && dx && dgamma && dbeta && dw, EVO_ERR_ARG,
                "layernorm_rowdot bwd: null pointer");
  EVO_CHECK_ARG(k == 8 && x_dtype == EVO_BF16, EVO_ERR_SHAPE, "layernorm_rowdot bwd: k == 8, bf16");
  if (rows == 0) return EVO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t need = (rows + 63) / 64, cap = (int64_t)sm_count() * 2;
  dim3 grid((unsigned)(need < cap ? need : cap));
#define RDB(VPT)                                                                                                 \
  ::evo::pdl_launch(ln_rowdot_bwd<bf16, VPT>, grid, 256, 0, st, (const bf16*)x, gamma, beta, w, dout, out_hs, mean, rstd,        \
                                                 (const bf16*)res, (bf16*)dx, dgamma, dbeta, dw, rows)
  switch (cols) {
    case 32: RDB(1); break;
    case 64: RDB(2); break;
    case 128: RDB(4); break;
    default: set_error("layernorm_rowdot bwd: unsupported width %lld", (long long)cols); return EVO_ERR_SHAPE;
  }
#undef RDB
  EVO_LAUNCH_CHECK("layernorm_rowdot bwd");
  return EVO_OK;
}

template <typename TD, typename TX, typename TO>
static int ln_bwd_impl(const void* dy, const void* x, int64_t x_rs, int64_t x_cs, const float* g, const float* mean,
                       const float* rstd, void* dx, const void* res, float* dg, float* db, float* dsum, int64_t rows,
                       int64_t cols, cudaStream_t st) {
  if (x_cs == 1 && (cols == 32 || cols == 64 || cols == 128 || cols == 256)) {
    const int64_t rpw = 32 / (cols / 8);
    int64_t need = (rows + 8 * rpw * 3 - 1) / (8 * rpw * 3), cap = (int64_t)sm_count() * 2;  // resident
    dim3 grid((unsigned)(need < cap ? need : cap));
#define LBG(CC)                                                                                               \
  ::evo::pdl_launch(ln_bwd_grp<TD, TX, TO, CC, 3>, grid, 256, 0, st, (const TD*)dy, (const TX*)x, x_rs, g, mean, \
                                                                        rstd, (TO*)dx, (const TO*)res, dg, db, dsum, rows)
    switch (cols) {
      case 32: LBG(32); break;
      case 64: LBG(64); break;
      case 128: LBG(128); break;
      default: LBG(256); break;
    }
#undef LBG
    EVO_LAUNCH_CHECK("layernorm bwd");
    return EVO_OK;
  }
  EVO_CHECK_ARG(dsum == nullptr, EVO_ERR_SHAPE, "layernorm bwd: fused dx column sums need 32/64/128/256 contiguous "
                "columns (got %lld)", (long long)cols);
  if (x_cs == 1 && cols % 32 == 0 && cols <= 1024) {
    int64_t need = (rows + 127) / 128, cap = (int64_t)sm_count() * 4;  // 4-row batches per warp
    dim3 grid((unsigned)(need < cap ? need : cap));
    size_t sm = 16 * cols * sizeof(float);
#define LNB(VPT)                                                                                            \
  ::evo::pdl_launch(ln_bwd_warp<TD, TX, TO, VPT>, grid, 256, sm, st, (const TD*)dy, (const TX*)x, x_rs, g, mean, rstd,     \
                                                      (TO*)dx, (const TO*)res, dg, db, rows)
    switch (cols) {
      case 32: LNB(1); break;
      case 64: LNB(2); break;
      case 128: LNB(4); break;
      case 256: LNB(8); break;
      case 384: LNB(12); break;
      case 512: LNB(16); break;
      default: set_error("layernorm bwd: unsupported width %lld", (long long)cols); return EVO_ERR_SHAPE;
    }
#undef LNB
    EVO_LAUNCH_CHECK("layernorm bwd");
    return EVO_OK;
  }
  if (sizeof(TD) == 2 && sizeof(TX) == 2 && sizeof(TO) == 2 && x_rs == 1 && x_cs % 8 == 0 &&
      (((uintptr_t)x | (uintptr_t)dx | (uintptr_t)dy) & 15) == 0 && (cols == 16 || cols == 32)) {
    dim3 gc((unsigned)((rows + CM_RT - 1) / CM_RT));
#define LBC(CC)                                                                                                   \
  ::evo::pdl_launch(ln_bwd_cm<CC>, gc, CM_RT, 0, st, (const bf16*)dy, (const bf16*)x, x_cs, g, mean, rstd, (bf16*)dx, (const bf16*)res, \
                                      dg, db, rows)
    if (cols == 16) LBC(16);
    else LBC(32);
#undef LBC
    EVO_LAUNCH_CHECK("layernorm bwd channel-major");
    return EVO_OK;
  }
  int64_t need = (rows + 255) / 256, cap = (int64_t)sm_count() * 4;
  dim3 grid((unsigned)(need < cap ? need : cap));
#define LNT(CC)                                                                                              \
  ::evo::pdl_launch(ln_bwd_thread<TD, TX, TO, CC>, grid, 256, 0, st, (const TD*)dy, (const TX*)x, x_rs, x_cs, g, mean, rstd, \
                                                      (TO*)dx, (const TO*)res, dg, db, rows)
  switch (cols) {
    case 2: LNT(2); break;
    case 4: LNT(4); break;
    case 8: LNT(8); break;
    case 16: LNT(16); break;
    case 32: LNT(32); break;
    case 64: LNT(64); break;
    default: set_error("layernorm bwd: strided width %lld unsupported", (long long)cols); return EVO_ERR_SHAPE;
  }
#undef LNT
  EVO_LAUNCH_CHECK("layernorm bwd strided");
  return EVO_OK;
}

static int ln_bwd_entry(const void* dy, int dy_dtype, const void* x, int x_dtype, int64_t x_rs, int64_t x_cs,
                        const float* gamma, const float* mean, const float* rstd, void* dx, int dx_dtype,
                        const void* res, float* dgamma, float* dbeta, float* dsum, int64_t rows, int64_t cols,
                        void* stream) {
  EVO_CHECK_ARG(dy && x && gamma && mean && rstd && dx, EVO_ERR_ARG, "layernorm bwd: null pointer");
  if (rows == 0) return EVO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  EVO_CHECK_ARG(x_dtype == dx_dtype, EVO_ERR_DTYPE, "layernorm bwd: x and dx dtypes must match");
  if (dy_dtype == EVO_BF16) {
    if (x_dtype == EVO_BF16)
      return ln_bwd_impl<bf16, bf16, bf16>(dy, x, x_rs, x_cs, gamma, mean, rstd, dx, res, dgamma, dbeta, dsum, rows,
                                           cols, st);
    return ln_bwd_impl<bf16, float, float>(dy, x, x_rs, x_cs, gamma, mean, rstd, dx, res, dgamma, dbeta, dsum, rows,
                                           cols, st);
  }
  if (x_dtype == EVO_BF16)
    return ln_bwd_impl<float, bf16, bf16>(dy, x, x_rs, x_cs, gamma, mean, rstd, dx, res, dgamma, dbeta, dsum, rows,
                                          cols, st);
  return ln_bwd_impl<float, float, float>(dy, x, x_rs, x_cs, gamma, mean, rstd, dx, res, dgamma, dbeta, dsum, rows,
                                          cols, st);
}

extern "C" int evo_layernorm_bwd(const void* dy, int dy_dtype, const void* x, int x_dtype, int64_t x_rs, int64_t x_cs,
                                 const float* gamma, const float* mean, const float* rstd, void* dx, int dx_dtype,
                                 const void* res, float* dgamma, float* dbeta, int64_t rows, int64_t cols,
                                 void* stream) {
  return ln_bwd_entry(dy, dy_dtype, x, x_dtype, x_rs, x_cs, gamma, mean, rstd, dx, dx_dtype, res, dgamma, dbeta,
                      nullptr, rows, cols, stream);
}

extern "C" int evo_layernorm_bwd_colsum(const void* dy, int dy_dtype, const void* x, int x_dtype, int64_t x_rs,
                                        int64_t x_cs, const float* gamma, const float* mean, const float* rstd,
                                        void* dx, int dx_dtype, const void* res, float* dgamma, float* dbeta,
                                        float* dx_colsum, int64_t rows, int64_t cols, void* stream) {
  return ln_bwd_entry(dy, dy_dtype, x, x_dtype, x_rs, x_cs, gamma, mean, rstd, dx, dx_dtype, res, dgamma, dbeta,
                      dx_colsum, rows, cols, stream);
}
