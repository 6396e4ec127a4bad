// Fused elementwise epilogues of the Evoformer block (HBM-bound, 16-byte vectors):
//   * gated residual  out = res + sigmoid(gp) * (y + bias)  - every residual add of
//     evoformer_block (evoformer.py:316-324) with the projection bias folded in,
//     and the triangle g-gate (evoformer.py:270);
//   * bias + ReLU of the transition hidden layer (evoformer.py:239);
//   * triangle gating a = sigmoid(.)*(.), b = sigmoid(.)*(.) (evoformer.py:261-264)
//     with a channel-major write (so the einsum is a batched GEMM over channels);
//   * non-finite counter (engine.py:186-187 DomainError twin).
// Backward kernels reduce bias gradients per column with a [32 x 8] thread tile,
// shared-memory partials and one atomicAdd per column per CTA.
#include "common.cuh"

namespace evo {
int sm_count();

template <typename T>
__device__ __forceinline__ void ld8(const T* p, float* v) {
  if constexpr (sizeof(T) == 2) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    unpack_bf16x2(u.x, v[0], v[1]); unpack_bf16x2(u.y, v[2], v[3]);
    unpack_bf16x2(u.z, v[4], v[5]); unpack_bf16x2(u.w, v[6], v[7]);
  } else {
    float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
}
template <typename T>
__device__ __forceinline__ void st8(T* p, const float* v) {
  if constexpr (sizeof(T) == 2) {
    uint4 u;
    u.x = pack_bf16x2(v[0], v[1]); u.y = pack_bf16x2(v[2], v[3]);
    u.z = pack_bf16x2(v[4], v[5]); u.w = pack_bf16x2(v[6], v[7]);
    *reinterpret_cast<uint4*>(p) = u;
  } else {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
  }
}

// ------------------------------------------------------------------ gated residual
// IDX: uint32_t when rows*cols/8 < 2^31 (one 32-bit division per vector instead of a 64-bit
// one, which costs more issue slots than the vector's arithmetic), else int64_t
template <typename T, typename IDX>
__global__ void __launch_bounds__(256) gated_residual_fwd_k(const T* __restrict__ res, const T* __restrict__ y,
                                                            int64_t y_rs, const float* __restrict__ bias,
                                                            const T* __restrict__ gp, int64_t gp_rs,
                                                            T* __restrict__ out, int64_t rows, int64_t cols) {
  pdl_wait();
  const IDX cpr = (IDX)(cols / 8);
  const IDX n = (IDX)(rows * (cols / 8));
  for (IDX i = (IDX)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (IDX)gridDim.x * blockDim.x) {
    const IDX rr = i / cpr;
    const int64_t r = rr, c = (int64_t)(i - rr * cpr) * 8;
    float rv[8], yv[8];
    ld8<T>(res + r * cols + c, rv);
    ld8<T>(y + r * y_rs + c, yv);
    if (bias) {
#pragma unroll
      for (int e = 0; e < 8; ++e) yv[e] += bias[c + e];
    }
    if (gp) {
      float gv[8];
      ld8<T>(gp + r * gp_rs + c, gv);
#pragma unroll
      for (int e = 0; e < 8; ++e) yv[e] = __fmul_rn(yv[e], sigmoidf_(gv[e]));  // no FMA contraction: bitwise
    }                                                                        // equal to residual_ln_k
#pragma unroll
    for (int e = 0; e < 8; ++e) rv[e] += yv[e];
    st8<T>(out + r * cols + c, rv);
  }
}

// Column-reduction layout shared by the backward epilogues and colsum:
// 256 threads, tpr = cols/8 threads per row (8 columns = 16 bytes each), rpi =
// 256/tpr rows per iteration; CTA b owns the contiguous row slab
// [b*slab, (b+1)*slab) and keeps its column partials in registers; one
// shared-memory pass and one atomicAdd per column per CTA at the end
// (grid ~ 2 x SMs, so each dbias address sees ~300 atomics, not ~rows/8).
struct ColTile {
  int tpr, rpi, tr, tc;
  int64_t r0, r1;
  __device__ ColTile(int64_t rows, int64_t cols) {
    tpr = (int)(cols / 8);
    rpi = blockDim.x / tpr;
    tr = threadIdx.x / tpr;
    tc = threadIdx.x % tpr;
    const int64_t slab = (rows + gridDim.x - 1) / gridDim.x;
    r0 = blockIdx.x * slab;
    r1 = r0 + slab < rows ? r0 + slab : rows;
  }
  __device__ bool active() const { return tr < rpi; }
};

// red: shared [rpi][cols]; adds the CTA's column sums into out (fp32)
__device__ __forceinline__ void col_flush(float* red, const ColTile& t, const float* acc, int64_t cols, float* out) {
  if (t.active()) {
#pragma unroll
    for (int e = 0; e < 8; ++e) red[t.tr * cols + t.tc * 8 + e] = acc[e];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    float s = 0.f;
    for (int r = 0; r < t.rpi; ++r) s += red[r * cols + c];
    atomicAdd(out + c, s);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) gated_residual_bwd_k(const T* __restrict__ dout, const T* __restrict__ y,
                                                            int64_t y_rs, const float* __restrict__ bias,
                                                            const T* __restrict__ gp, int64_t gp_rs, T* __restrict__ dy,
                                                            T* __restrict__ dgp, int64_t dgp_rs,
                                                            float* __restrict__ dbias, float* __restrict__ dgp_sum,
                                                            int64_t rows, int64_t cols) {
  pdl_wait();
  extern __shared__ float red[];
  const ColTile t(rows, cols);
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  float acc_g[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // fp32 column sums of dgp (its bias gradient, pre-rounding)
  if (t.active()) {
    const int64_t c = t.tc * 8;
    float b[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (bias && gp) {
#pragma unroll
      for (int e = 0; e < 8; ++e) b[e] = bias[c + e];
    }
    // two rows per step with all loads first (outputs may alias inputs)
    int64_t r = t.r0 + t.tr;
    for (; r < t.r1; r += 2 * t.rpi) {
      const bool two = r + t.rpi < t.r1;
      float d[2][8], gv[2][8], yv[2][8];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (u == 1 && !two) break;
        const int64_t ru = r + u * t.rpi;
        ld8<T>(dout + ru * cols + c, d[u]);
        if (gp) {
          ld8<T>(gp + ru * gp_rs + c, gv[u]);
          ld8<T>(y + ru * y_rs + c, yv[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (u == 1 && !two) break;
        const int64_t ru = r + u * t.rpi;
        if (gp) {
          float dg[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            float s = sigmoidf_(gv[u][e]);
            dg[e] = d[u][e] * (yv[u][e] + b[e]) * s * (1.f - s);
            d[u][e] *= s;
            acc_g[e] += dg[e];
          }
          st8<T>(dgp + ru * dgp_rs + c, dg);
        }
        if (dy) st8<T>(dy + ru * cols + c, d[u]);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += d[u][e];
      }
    }
  }
  if (dbias) col_flush(red, t, acc, cols, dbias);
  if (dgp_sum) {
    if (dbias) __syncthreads();  // red reused
    col_flush(red, t, acc_g, cols, dgp_sum);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) colsum_k(const T* __restrict__ x, int64_t ld, int64_t rows, int64_t cols,
                                                float* __restrict__ out) {
  pdl_wait();
  extern __shared__ float red[];
  const ColTile t(rows, cols);
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (t.active()) {
    const int64_t c = t.tc * 8;
    int64_t r = t.r0 + t.tr;
    for (; r + 3 * t.rpi < t.r1; r += 4 * t.rpi) {  // four rows in flight
      float u[4][8];
#pragma unroll
      for (int q = 0; q < 4; ++q) ld8<T>(x + (r + q * t.rpi) * ld + c, u[q]);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += (u[0][e] + u[1][e]) + (u[2][e] + u[3][e]);
    }
    for (; r < t.r1; r += t.rpi) {
      float u[8];
      ld8<T>(x + r * ld + c, u);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += u[e];
    }
  }
  col_flush(red, t, acc, cols, out);
}

// ------------------------------------------------------------------ bias + activation
template <typename T, typename IDX>
__global__ void __launch_bounds__(256) bias_act_fwd_k(T* __restrict__ y, const float* __restrict__ bias, int64_t rows,
                                                      int64_t cols, int act) {
  pdl_wait();
  const IDX cpr = (IDX)(cols / 8), n = (IDX)(rows * (cols / 8));
  for (IDX i = (IDX)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (IDX)gridDim.x * blockDim.x) {
    const IDX rr = i / cpr;
    const int64_t r = rr, c = (int64_t)(i - rr * cpr) * 8;
    float v[8];
    ld8<T>(y + r * cols + c, v);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      v[e] += bias ? bias[c + e] : 0.f;
      if (act == 1) v[e] = fmaxf(v[e], 0.f);
    }
    st8<T>(y + r * cols + c, v);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) bias_act_bwd_k(const T* __restrict__ dh, const T* __restrict__ h,
                                                      T* __restrict__ dy, float* __restrict__ dbias, int64_t rows,
                                                      int64_t cols, int act) {
  pdl_wait();
  extern __shared__ float red[];
  const ColTile t(rows, cols);
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (t.active()) {
    const int64_t c = t.tc * 8;
    // U rows per step with every load issued before the (possibly in-place) stores: dy may
    // alias dh, so without this the compiler keeps one row in flight per thread
    constexpr int U = 4;
    int64_t r = t.r0 + t.tr;
    for (; r + (U - 1) * t.rpi < t.r1; r += U * t.rpi) {
      float d[U][8], hv[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ld8<T>(dh + (r + u * t.rpi) * cols + c, d[u]);
        if (act == 1) ld8<T>(h + (r + u * t.rpi) * cols + c, hv[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (act == 1) {
#pragma unroll
          for (int e = 0; e < 8; ++e) d[u][e] = hv[u][e] > 0.f ? d[u][e] : 0.f;
        }
        st8<T>(dy + (r + u * t.rpi) * cols + c, d[u]);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += d[u][e];
      }
    }
    for (; r < t.r1; r += t.rpi) {
      float d[8], hv[8];
      ld8<T>(dh + r * cols + c, d);
      if (act == 1) {
        ld8<T>(h + r * cols + c, hv);
#pragma unroll
        for (int e = 0; e < 8; ++e) d[e] = hv[e] > 0.f ? d[e] : 0.f;
      }
      st8<T>(dy + r * cols + c, d);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += d[e];
    }
  }
  if (dbias) col_flush(red, t, acc, cols, dbias);
}

// ------------------------------------------------------------------ triangle gating
// RB rows per CTA; Y row slice [hz, hz+4p) staged in shared memory as fp32
template <int P>
__global__ void __launch_bounds__(256) tri_gate_fwd_k(const bf16* __restrict__ y, int64_t rows, int hz,
                                                      bf16* __restrict__ a_cm, bf16* __restrict__ b_cm,
                                                      bool pairs) {
  pdl_wait();
  constexpr int W = 4 * P;
  constexpr int RB = P <= 32 ? 64 : 32;
  __shared__ float ys[RB][W + 1];
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const int64_t ld = hz + W;
  for (int i = threadIdx.x; i < RB * W / 8; i += blockDim.x) {
    const int r = i / (W / 8), c = (i % (W / 8)) * 8;
    float v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (r0 + r < rows) ld8<bf16>(y + (r0 + r) * ld + hz + c, v);
#pragma unroll
    for (int e = 0; e < 8; ++e) ys[r][c + e] = v[e];
  }
  __syncthreads();
  // write a[h][r], b[h][r]: consecutive threads -> consecutive row pairs (coalesced 4-byte
  // stores of two rows; scalar when the host found rows odd or a_cm / b_cm not 4-byte
  // aligned, and at the ragged end)
  for (int i = threadIdx.x; i < P * RB; i += blockDim.x) {
    const int r = (i % (RB / 2)) * 2, ch = i / (RB / 2);  // ch < 2P
    if (r0 + r >= rows) continue;
    const int h = ch % P, which = ch / P;  // 0 = a, 1 = b
    const int cs = which * 2 * P + h, cl = cs + P;
    const float v0 = sigmoidf_(ys[r][cs]) * ys[r][cl];
    const float v1 = sigmoidf_(ys[r + 1][cs]) * ys[r + 1][cl];
    bf16* dst = (which ? b_cm : a_cm) + (int64_t)h * rows + r0 + r;
    if (pairs && r0 + r + 1 < rows) {
      *reinterpret_cast<uint32_t*>(dst) = pack_bf16x2(v0, v1);
    } else {
      dst[0] = f2bf(v0);
      if (r0 + r + 1 < rows) dst[1] = f2bf(v1);
    }
  }
}

template <int P, typename TD>
__global__ void __launch_bounds__(256) tri_gate_bwd_k(const bf16* __restrict__ y, const TD* __restrict__ da,
                                                      const TD* __restrict__ db, int64_t rows, int hz,
                                                      bf16* __restrict__ dy, float* __restrict__ dsum) {
  pdl_wait();
  constexpr int W = 4 * P;
  __shared__ float gs[64][2 * P + 1];
  __shared__ float cs[256 / (W / 8 < 256 ? W / 8 : 256)][W + 1];  // per row-group column partials
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};                         // fp32 sums of dY[:, hz:] (its bias grad)
  const int64_t r0 = (int64_t)blockIdx.x * 64;
  const int64_t ld = hz + W;
  for (int i = threadIdx.x; i < 2 * P * 64; i += blockDim.x) {
    const int r = i & 63, ch = i >> 6;
    float v = 0.f;
    if (r0 + r < rows) {
      const int h = ch % P;
      const TD* src = ch < P ? da : db;
      v = ldf<TD>(src + (int64_t)h * rows + r0 + r);
    }
    gs[r][ch] = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 64 * W / 8; i += blockDim.x) {
    const int r = i / (W / 8), c = (i % (W / 8)) * 8;  // c in [0, 4P)
    if (r0 + r >= rows) continue;
    float o[8];
    if constexpr (P % 8 == 0) {
      // the chunk's 8 columns share the block (a / b) and the part (sig / lin): its sig (and
      // lin) inputs are 8 consecutive channels of the row -> 16-byte loads, not 16 scalar ones
      const int which = c / (2 * P), cc0 = c % (2 * P), h0 = cc0 % P;
      const bf16* yrow = y + (r0 + r) * ld + hz + which * 2 * P;
      float sv[8], lv[8];
      const uint4 us = *reinterpret_cast<const uint4*>(yrow + h0);
      unpack_bf16x2(us.x, sv[0], sv[1]); unpack_bf16x2(us.y, sv[2], sv[3]);
      unpack_bf16x2(us.z, sv[4], sv[5]); unpack_bf16x2(us.w, sv[6], sv[7]);
      if (cc0 < P) {
        const uint4 ul = *reinterpret_cast<const uint4*>(yrow + P + h0);
        unpack_bf16x2(ul.x, lv[0], lv[1]); unpack_bf16x2(ul.y, lv[2], lv[3]);
        unpack_bf16x2(ul.z, lv[4], lv[5]); unpack_bf16x2(ul.w, lv[6], lv[7]);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float sg = sigmoidf_(sv[e]);
        const float g = gs[r][which * P + h0 + e];
        o[e] = cc0 < P ? g * lv[e] * sg * (1.f - sg) : g * sg;
        acc[e] += o[e];
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int which = (c + e) / (2 * P);              // 0: a block, 1: b block
        const int cc = (c + e) % (2 * P);                 // [0, P) = sig part, [P, 2P) = lin part
        const bf16* yrow = y + (r0 + r) * ld + hz + which * 2 * P;
        const int h = cc % P;
        const float s = bf2f(yrow[h]), l = bf2f(yrow[P + h]);
        const float sg = sigmoidf_(s);
        const float g = gs[r][which * P + h];
        o[e] = cc < P ? g * l * sg * (1.f - sg) : g * sg;
        acc[e] += o[e];
      }
    }
    st8<bf16>(dy + (r0 + r) * ld + hz + c, o);
  }
  if (dsum) {  // the thread's column chunk is fixed (256 % (W/8) == 0): one smem pass, one atomic per column
    constexpr int CPR = W / 8, RG = 256 / CPR;
    const int rg = threadIdx.x / CPR, c = (threadIdx.x % CPR) * 8;
#pragma unroll
    for (int e = 0; e < 8; ++e) cs[rg][c + e] = acc[e];
    __syncthreads();
    for (int col = threadIdx.x; col < W; col += blockDim.x) {
      float sum = 0.f;
      for (int g2 = 0; g2 < RG; ++g2) sum += cs[g2][col];
      atomicAdd(dsum + col, sum);
    }
  }
}

template <typename T>
__global__ void count_nonfinite_k(const T* __restrict__ x, int64_t n, unsigned int* counter) {
  pdl_wait();
  unsigned int local = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    local += isfinite(ldf<T>(x + i)) ? 0u : 1u;
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(counter, local);
}

// ------------------------------------------------------------------ residual + LayerNorm
// out = res + [sigmoid(gp) *] (y + bias)   (the module's residual epilogue), then the next
// module's LayerNorm of out (engine.layernorm_raw, engine.py:206-217) in the same pass:
// ln = (out - mean) * rstd * gamma + beta, mean/rstd saved.  Saves the LayerNorm's re-read
// of out and a launch per module boundary.  LPR = COLS/8 lanes per row (16-byte lanes),
// U rows per lane group per step with every load issued first.
// measured (scripts/rln_micro.py): 2 row groups per lane at 3 CTAs/SM beat 4 at 2 CTAs/SM
// (e.g. [65536,128] 13.9 -> 13.1 us, gated 16.6 -> 15.2 us)
// RLN_PIPE (default): one row group per lane, software-pipelined (the next group's loads issued
// before this group's math), 3 CTAs/SM - scripts/rln_micro.py: [65536,128] 12.9 -> 12.1 us, gated
// 14.9 -> 13.5 us, [32768,256] 13.1 -> 12.4 us against the unpipelined two-group form (RLN_PIPE=0)
#ifndef RLN_PIPE
#define RLN_PIPE 1
#endif
#if RLN_PIPE
#ifndef RLN_MINB_PIPE
#define RLN_MINB_PIPE 3
#endif
constexpr int RLN_U = 1, RLN_MINB = RLN_MINB_PIPE;
#else
constexpr int RLN_U = 2, RLN_MINB = 3;
#endif
template <int COLS, int U>
__global__ void __launch_bounds__(256, RLN_MINB) residual_ln_k(const bf16* __restrict__ res, const bf16* __restrict__ y,
                                                        int64_t y_rs, const float* __restrict__ bias,
                                                        const bf16* __restrict__ gp, int64_t gp_rs,
                                                        bf16* __restrict__ out, const float* __restrict__ gamma,
                                                        const float* __restrict__ beta, bf16* __restrict__ ln,
                                                        float* __restrict__ mean, float* __restrict__ rstd,
                                                        int64_t rows, float eps) {
  pdl_wait();
  // loads stay raw (one uint4 per 8 bf16) until used and the per-column vectors are re-read
  // through smem at use: RLN_MINB CTAs per SM, RLN_U row-groups of 3 loads in flight per lane
  constexpr int LPR = COLS / 8, RPW = 32 / LPR;
  __shared__ float4 cv[3][COLS / 4];  // bias, gamma, beta (volatile reads: not hoisted into registers)
  for (int i = threadIdx.x; i < COLS; i += blockDim.x) {
    reinterpret_cast<float*>(cv[0])[i] = bias ? bias[i] : 0.f;
    reinterpret_cast<float*>(cv[1])[i] = gamma[i];
    reinterpret_cast<float*>(cv[2])[i] = beta[i];
  }
  __syncthreads();
  const volatile float4* vb = cv[0];
  const volatile float4* vg = cv[1];
  const volatile float4* vt = cv[2];
  const int lane = threadIdx.x & 31, sub = lane / LPR, cl = (lane % LPR) * 8;
#if RLN_PIPE
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t step = nw * RPW * U;
  uint4 rr[U], yr[U], gr[U];
  auto load = [&](int64_t rb_) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = rb_ + u * RPW + sub;
      if (row < rows) {
        rr[u] = __ldcs(reinterpret_cast<const uint4*>(res + row * COLS + cl));
        yr[u] = __ldcs(reinterpret_cast<const uint4*>(y + row * y_rs + cl));
        if (gp) gr[u] = __ldcs(reinterpret_cast<const uint4*>(gp + row * gp_rs + cl));
      }
    }
  };
  int64_t rb = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * RPW * U;
  if (rb < rows) load(rb);
  for (; rb < rows; rb += step) {
    // software pipeline (RLN_PIPE): the raw loads of this lane's next row group are issued before this
    // group's math and stores, so the memory pipe never drains between groups
    uint4 rc[U], yc[U], gc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { rc[u] = rr[u]; yc[u] = yr[u]; gc[u] = gr[u]; }
    if (rb + step < rows) load(rb + step);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = rb + u * RPW + sub;
      float o[8], t[8], s = 0.f;
      unpack_bf16x2(rc[u].x, o[0], o[1]); unpack_bf16x2(rc[u].y, o[2], o[3]);
      unpack_bf16x2(rc[u].z, o[4], o[5]); unpack_bf16x2(rc[u].w, o[6], o[7]);
      unpack_bf16x2(yc[u].x, t[0], t[1]); unpack_bf16x2(yc[u].y, t[2], t[3]);
      unpack_bf16x2(yc[u].z, t[4], t[5]); unpack_bf16x2(yc[u].w, t[6], t[7]);
      {
        const float4 b0 = const_cast<const float4&>(vb[cl / 4]);
        const float4 b1 = const_cast<const float4&>(vb[cl / 4 + 1]);
        t[0] += b0.x; t[1] += b0.y; t[2] += b0.z; t[3] += b0.w;
        t[4] += b1.x; t[5] += b1.y; t[6] += b1.z; t[7] += b1.w;
      }
      if (gp) {
        float gv[8];
        unpack_bf16x2(gc[u].x, gv[0], gv[1]); unpack_bf16x2(gc[u].y, gv[2], gv[3]);
        unpack_bf16x2(gc[u].z, gv[4], gv[5]); unpack_bf16x2(gc[u].w, gv[6], gv[7]);
#pragma unroll
        for (int e = 0; e < 8; ++e) t[e] = __fmul_rn(t[e], sigmoidf_(gv[e]));
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] += t[e];
      // LayerNorm statistics of the bf16-rounded residual stream (what the next module reads)
      uint4 w;
      w.x = pack_bf16x2(o[0], o[1]); w.y = pack_bf16x2(o[2], o[3]);
      w.z = pack_bf16x2(o[4], o[5]); w.w = pack_bf16x2(o[6], o[7]);
      unpack_bf16x2(w.x, o[0], o[1]); unpack_bf16x2(w.y, o[2], o[3]);
      unpack_bf16x2(w.z, o[4], o[5]); unpack_bf16x2(w.w, o[6], o[7]);
#pragma unroll
      for (int e = 0; e < 8; ++e) s += o[e];
#pragma unroll
      for (int off = LPR / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      const float mu = s * (1.0f / COLS);
      float q = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) q += (o[e] - mu) * (o[e] - mu);
#pragma unroll
      for (int off = LPR / 2; off > 0; off >>= 1) q += __shfl_xor_sync(0xffffffffu, q, off);
      const float rs = rsqrtf(q * (1.0f / COLS) + eps);
      if (row < rows) {
        *reinterpret_cast<uint4*>(out + row * COLS + cl) = w;
        const float4 g0 = const_cast<const float4&>(vg[cl / 4]);
        const float4 g1 = const_cast<const float4&>(vg[cl / 4 + 1]);
        const float4 c0 = const_cast<const float4&>(vt[cl / 4]);
        const float4 c1 = const_cast<const float4&>(vt[cl / 4 + 1]);
        const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float bb[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
        float lv[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) lv[e] = (o[e] - mu) * rs * gg[e] + bb[e];
        st8<bf16>(ln + row * COLS + cl, lv);
        if (cl == 0 && mean) {
          mean[row] = mu;
          rstd[row] = rs;
        }
      }
    }
  }
}

#else
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t rb = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * RPW * U; rb < rows;
       rb += nw * RPW * U) {
    uint4 rr[U], yr[U], gr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = rb + u * RPW + sub;
      if (row < rows) {
        rr[u] = __ldcs(reinterpret_cast<const uint4*>(res + row * COLS + cl));
        yr[u] = __ldcs(reinterpret_cast<const uint4*>(y + row * y_rs + cl));
        if (gp) gr[u] = __ldcs(reinterpret_cast<const uint4*>(gp + row * gp_rs + cl));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = rb + u * RPW + sub;
      float o[8], t[8], s = 0.f;
      unpack_bf16x2(rr[u].x, o[0], o[1]); unpack_bf16x2(rr[u].y, o[2], o[3]);
      unpack_bf16x2(rr[u].z, o[4], o[5]); unpack_bf16x2(rr[u].w, o[6], o[7]);
      unpack_bf16x2(yr[u].x, t[0], t[1]); unpack_bf16x2(yr[u].y, t[2], t[3]);
      unpack_bf16x2(yr[u].z, t[4], t[5]); unpack_bf16x2(yr[u].w, t[6], t[7]);
      {
        const float4 b0 = const_cast<const float4&>(vb[cl / 4]);
        const float4 b1 = const_cast<const float4&>(vb[cl / 4 + 1]);
        t[0] += b0.x; t[1] += b0.y; t[2] += b0.z; t[3] += b0.w;
        t[4] += b1.x; t[5] += b1.y; t[6] += b1.z; t[7] += b1.w;
      }
      if (gp) {
        float gv[8];
        unpack_bf16x2(gr[u].x, gv[0], gv[1]); unpack_bf16x2(gr[u].y, gv[2], gv[3]);
        unpack_bf16x2(gr[u].z, gv[4], gv[5]); unpack_bf16x2(gr[u].w, gv[6], gv[7]);
#pragma unroll
        for (int e = 0; e < 8; ++e) t[e] = __fmul_rn(t[e], sigmoidf_(gv[e]));
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] += t[e];
      // LayerNorm statistics of the bf16-rounded residual stream (what the next module reads)
      uint4 w;
      w.x = pack_bf16x2(o[0], o[1]); w.y = pack_bf16x2(o[2], o[3]);
      w.z = pack_bf16x2(o[4], o[5]); w.w = pack_bf16x2(o[6], o[7]);
      unpack_bf16x2(w.x, o[0], o[1]); unpack_bf16x2(w.y, o[2], o[3]);
      unpack_bf16x2(w.z, o[4], o[5]); unpack_bf16x2(w.w, o[6], o[7]);
#pragma unroll
      for (int e = 0; e < 8; ++e) s += o[e];
#pragma unroll
      for (int off = LPR / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      const float mu = s * (1.0f / COLS);
      float q = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) q += (o[e] - mu) * (o[e] - mu);
#pragma unroll
      for (int off = LPR / 2; off > 0; off >>= 1) q += __shfl_xor_sync(0xffffffffu, q, off);
      const float rs = rsqrtf(q * (1.0f / COLS) + eps);
      if (row < rows) {
        *reinterpret_cast<uint4*>(out + row * COLS + cl) = w;
        const float4 g0 = const_cast<const float4&>(vg[cl / 4]);
        const float4 g1 = const_cast<const float4&>(vg[cl / 4 + 1]);
        const float4 c0 = const_cast<const float4&>(vt[cl / 4]);
        const float4 c1 = const_cast<const float4&>(vt[cl / 4 + 1]);
        const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float bb[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
        float lv[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) lv[e] = (o[e] - mu) * rs * gg[e] + bb[e];
        st8<bf16>(ln + row * COLS + cl, lv);
        if (cl == 0 && mean) {
          mean[row] = mu;
          rstd[row] = rs;
        }
      }
    }
  }
}

#endif
static unsigned grid_for(int64_t work, int threads) {
  int64_t need = (work + threads - 1) / threads;
  int64_t cap = (int64_t)sm_count() * 16;
  return (unsigned)(need < 1 ? 1 : (need < cap ? need : cap));
}

static bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

}  // namespace evo

using namespace evo;

extern "C" int evo_gated_residual_fwd(const void* res, const void* y, int64_t y_rs, const float* bias, const void* gp,
                                      int64_t gp_rs, void* out, int dtype, int64_t rows, int64_t cols, void* stream) {
  EVO_CHECK_ARG(res && y && out, EVO_ERR_ARG, "gated_residual: null pointer");
  EVO_CHECK_ARG(cols % 8 == 0 && y_rs % 8 == 0 && (!gp || gp_rs % 8 == 0), EVO_ERR_ALIGN,
                "gated_residual: cols and row strides must be multiples of 8");
  EVO_CHECK_ARG(al16(res) && al16(y) && al16(out) && (!gp || al16(gp)), EVO_ERR_ALIGN,
                "gated_residual: pointers must be 16B aligned");
  if (rows == 0) return EVO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned g = grid_for(rows * cols / 8, 256);
  const bool i32 = rows * (cols / 8) < (1LL << 31);
#define GRF(T, I) ::evo::pdl_launch(gated_residual_fwd_k<T, I>, g, 256, 0, st, (const T*)res, (const T*)y, y_rs, bias, (const T*)gp, \
                                                                gp_rs, (T*)out, rows, cols)
  if (dtype == EVO_BF16) {
    if (i32) GRF(bf16, uint32_t); else GRF(bf16, int64_t);
  } else {
    if (i32) GRF(float, uint32_t); else GRF(float, int64_t);
  }
#undef GRF
  EVO_LAUNCH_CHECK("gated_residual fwd");
  return EVO_OK;
}

static int col_grid(int64_t rows, int64_t cols, dim3& grid, size_t& smem) {
  if (cols % 8 || cols / 8 > 256) {
    set_error("column reduction: cols must be a multiple of 8 and <= 2048 (got %lld)", (long long)cols);
    return EVO_ERR_SHAPE;
  }
  const int tpr = (int)(cols / 8), rpi = 256 / tpr;
  int64_t want = (rows + 8 * rpi - 1) / (8 * rpi);  // >= 8 row-iterations per CTA
  int64_t cap = (int64_t)sm_count() * 2;
  grid = dim3((unsigned)(want < 1 ? 1 : (want < cap ? want : cap)));
  smem = (size_t)rpi * cols * sizeof(float);
  return EVO_OK;
}

extern "C" int evo_gated_residual_bwd(const void* dout, const void* y, int64_t y_rs, const float* bias, const void* gp,
                                      int64_t gp_rs, void* dy, void* dgp, int64_t dgp_rs, float* dbias,
                                      float* dgp_sum, int dtype, int64_t rows, int64_t cols, void* stream) {
  EVO_CHECK_ARG(dout, EVO_ERR_ARG, "gated_residual bwd: null dout");
  EVO_CHECK_ARG(!gp || (y && dgp), EVO_ERR_ARG, "gated_residual bwd: gp needs y and dgp");
  EVO_CHECK_ARG(!dgp_sum || gp, EVO_ERR_ARG, "gated_residual bwd: dgp_sum needs gp");
  if (rows == 0) return EVO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid;
  size_t smem;
  int rc = col_grid(rows, cols, grid, smem);
  if (rc) return rc;
  if (dtype == EVO_BF16)
    ::evo::pdl_launch(gated_residual_bwd_k<bf16>, grid, 256, smem, st, (const bf16*)dout, (const bf16*)y, y_rs, bias,
                                                        (const bf16*)gp, gp_rs, (bf16*)dy, (bf16*)dgp, dgp_rs, dbias,
                                                        dgp_sum, rows, cols);
  else
    ::evo::pdl_launch(gated_residual_bwd_k<float>, grid, 256, smem, st, (const float*)dout, (const float*)y, y_rs, bias,
                                                         (const float*)gp, gp_rs, (float*)dy, (float*)dgp, dgp_rs,
                                                         dbias, dgp_sum, rows, cols);
  EVO_LAUNCH_CHECK("gated_residual bwd");
  return EVO_OK;
}

extern "C" int evo_colsum(const void* x, int dtype, int64_t ld, int64_t rows, int64_t cols, float* out, void* stream) {
  EVO_CHECK_ARG(x && out, EVO_ERR_ARG, "colsum: null pointer");
  EVO_CHECK_ARG(ld % 8 == 0 && al16(x), EVO_ERR_ALIGN, "colsum: 16B-aligned rows required");
  if (rows == 0) return EVO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid;
  size_t smem;
  int rc = col_grid(rows, cols, grid, smem);
  if (rc) return rc;
  if (dtype == EVO_BF16) ::evo::pdl_launch(colsum_k<bf16>, grid, 256, smem, st, (const bf16*)x, ld, rows, cols, out);
  else ::evo::pdl_launch(colsum_k<float>, grid, 256, smem, st, (const float*)x, ld, rows, cols, out);
  EVO_LAUNCH_CHECK("colsum");
  return EVO_OK;
}

extern "C" int evo_bias_act_fwd(void* y, const float* bias, int64_t rows, int64_t cols, int act, int dtype,
                                void* stream) {
  EVO_CHECK_ARG(y, EVO_ERR_ARG, "bias_act: null y");
  EVO_CHECK_ARG(cols % 8 == 0 && al16(y), EVO_ERR_ALIGN, "bias_act: cols %% 8 and 16B alignment");
  if (rows == 0) return EVO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned g = grid_for(rows * cols / 8, 256);
  const bool i32 = rows * (cols / 8) < (1LL << 31);
  if (dtype == EVO_BF16) {
    if (i32) ::evo::pdl_launch(bias_act_fwd_k<bf16, uint32_t>, g, 256, 0, st, (bf16*)y, bias, rows, cols, act);
    else ::evo::pdl_launch(bias_act_fwd_k<bf16, int64_t>, g, 256, 0, st, (bf16*)y, bias, rows, cols, act);
  } else {
    if (i32) ::evo::pdl_launch(bias_act_fwd_k<float, uint32_t>, g, 256, 0, st, (float*)y, bias, rows, cols, act);
    else ::evo::pdl_launch(bias_act_fwd_k<float, int64_t>, g, 256, 0, st, (float*)y, bias, rows, cols, act);
  }
  EVO_LAUNCH_CHECK("bias_act fwd");
  return EVO_OK;
}

extern "C" int evo_bias_act_bwd(const void* dh, const void* h, void* dy, float* dbias, int64_t rows, int64_t cols,
                                int act, int dtype, void* stream) {
  EVO_CHECK_ARG(dh && dy && (act == 0 || h), EVO_ERR_ARG, "bias_act bwd: null pointer");
  if (rows == 0) return EVO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid;
  size_t smem;
  int rc = col_grid(rows, cols, grid, smem);
  if (rc) return rc;
  if (dtype == EVO_BF16)
    ::evo::pdl_launch(bias_act_bwd_k<bf16>, grid, 256, smem, st, (const bf16*)dh, (const bf16*)h, (bf16*)dy, dbias, rows, cols, act);
  else
    ::evo::pdl_launch(bias_act_bwd_k<float>, grid, 256, smem, st, (const float*)dh, (const float*)h, (float*)dy, dbias, rows, cols,
                                                   act);
  EVO_LAUNCH_CHECK("bias_act bwd");
  return EVO_OK;
}

extern "C" int evo_tri_gate_fwd(const void* y, int64_t rows, int hz, int p, void* a_cm, void* b_cm, void* stream) {
  EVO_CHECK_ARG(y && a_cm && b_cm, EVO_ERR_ARG, "tri_gate: null pointer");
  EVO_CHECK_ARG(hz % 8 == 0 && al16(y), EVO_ERR_ALIGN, "tri_gate: hz %% 8 and 16B aligned Y");
  if (rows == 0) return EVO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned g = (unsigned)((rows + (p <= 32 ? 63 : 31)) / (p <= 32 ? 64 : 32));
  // paired 4-byte stores need an even row count and 4-byte aligned channel-major outputs
  const bool pairs = (rows & 1) == 0 && ((uintptr_t)a_cm & 3) == 0 && ((uintptr_t)b_cm & 3) == 0;
#define TG(PP) ::evo::pdl_launch(tri_gate_fwd_k<PP>, g, 256, 0, st, (const bf16*)y, rows, hz, (bf16*)a_cm, (bf16*)b_cm, pairs)
  switch (p) {
    case 2: TG(2); break;
    case 4: TG(4); break;
    case 8: TG(8); break;
    case 16: TG(16); break;
    case 32: TG(32); break;
    case 64: TG(64); break;
    default: set_error("tri_gate: hidden_proj %d unsupported (2,4,8,16,32,64)", p); return EVO_ERR_SHAPE;
  }
#undef TG
  EVO_LAUNCH_CHECK("tri_gate fwd");
  return EVO_OK;
}

extern "C" int evo_tri_gate_bwd(const void* y, const void* da_cm, const void* db_cm, int d_dtype, int64_t rows, int hz,
                                int p, void* dy, float* dsum, void* stream) {
  EVO_CHECK_ARG(y && da_cm && db_cm && dy, EVO_ERR_ARG, "tri_gate bwd: null pointer");
  EVO_CHECK_ARG(hz % 8 == 0 && al16(y) && al16(dy), EVO_ERR_ALIGN, "tri_gate bwd: alignment");
  if (rows == 0) return EVO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned g = (unsigned)((rows + 63) / 64);
#define TGB(PP)                                                                                                  \
  (d_dtype == EVO_BF16                                                                                           \
       ? ::evo::pdl_launch(tri_gate_bwd_k<PP, bf16>, g, 256, 0, st, (const bf16*)y, (const bf16*)da_cm, (const bf16*)db_cm, rows, \
                                                     hz, (bf16*)dy, dsum)                                        \
       : ::evo::pdl_launch(tri_gate_bwd_k<PP, float>, g, 256, 0, st, (const bf16*)y, (const float*)da_cm, (const float*)db_cm,    \
                                                      rows, hz, (bf16*)dy, dsum))
  switch (p) {
    case 2: TGB(2); break;
    case 4: TGB(4); break;
    case 8: TGB(8); break;
    case 16: TGB(16); break;
    case 32: TGB(32); break;
    case 64: TGB(64); break;
    default: set_error("tri_gate bwd: hidden_proj %d unsupported", p); return EVO_ERR_SHAPE;
  }
#undef TGB
  EVO_LAUNCH_CHECK("tri_gate bwd");
  return EVO_OK;
}

extern "C" int evo_count_nonfinite(const void* x, int dtype, int64_t n, unsigned int* counter, void* stream) {
  EVO_CHECK_ARG(x && counter, EVO_ERR_ARG, "count_nonfinite: null pointer");
  if (n == 0) return EVO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned g = grid_for(n, 256);
  if (dtype == EVO_BF16) ::evo::pdl_launch(count_nonfinite_k<bf16>, g, 256, 0, st, (const bf16*)x, n, counter);
  else ::evo::pdl_launch(count_nonfinite_k<float>, g, 256, 0, st, (const float*)x, n, counter);
  EVO_LAUNCH_CHECK("count_nonfinite");
  return EVO_OK;
}

extern "C" int evo_residual_layernorm_fwd(const void* res, const void* y, int64_t y_rs, const float* bias,
                                          const void* gp, int64_t gp_rs, void* out, const float* gamma,
                                          const float* beta, void* ln, float* mean, float* rstd, int64_t rows,
                                          int64_t cols, float eps, void* stream) {
  EVO_CHECK_ARG(res && y && out && gamma && beta && ln, EVO_ERR_ARG, "residual_layernorm: null pointer");
  EVO_CHECK_ARG(cols == 32 || cols == 64 || cols == 128 || cols == 256, EVO_ERR_SHAPE,
                "residual_layernorm: cols must be 32/64/128/256 (got %lld)", (long long)cols);
  EVO_CHECK_ARG(y_rs % 8 == 0 && (!gp || gp_rs % 8 == 0) && al16(res) && al16(y) && al16(out) && al16(ln) &&
                    (!gp || al16(gp)),
                EVO_ERR_ALIGN, "residual_layernorm: 16-byte aligned rows required");
  if (rows == 0) return EVO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rpw = 32 / (cols / 8);
  int64_t need = (rows + 8 * rpw * RLN_U - 1) / (8 * rpw * RLN_U), cap = (int64_t)sm_count() * RLN_MINB;
  dim3 g((unsigned)(need < cap ? need : cap));
#define RLN(CC) ::evo::pdl_launch(residual_ln_k<CC, RLN_U>, g, 256, 0, st, (const bf16*)res, (const bf16*)y, y_rs, bias, (const bf16*)gp, \
                                                        gp_rs, (bf16*)out, gamma, beta, (bf16*)ln, mean, rstd, rows, eps)
  switch (cols) {
    case 32: RLN(32); break;
    case 64: RLN(64); break;
    case 128: RLN(128); break;
    default: RLN(256); break;
  }
#undef RLN
  EVO_LAUNCH_CHECK("residual_layernorm fwd");
  return EVO_OK;
}

// ------------------------------------------------------------------ gate multiply
// out = act(gate) * (y + bias) elementwise over a [rows, cols] view with row strides;
// gate NULL -> factor 1, y NULL -> (y + bias) = 1.  The reference's private triangle helpers
// (_triangle_projections g = sigmoid(.), _triangle_finish g * (.), evoformer.py:258-270) and
// the engine's sigmoid_raw / relu_raw (engine.py:220-225) on the reference-API path; the
// block itself fuses these into its epilogues.
template <typename T>
__global__ void __launch_bounds__(256) gate_mul_k(const T* __restrict__ gate, int64_t gate_rs, int act,
                                                  const T* __restrict__ y, int64_t y_rs,
                                                  const float* __restrict__ bias, T* __restrict__ out,
                                                  int64_t out_rs, int64_t rows, int64_t cols) {
  pdl_wait();
  const int64_t n = rows * cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    float f = 1.f;
    if (y) f = (float)y[r * y_rs + c] + (bias ? bias[c] : 0.f);
    if (gate) {
      float gv = (float)gate[r * gate_rs + c];
      gv = act == 1 ? sigmoidf_(gv) : (act == 2 ? fmaxf(gv, 0.f) : gv);
      f = __fmul_rn(gv, f);
    }
    out[r * out_rs + c] = (T)f;
  }
}

extern "C" int evo_gate_mul_fwd(const void* gate, int64_t gate_rs, int gate_act, const void* y, int64_t y_rs,
                                const float* bias, void* out, int64_t out_rs, int dtype, int64_t rows, int64_t cols,
                                void* stream) {
  EVO_CHECK_ARG(out && (gate || y), EVO_ERR_ARG, "gate_mul: need out and at least one of gate / y");
  EVO_CHECK_ARG(gate_act >= 0 && gate_act <= 2, EVO_ERR_ARG, "gate_mul: act must be 0 (identity), 1 (sigmoid), 2 (relu)");
  EVO_CHECK_ARG(rows >= 0 && cols >= 0, EVO_ERR_SHAPE, "gate_mul: negative extent");
  if (rows == 0 || cols == 0) return EVO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned g = grid_for(rows * cols, 256);
  if (dtype == EVO_BF16)
    ::evo::pdl_launch(gate_mul_k<bf16>, g, 256, 0, st, (const bf16*)gate, gate_rs, gate_act, (const bf16*)y, y_rs, bias, (bf16*)out,
                                        out_rs, rows, cols);
  else
    ::evo::pdl_launch(gate_mul_k<float>, g, 256, 0, st, (const float*)gate, gate_rs, gate_act, (const float*)y, y_rs, bias,
                                         (float*)out, out_rs, rows, cols);
  EVO_LAUNCH_CHECK("gate_mul fwd");
  return EVO_OK;
}

// Per-key bias gradient (fp32 [B][nh][L], accumulated by the attention backward) into the bias
// columns of the qkv gradient: dst[b, l, h] = bf16(dbias[b, h, l]) for h < nh, 0 for nh <= h <
// cols (the row padding of the fused projection).  One thread per (b, l): nh coalesced reads
// across the warp, one 16-byte store for the usual 8 columns.
__global__ void __launch_bounds__(256) key_bias_cols_k(const float* __restrict__ dbias, int64_t B, int nh, int64_t L,
                                                       bf16* __restrict__ dst, int64_t sb, int64_t sl, int cols) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * L) return;
  const int64_t b = i / L, l = i - b * L;
  bf16* d = dst + b * sb + l * sl;
  float v[8];
#pragma unroll
  for (int h = 0; h < 8; ++h) v[h] = h < nh ? dbias[(b * nh + h) * L + l] : 0.f;
  if (cols == 8 && ((uintptr_t)d & 15) == 0) {
    uint4 u;
    u.x = pack_bf16x2(v[0], v[1]); u.y = pack_bf16x2(v[2], v[3]);
    u.z = pack_bf16x2(v[4], v[5]); u.w = pack_bf16x2(v[6], v[7]);
    *reinterpret_cast<uint4*>(d) = u;
  } else {
    for (int h = 0; h < cols; ++h) d[h] = f2bf(h < 8 ? v[h] : (h < nh ? dbias[(b * nh + h) * L + l] : 0.f));
  }
}

extern "C" int evo_key_bias_grad_cols(const float* dbias, int64_t B, int nh, int64_t L, void* dst, int64_t dst_sb,
                                      int64_t dst_sl, int cols, void* stream) {
  EVO_CHECK_ARG(dbias && dst, EVO_ERR_ARG, "key_bias_grad_cols: null pointer");
  EVO_CHECK_ARG(B >= 0 && L >= 0 && nh >= 1 && cols >= nh, EVO_ERR_SHAPE, "key_bias_grad_cols: bad extents");
  if (B * L == 0) return EVO_OK;
  ::evo::pdl_launch(key_bias_cols_k, grid_for(B * L, 256), 256, 0, (cudaStream_t)stream, dbias, B, nh, L, (bf16*)dst, dst_sb, dst_sl,
                                                                          cols);
  EVO_LAUNCH_CHECK("key_bias_grad_cols");
  return EVO_OK;
}
