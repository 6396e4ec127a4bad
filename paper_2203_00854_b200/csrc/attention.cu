// Gated multi-head attention with bias on tcgen05 (replaces the per-head loop of
// _attention_core, evoformer.py:173-198, for msa_row / msa_col / pair_row / pair_col).
//
// One CTA (4 warps, 128 threads) owns 128 queries of one (batch, head) and streams
// the keys in tiles of 64 (flash-style online softmax, so N_r = 4096 never
// materialises a logit matrix).  <= 128 registers, 64 TMEM columns and ~41 KB of
// shared memory per CTA -> 4 CTAs (16 warps) per SM hide each other's latency:
//   S   = Q K^T                 tcgen05.mma M=128 N=64 K=16..64   -> TMEM (fp32)
//   s   = (S + bias) * scale    thread r owns query row r (tcgen05.ld 32x32b),
//   p   = exp2(s - m)           running max / sum in registers (no shuffles)
//   P  -> smem (bf16, canonical K-major, conflict-free 16-byte stores)
//   O  += P V                   tcgen05.mma M=128 N=c K=64 -> TMEM -> registers
// Epilogue: o = O / l, out = sigmoid(g) * o (gate on raw x, G2), log-sum-exp saved.
// K/V tiles are double-buffered with cp.async; several CTAs per SM overlap the
// MMA of one CTA with the softmax of another.
#include "attn.cuh"

namespace evo {

constexpr int ATT_BQ = 128;
constexpr int ATT_BK = 64;   // keys per tile: S = 64 TMEM columns, P = 16 KB
constexpr float LOG2E = 1.4426950408889634f;


template <int CP>
struct AttnSmem {
  static constexpr uint32_t Q = 0;
  static constexpr uint32_t KT = Q + ATT_BQ * CP * 2;          // 2 stages
  static constexpr uint32_t VT = KT + 2 * ATT_BK * CP * 2;     // 2 stages
  static constexpr uint32_t P = VT + 2 * ATT_BK * CP * 2;
  static constexpr uint32_t BIAS = P + ATT_BQ * ATT_BK * 2;    // 2 x 128 fp32 (per-key bias)
  static constexpr uint32_t TOTAL = BIAS + 2 * ATT_BK * 4;
};

// ROWS x CP K-major tile from a strided [row][col] source (cols contiguous)
template <int CP, int ROWS>
__device__ __forceinline__ void att_load_kmajor(uint32_t sdst, const bf16* base, int64_t row_stride, int row0,
                                                int nrows_valid, int c) {
  constexpr int CPR = CP / 8;
#pragma unroll
  for (int it = 0; it < ROWS * CPR / 128; ++it) {
    const int ch = threadIdx.x + it * 128;
    const int r = ch / CPR, d = (ch % CPR) * 8;
    const bool ok = (r < nrows_valid) && (d < c);
    const bf16* src = ok ? base + (int64_t)(row0 + r) * row_stride + d : base;
    cp_async16(sdst + kmajor_off(r, d, ROWS), src, ok);
  }
}
// keys x CP tile stored MN-major over d (the PV B operand: N = d, K = key)
template <int CP>
__device__ __forceinline__ void att_load_v(uint32_t sdst, const bf16* base, int64_t row_stride, int row0,
                                           int nrows_valid, int c) {
  constexpr int CPR = CP / 8;
#pragma unroll
  for (int it = 0; it < ATT_BK * CPR / 128; ++it) {
    const int ch = threadIdx.x + it * 128;
    const int r = ch / CPR, d = (ch % CPR) * 8;
    const bool ok = (r < nrows_valid) && (d < c);
    const bf16* src = ok ? base + (int64_t)(row0 + r) * row_stride + d : base;
    cp_async16(sdst + mnmajor_off(d, r, CP), src, ok);
  }
}

template <int CP>
__global__ void __launch_bounds__(128, CP == 32 ? 4 : 3) attn_fwd_kernel(AttnParams P) {
  using SM = AttnSmem<CP>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_s, bar_o;
  __shared__ uint32_t tmem_sh;
  const uint32_t sb = smem_u32(smem);
  float* sbias = reinterpret_cast<float*>(smem + SM::BIAS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = blockIdx.x * ATT_BQ;
  const int h = blockIdx.y;
  const int64_t b = blockIdx.z;
  const int L = P.L, c = P.c;
  const int r = warp * 32 + lane;  // query row inside the tile
  const int qi = q0 + r;
  const bool per_key_bias = P.bias && P.bs2 == 0;

  if (warp == 0) tmem_alloc(&tmem_sh, ATT_BK);
  if (threadIdx.x == 0) {
    mbar_init(&bar_s, 1);
    mbar_init(&bar_o, 1);
    fence_mbar_init();
  }

  const bf16* qb = P.q + b * P.q_sb + (int64_t)h * c;
  const bf16* kb = P.k + b * P.k_sb + (int64_t)h * c;
  const bf16* vb = P.v + b * P.v_sb + (int64_t)h * c;
  att_load_kmajor<CP, ATT_BQ>(sb + SM::Q, qb, P.q_sl, q0, L - q0, c);
  att_load_kmajor<CP, ATT_BK>(sb + SM::KT, kb, P.k_sl, 0, L, c);
  att_load_v<CP>(sb + SM::VT, vb, P.v_sl, 0, L, c);
  cp_async_commit();

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;
  const uint32_t t_row = tmem + ((uint32_t)(warp * 32) << 16);

  constexpr uint32_t IDESC_S = make_idesc_bf16(128, ATT_BK, 0, 0);
  constexpr uint32_t IDESC_O = make_idesc_bf16(128, CP, 0, 1);

  float m_run = -INFINITY, l_run = 0.f;
  float o_acc[CP];
#pragma unroll
  for (int d = 0; d < CP; ++d) o_acc[d] = 0.f;

  const int nkt = (L + ATT_BK - 1) / ATT_BK;
  const bf16* brow = nullptr;
  if (P.bias && !per_key_bias && qi < L) brow = P.bias + b * P.bs0 + (int64_t)h * P.bs1 + (int64_t)qi * P.bs2;

  for (int j = 0; j < nkt; ++j) {
    const int k0 = j * ATT_BK;
    const int st = j & 1;
    if (per_key_bias) {
      const bf16* bp = P.bias + b * P.bs0 + (int64_t)h * P.bs1;
      const int kk = threadIdx.x;
      if (kk < ATT_BK) sbias[st * ATT_BK + kk] = (k0 + kk < L) ? bf2f(bp[(int64_t)(k0 + kk) * P.bs3]) : 0.f;
    }
    cp_async_wait<0>();
    fence_async_smem();
    __syncthreads();
    // prefetch the next K/V tile into the other stage (its MMAs finished last iteration)
    if (j + 1 < nkt) {
      att_load_kmajor<CP, ATT_BK>(sb + SM::KT + (st ^ 1) * ATT_BK * CP * 2, kb, P.k_sl, k0 + ATT_BK,
                                  L - k0 - ATT_BK, c);
      att_load_v<CP>(sb + SM::VT + (st ^ 1) * ATT_BK * CP * 2, vb, P.v_sl, k0 + ATT_BK, L - k0 - ATT_BK, c);
    }
    cp_async_commit();

    if (threadIdx.x == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < CP / 16; ++kk) {
        uint64_t ad = make_sdesc(sb + SM::Q + kk * 2 * (128 / 8) * 128, (128 / 8) * 128, 128);
        uint64_t bd = make_sdesc(sb + SM::KT + st * ATT_BK * CP * 2 + kk * 2 * (ATT_BK / 8) * 128,
                                 (ATT_BK / 8) * 128, 128);
        mma_bf16(tmem, ad, bd, IDESC_S, kk != 0);
      }
      mma_commit(&bar_s);
    }
    mbar_wait(&bar_s, j & 1);
    tc_fence_after();

    float s[ATT_BK];
#pragma unroll
    for (int cc = 0; cc < ATT_BK; cc += 32) tmem_ld32(t_row + cc, s + cc);
    tmem_ld_wait();

    // bias (before the scale, G1); keys >= L masked on the last tile only
    const bool full_tile = k0 + ATT_BK <= L;
    if (brow) {
      if (P.bias_vec && full_tile) {
#pragma unroll
        for (int kk = 0; kk < ATT_BK; kk += 8) {
          uint4 u = *reinterpret_cast<const uint4*>(brow + k0 + kk);
          float t[8];
          unpack_bf16x2(u.x, t[0], t[1]); unpack_bf16x2(u.y, t[2], t[3]);
          unpack_bf16x2(u.z, t[4], t[5]); unpack_bf16x2(u.w, t[6], t[7]);
#pragma unroll
          for (int e = 0; e < 8; ++e) s[kk + e] += t[e];
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < ATT_BK; ++kk)
          if (k0 + kk < L) s[kk] += bf2f(brow[(int64_t)(k0 + kk) * P.bs3]);
      }
    } else if (per_key_bias) {
#pragma unroll
      for (int kk = 0; kk < ATT_BK; kk += 4) {
        const float4 bv = *reinterpret_cast<const float4*>(sbias + st * ATT_BK + kk);
        s[kk] += bv.x; s[kk + 1] += bv.y; s[kk + 2] += bv.z; s[kk + 3] += bv.w;
      }
    }
    if (!full_tile) {
#pragma unroll
      for (int kk = 0; kk < ATT_BK; ++kk)
        if (k0 + kk >= L) s[kk] = -INFINITY;
    }
    // running max on the unscaled logits (scale > 0), p = 2^(s*scale*log2e - m*scale*log2e)
    float mx = m_run;
#pragma unroll
    for (int kk = 0; kk < ATT_BK; kk += 2) mx = fmaxf(mx, fmaxf(s[kk], s[kk + 1]));
    const float corr = ex2f((m_run - mx) * P.scale_log2);  // m_run = -inf on the first tile -> 0
    const float mxs = mx * P.scale_log2;
    float lsum = 0.f;
    const uint32_t prow = sb + SM::P;
#pragma unroll
    for (int kk = 0; kk < ATT_BK; kk += 8) {
      float pv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        pv[e] = ex2f(fmaf(s[kk + e], P.scale_log2, -mxs));
        lsum += pv[e];
      }
      st_shared_v4(prow + kmajor_off(r, kk, ATT_BQ), pack_bf16x2(pv[0], pv[1]), pack_bf16x2(pv[2], pv[3]),
                   pack_bf16x2(pv[4], pv[5]), pack_bf16x2(pv[6], pv[7]));
    }
    l_run = l_run * corr + lsum;
    m_run = mx;
#pragma unroll
    for (int d = 0; d < CP; ++d) o_acc[d] *= corr;

    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < ATT_BK / 16; ++kk) {
        uint64_t ad = make_sdesc(sb + SM::P + kk * 2 * (128 / 8) * 128, (128 / 8) * 128, 128);
        uint64_t bd = make_sdesc(sb + SM::VT + st * ATT_BK * CP * 2 + kk * 2 * (CP / 8) * 128, (CP / 8) * 128, 128);
        mma_bf16(tmem, ad, bd, IDESC_O, kk != 0);
      }
      mma_commit(&bar_o);
    }
    mbar_wait(&bar_o, j & 1);
    tc_fence_after();
    float ov[CP];
    if constexpr (CP == 16) {
      tmem_ld16(t_row, ov);
    } else {
#pragma unroll
      for (int cc = 0; cc < CP; cc += 32) tmem_ld32(t_row + cc, ov + cc);
    }
    tmem_ld_wait();
#pragma unroll
    for (int d = 0; d < CP; ++d) o_acc[d] += ov[d];
    tc_fence_before();
    __syncthreads();  // all TMEM reads done before the next S MMA overwrites the columns
  }

  if (qi < L) {
    const float inv = rcpf(l_run);
    const bf16* gp = P.g + b * P.g_sb + (int64_t)qi * P.g_sl + (int64_t)h * c;
    bf16* og = P.og + b * P.o_sb + (int64_t)qi * P.o_sl + (int64_t)h * c;
    bf16* orw = P.orw ? P.orw + b * P.r_sb + (int64_t)qi * P.r_sl + (int64_t)h * c : nullptr;
#pragma unroll
    for (int d = 0; d < CP; d += 8) {
      if (d < c) {
        float o[8], gv[8];
        uint4 u = *reinterpret_cast<const uint4*>(gp + d);
        unpack_bf16x2(u.x, gv[0], gv[1]); unpack_bf16x2(u.y, gv[2], gv[3]);
        unpack_bf16x2(u.z, gv[4], gv[5]); unpack_bf16x2(u.w, gv[6], gv[7]);
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = o_acc[d + e] * inv;
        if (orw) {
          uint4 w;
          w.x = pack_bf16x2(o[0], o[1]); w.y = pack_bf16x2(o[2], o[3]);
          w.z = pack_bf16x2(o[4], o[5]); w.w = pack_bf16x2(o[6], o[7]);
          *reinterpret_cast<uint4*>(orw + d) = w;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] *= sigmoidf_(gv[e]);
        uint4 w;
        w.x = pack_bf16x2(o[0], o[1]); w.y = pack_bf16x2(o[2], o[3]);
        w.z = pack_bf16x2(o[4], o[5]); w.w = pack_bf16x2(o[6], o[7]);
        *reinterpret_cast<uint4*>(og + d) = w;
      }
    }
    if (P.lse) P.lse[(b * P.H + h) * (int64_t)L + qi] = (m_run * P.scale_log2 + log2f(l_run)) * 0.6931471805599453f;
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, ATT_BK);
}

static bool a16(const void* p) { return ((uintptr_t)p & 15) == 0; }

template <int CP>
static int launch_attn_fwd(const AttnParams& p, int64_t B, cudaStream_t st) {
  using SM = AttnSmem<CP>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel<CP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM::TOTAL);
    if (e != cudaSuccess) return cuda_status(e, "attn fwd attr");
    attr = true;
  }
  dim3 grid((unsigned)((p.L + ATT_BQ - 1) / ATT_BQ), (unsigned)p.H, (unsigned)B);
  attn_fwd_kernel<CP><<<grid, 128, SM::TOTAL, st>>>(p);
  EVO_LAUNCH_CHECK("attention fwd");
  return EVO_OK;
}

int attn_params_from_desc(const EvoAttnDesc* d, AttnParams& p) {
  EVO_CHECK_ARG(d && d->q && d->k && d->v && d->g && d->o_gated, EVO_ERR_ARG, "attention: null pointer");
  EVO_CHECK_ARG(d->B >= 1 && d->L >= 1 && d->H >= 1 && d->c >= 8, EVO_ERR_SHAPE, "attention: bad extents");
  EVO_CHECK_ARG(d->c % 8 == 0 && d->c <= 64, EVO_ERR_SHAPE, "attention: head dim must be a multiple of 8, <= 64 (got %d)", d->c);
  EVO_CHECK_ARG(d->B < 65536 && d->H < 65536 && d->L < (1 << 30), EVO_ERR_SHAPE, "attention: extents too large");
  EVO_CHECK_ARG(d->scale > 0.f, EVO_ERR_ARG, "attention: scale must be positive");
  const int64_t strides[] = {d->q_sb, d->q_sl, d->k_sb, d->k_sl, d->v_sb, d->v_sl, d->g_sb, d->g_sl,
                             d->o_sb, d->o_sl, d->r_sb, d->r_sl};
  for (int64_t s : strides) EVO_CHECK_ARG(s % 8 == 0, EVO_ERR_ALIGN, "attention: strides must be multiples of 8");
  EVO_CHECK_ARG(a16(d->q) && a16(d->k) && a16(d->v) && a16(d->g) && a16(d->o_gated) && a16(d->o_raw), EVO_ERR_ALIGN,
                "attention: pointers must be 16B aligned");
  p.q = (const bf16*)d->q; p.k = (const bf16*)d->k; p.v = (const bf16*)d->v; p.g = (const bf16*)d->g;
  p.bias = (const bf16*)d->bias;
  p.q_sb = d->q_sb; p.q_sl = d->q_sl; p.k_sb = d->k_sb; p.k_sl = d->k_sl;
  p.v_sb = d->v_sb; p.v_sl = d->v_sl; p.g_sb = d->g_sb; p.g_sl = d->g_sl;
  p.bs0 = d->bias_s[0]; p.bs1 = d->bias_s[1]; p.bs2 = d->bias_s[2]; p.bs3 = d->bias_s[3];
  p.bias_vec = p.bias && p.bs3 == 1 && a16(p.bias) && p.bs0 % 8 == 0 && p.bs1 % 8 == 0 && p.bs2 % 8 == 0;
  p.og = (bf16*)d->o_gated; p.orw = (bf16*)d->o_raw;
  p.o_sb = d->o_sb; p.o_sl = d->o_sl; p.r_sb = d->r_sb; p.r_sl = d->r_sl;
  p.lse = d->lse;
  p.L = (int)d->L; p.H = d->H; p.c = d->c;
  p.scale_log2 = d->scale * LOG2E;
  return EVO_OK;
}

}  // namespace evo

using namespace evo;

namespace evo {
template <int CP>
int launch_attn_fwd_ws(const AttnParams& p, int64_t B, cudaStream_t st);
// sequences at least this long take the warp-specialised kernel (attention_ws.cu)
static int g_ws_min_len = 2048;  // measured: faster than attn_fwd_kernel from N_r = 2048 on
}  // namespace evo

extern "C" int evo_attention_fwd_ws_min_len(int len) {
  const int old = g_ws_min_len;
  if (len > 0) g_ws_min_len = len;
  return old;
}

extern "C" int evo_gated_attention_fwd(const EvoAttnDesc* d, void* stream) {
  AttnParams p;
  int rc = attn_params_from_desc(d, p);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const bool ws_bias_ok = true;
  if (p.L >= g_ws_min_len && ws_bias_ok) {
    if (p.c <= 16) return launch_attn_fwd_ws<16>(p, d->B, st);
    if (p.c <= 32) return launch_attn_fwd_ws<32>(p, d->B, st);
    return launch_attn_fwd_ws<64>(p, d->B, st);
  }
  if (p.c <= 16) return launch_attn_fwd<16>(p, d->B, st);
  if (p.c <= 32) return launch_attn_fwd<32>(p, d->B, st);
  return launch_attn_fwd<64>(p, d->B, st);
}
