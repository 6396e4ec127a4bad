// Backward of the gated attention with bias (evoformer.py:173-198), flash-style on
// tcgen05.  The reference has no backward; the gradient oracle is
// the torch float64 restatement in oracle/evoformer_torch.py.
//
//   prep   one warp per (batch, position) row: dO = dout*sigmoid(g) (bf16), dg = dout*O*s(1-s),
//          D = rowsum(dO*O) and lse*log2(e) per (batch, head, query), so the main loop's
//          per-tile operands are all plain cp.async copies prefetched behind the TMEM drain
//   main   one CTA = (batch, head, 128-key tile), 8 warps, loops over 128-query tiles:
//            S^T  = K Q^T            (tcgen05, M=keys N=queries)  -> TMEM cols [0,128)
//            dP^T = V dO^T           (tcgen05)                    -> TMEM cols [128,256)
//            P^T  = exp2(S^T*scale + bias - lse), dS^T = P^T (dP^T - D)   (registers)
//            P^T, dS^T -> smem (bf16, canonical K-major [key][query])
//            dV  += P^T dO,  dK += dS^T Q   (accumulated in TMEM over query tiles)
//            dQ_t = dS K  (same smem tile read as its transpose by swapping the
//                   descriptor's LBO/SBO and the major bit) -> fp32 atomics
//            dbias: per-key bias pre-reduced over queries (one atomic per key); a bias shared
//            over the batch (msa_row) copies the dS^T smem tile to a bf16 workspace with
//            16-byte stores and attn_dbias_reduce sums it over the batch (deterministic)
//   finish dq = bf16(dQ accumulator)
#include <cstdlib>
#include <cstring>

#include "attn.cuh"
#include "tma.cuh"

#ifndef EVO_EXP
#define EVO_EXP 0
#endif

namespace evo {

#if EVO_EXP == 10 || EVO_EXP == 11
__device__ unsigned long long g_bwd_trace[8192];
#define BTRACE(i)                                                                              \
  do {                                                                                         \
    if (blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == 128) && (i) < 4096) {           \
      unsigned long long t_;                                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                   \
      g_bwd_trace[(threadIdx.x == 128 ? 4096 : 0) + (i)] = t_;                                 \
    }                                                                                          \
  } while (0)
#else
#define BTRACE(i) (void)0
#endif


struct AttnBwdParams {
  AttnParams f;
  const bf16* dout;
  int64_t do_sb, do_sl;
  bf16 *dq, *dk, *dv, *dg;
  int64_t dq_sb, dq_sl, dk_sb, dk_sl, dv_sb, dv_sl, dg_sb, dg_sl;
  float* dbias;
  int64_t db0, db1, db2, db3;
  bf16* dO;      // workspace [B][L][H*c]
  float* dQacc;  // workspace [B][L][H*c]
  float* Dsum;   // workspace [B][H][L]
  float* lse2;   // workspace [B][H][L]: lse * log2(e)
  bf16* dS;      // workspace [B][H][key][query] (batch-shared bias only, unscaled) or null
  float scale;
  int64_t B;
};

// dbias[h][q][k] += scale * sum_b dS[b][h][k][q]   (batch-shared bias: msa_row, evoformer.py:214).
// CTA = one (head, 32-key, 32-query) tile; 256 threads = 2 batch slices x 32 keys x 4 16-byte query
// vectors, each thread keeping U loads of its slice's batches in flight (each warp reads 8 key rows
// x 64 contiguous bytes).  The two slices meet in smem in a fixed order (deterministic, no
// atomics) and the tile leaves transposed: a warp writes 32 consecutive keys of one query
// (coalesced; the dS^T workspace is key-major because the backward's threads own keys).
__global__ void __launch_bounds__(256) attn_dbias_reduce(const bf16* __restrict__ dS, float* __restrict__ dbias,
                                                         int64_t B, int H, int L, int64_t d1, int64_t d2, int64_t d3,
                                                         float scale) {
  pdl_wait();
  constexpr int U = 8;
  __shared__ float part[2][32][33];
  const int h = blockIdx.z, k0 = blockIdx.y * 32, q0 = blockIdx.x * 32;
  const int t = threadIdx.x, slice = t >> 7, key = (t >> 2) & 31, qv = t & 3;
  const int64_t per = (int64_t)H * L * L;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  if (k0 + key < L && q0 + qv * 8 < L) {  // L % 8 == 0 (host-checked): whole vectors
    const bf16* src = dS + ((int64_t)h * L + k0 + key) * L + q0 + qv * 8;
    int64_t b = slice;
    for (; b + 2 * (U - 1) < B; b += 2 * U) {
      uint4 u[U];
#pragma unroll
      for (int i = 0; i < U; ++i) u[i] = __ldcs(reinterpret_cast<const uint4*>(src + (b + 2 * i) * per));
#pragma unroll
      for (int i = 0; i < U; ++i) {
        float v[8];
        unpack_bf16x2(u[i].x, v[0], v[1]); unpack_bf16x2(u[i].y, v[2], v[3]);
        unpack_bf16x2(u[i].z, v[4], v[5]); unpack_bf16x2(u[i].w, v[6], v[7]);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += v[e];
      }
    }
    for (; b < B; b += 2) {
      const uint4 u = __ldcs(reinterpret_cast<const uint4*>(src + b * per));
      float v[8];
      unpack_bf16x2(u.x, v[0], v[1]); unpack_bf16x2(u.y, v[2], v[3]);
      unpack_bf16x2(u.z, v[4], v[5]); unpack_bf16x2(u.w, v[6], v[7]);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += v[e];
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) part[slice][key][qv * 8 + e] = acc[e];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int q = (t >> 5) + 8 * i, k = t & 31;
    if (q0 + q < L && k0 + k < L)
      dbias[h * d1 + (int64_t)(q0 + q) * d2 + (int64_t)(k0 + k) * d3] += scale * (part[0][k][q] + part[1][k][q]);
  }
}

// Same reduction with 64-query tiles (L % 64 == 0): 512 threads = 2 batch slices x 32 keys x 8 16-byte
// query vectors, so every warp reads 4 key rows x 128 contiguous bytes (whole DRAM bursts instead of
// 64-byte halves)
__global__ void __launch_bounds__(512) attn_dbias_reduce64(const bf16* __restrict__ dS, float* __restrict__ dbias,
                                                           int64_t B, int H, int L, int64_t d1, int64_t d2, int64_t d3,
                                                           float scale) {
  pdl_wait();
  constexpr int U = 8;
  __shared__ float part[2][32][65];
  const int h = blockIdx.z, k0 = blockIdx.y * 32, q0 = blockIdx.x * 64;
  const int t = threadIdx.x, slice = t >> 8, key = (t >> 3) & 31, qv = t & 7;
  const int64_t per = (int64_t)H * L * L;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  if (k0 + key < L) {
    const bf16* src = dS + ((int64_t)h * L + k0 + key) * L + q0 + qv * 8;
    int64_t b = slice;
    for (; b + 2 * (U - 1) < B; b += 2 * U) {
      uint4 u[U];
#pragma unroll
      for (int i = 0; i < U; ++i) u[i] = __ldcs(reinterpret_cast<const uint4*>(src + (b + 2 * i) * per));
#pragma unroll
      for (int i = 0; i < U; ++i) {
        float v[8];
        unpack_bf16x2(u[i].x, v[0], v[1]); unpack_bf16x2(u[i].y, v[2], v[3]);
        unpack_bf16x2(u[i].z, v[4], v[5]); unpack_bf16x2(u[i].w, v[6], v[7]);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += v[e];
      }
    }
    for (; b < B; b += 2) {
      const uint4 u = __ldcs(reinterpret_cast<const uint4*>(src + b * per));
      float v[8];
      unpack_bf16x2(u.x, v[0], v[1]); unpack_bf16x2(u.y, v[2], v[3]);
      unpack_bf16x2(u.z, v[4], v[5]); unpack_bf16x2(u.w, v[6], v[7]);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += v[e];
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) part[slice][key][qv * 8 + e] = acc[e];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int q = (t >> 5) + 16 * i, k = t & 31;
    if (k0 + k < L)
      dbias[h * d1 + (int64_t)(q0 + q) * d2 + (int64_t)(k0 + k) * d3] += scale * (part[0][k][q] + part[1][k][q]);
  }
}

// bias_t[h][k][q] = bias[h*s1 + q*s2 + k]  (batch-shared full bias, keys contiguous in the
// source): the backward's threads own keys, so the transposed copy turns 16 strided 2-byte
// loads per thread and query group into two 16-byte loads.  32x32 tiles through smem.
__global__ void __launch_bounds__(256) attn_bias_transpose(const bf16* __restrict__ bias, int64_t s1, int64_t s2,
                                                           bf16* __restrict__ bias_t, int L) {
  pdl_wait();
  __shared__ bf16 tile[32][33];
  const int h = blockIdx.z;
  const int q0 = blockIdx.y * 32, k0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int q = q0 + r, k = k0 + tx;
    tile[r][tx] = (q < L && k < L) ? bias[h * s1 + (int64_t)q * s2 + k] : f2bf(0.f);
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int k = k0 + r, q = q0 + tx;
    if (q < L && k < L) bias_t[((int64_t)h * L + k) * L + q] = tile[tx][r];
  }
}

// 64-byte-swizzled operand tiles (TMA path, head dim 32): [128 rows][32 elements], 8-row atoms of 512 B.
// K-major read (k = the 32 channels): k-step of 16 = +32 B inside the row; MN-major view of the same
// tile (mn = channels, k = rows): k-step of 16 rows = +1024 B
__device__ __forceinline__ uint64_t bw_sw64_k(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(512 >> 4) << 32) | (1ull << 46) | (4ull << 61);
}
__device__ __forceinline__ uint64_t bw_sw64_mn(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(4096 >> 4) << 16) | ((uint64_t)(512 >> 4) << 32) |
         (1ull << 46) | (4ull << 61);
}

struct BwdMaps {  // tensor maps of the per-tile operands (TMA path): element (d, h, l, b)
  CUtensorMap q, k, v, dO;
  CUtensorMap bt;  // msa_row: transposed batch-shared bias [h][key][query], box [136 q][128 keys]
  CUtensorMap ws;  // msa_row: dS^T workspace [b*H + h][key][query] in the canonical tile order (store)
};
__device__ __forceinline__ void tma_st5(uint64_t m, uint32_t src, int c0, int c1, int c2, int c3, int c4) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];\n"
               ::"l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(src) : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

// ---------------------------------------------------------------------------------- prep
// The (row = (b, l), 8-channel chunk) pairs are flattened; a warp owns PREP_PASSES x 32
// consecutive pairs (no idle lanes for any H*c), and issues every global load of them (dout,
// g, o, lse) before any math, so it pays one memory latency per PREP_PASSES passes.  The
// lanes of one head are consecutive and never straddle rows (c/8 divides 32 and H*c/8).
constexpr int PREP_PASSES = 2;  // measured: 2 beats 4 (more resident CTAs, load/store phases overlap) and 1
// STAGED (when H*c/8 divides the CTA's 8*32*PREP_PASSES chunks: the CTA covers whole rows): the
// per-(b, h, l) statistics D and lse*log2e go through smem and are written (and lse read) as
// runs of consecutive l per head instead of one scattered 4-byte access per head and row.
// Index math: the (row, chunk), (b, l) and (chunk -> head) splits are shifts when H*c/8, L and c are
// powers of two (every Evoformer shape; POW2), else 32-bit divisions.  The division form dominated
// the instruction count (ncu: issue-active 68 %, ~12 emulated divisions per thread), so the splits are
// also computed once per pass and reused by the math loop.
struct PrepIdx {
  uint32_t nch, L, c;
  int sh_nch, sh_L, sh_c;
};
template <bool POW2>
__device__ __forceinline__ uint32_t pdiv(uint32_t x, uint32_t d, int sh) { return POW2 ? x >> sh : x / d; }

template <bool STAGED, bool POW2>
__global__ void __launch_bounds__(256) attn_bwd_prep(AttnBwdParams P, int64_t B, PrepIdx ix) {
  pdl_wait();
  constexpr int PER_CTA = 8 * PREP_PASSES * 32;
  __shared__ float s_D[STAGED ? PER_CTA : 1];
  const int lane = threadIdx.x & 31;
  const int L = P.f.L, H = P.f.H, c = P.f.c;
  const uint32_t nch = ix.nch;
  // 32-bit (row, chunk) / (b, l) splits: the host guarantees B*L*nch < 2^31
  const uint32_t total = (uint32_t)(B * L * nch);
  const uint32_t f0 = ((uint32_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * (PREP_PASSES * 32);
  if (!STAGED && f0 >= total) return;
  const int lanes_per_head = c / 8;  // 1, 2, 4 or 8
  const uint32_t row0 = (uint32_t)blockIdx.x * (PER_CTA / nch);  // STAGED: first row of this CTA
  uint4 ud[PREP_PASSES], ug[PREP_PASSES], uo[PREP_PASSES];
  float lse[PREP_PASSES];
  uint32_t rw[PREP_PASSES], bb[PREP_PASSES], ll[PREP_PASSES];
  int cl[PREP_PASSES];
#pragma unroll
  for (int t = 0; t < PREP_PASSES; ++t) {
    const uint32_t f = f0 + t * 32 + lane;
    const uint32_t row = pdiv<POW2>(f, nch, ix.sh_nch);
    const uint32_t bu = pdiv<POW2>(row, (uint32_t)L, ix.sh_L);
    rw[t] = row;
    bb[t] = bu;
    ll[t] = row - bu * (uint32_t)L;
    cl[t] = (int)(f - row * nch) * 8;
    if (f < total) {
      const int64_t b = bu, l = ll[t];
      const int col = cl[t];
      ud[t] = *reinterpret_cast<const uint4*>(P.dout + b * P.do_sb + l * P.do_sl + col);
      ug[t] = *reinterpret_cast<const uint4*>(P.f.g + b * P.f.g_sb + l * P.f.g_sl + col);
      uo[t] = *reinterpret_cast<const uint4*>(P.f.orw + b * P.f.r_sb + l * P.f.r_sl + col);
      if (!STAGED)
        lse[t] = (lane % lanes_per_head) == 0 ? P.f.lse[(b * H + pdiv<POW2>(col, c, ix.sh_c)) * (int64_t)L + l] : 0.f;
    }
  }
#pragma unroll
  for (int t = 0; t < PREP_PASSES; ++t) {
    const uint32_t f = f0 + t * 32 + lane;
    const bool ok = f < total;
    const uint32_t row = rw[t];
    const int col = cl[t];
    const int64_t b = bb[t], l = ll[t];
    float dsum = 0.f;
    if (ok) {
      float dout[8], g[8], o[8], dO[8], dg[8];
      unpack_bf16x2(ud[t].x, dout[0], dout[1]); unpack_bf16x2(ud[t].y, dout[2], dout[3]);
      unpack_bf16x2(ud[t].z, dout[4], dout[5]); unpack_bf16x2(ud[t].w, dout[6], dout[7]);
      unpack_bf16x2(ug[t].x, g[0], g[1]); unpack_bf16x2(ug[t].y, g[2], g[3]);
      unpack_bf16x2(ug[t].z, g[4], g[5]); unpack_bf16x2(ug[t].w, g[6], g[7]);
      unpack_bf16x2(uo[t].x, o[0], o[1]); unpack_bf16x2(uo[t].y, o[2], o[3]);
      unpack_bf16x2(uo[t].z, o[4], o[5]); unpack_bf16x2(uo[t].w, o[6], o[7]);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float sg = sigmoidf_(g[e]);
        dO[e] = dout[e] * sg;
        dg[e] = dout[e] * o[e] * sg * (1.f - sg);
      }
      uint4 w;
      w.x = pack_bf16x2(dO[0], dO[1]); w.y = pack_bf16x2(dO[2], dO[3]);
      w.z = pack_bf16x2(dO[4], dO[5]); w.w = pack_bf16x2(dO[6], dO[7]);
      // D of the bf16 dO the MMAs see (the packed values, unpacked: no second rounding pass)
      float r[8];
      unpack_bf16x2(w.x, r[0], r[1]); unpack_bf16x2(w.y, r[2], r[3]);
      unpack_bf16x2(w.z, r[4], r[5]); unpack_bf16x2(w.w, r[6], r[7]);
#pragma unroll
      for (int e = 0; e < 8; ++e) dsum = fmaf(r[e], o[e], dsum);
      *reinterpret_cast<uint4*>(P.dO + (int64_t)row * (H * c) + col) = w;
      w.x = pack_bf16x2(dg[0], dg[1]); w.y = pack_bf16x2(dg[2], dg[3]);
      w.z = pack_bf16x2(dg[4], dg[5]); w.w = pack_bf16x2(dg[6], dg[7]);
      *reinterpret_cast<uint4*>(P.dg + b * P.dg_sb + l * P.dg_sl + col) = w;
    }
    // segmented reduction over the lanes of one head (lanes_per_head is a power of 2)
    for (int o = 1; o < lanes_per_head; o <<= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
    if (ok && (lane % lanes_per_head) == 0) {
      const int hh = (int)pdiv<POW2>(col, c, ix.sh_c);
      if (STAGED) {
        s_D[(row - row0) * H + hh] = dsum;
      } else {
        const int64_t ixo = (b * H + hh) * (int64_t)L + l;
        P.Dsum[ixo] = dsum;
        P.lse2[ixo] = lse[t] * 1.4426950408889634f;
      }
    }
  }
  if (STAGED) {
    __syncthreads();
    const int R = PER_CTA / (int)nch;  // rows per CTA (a power of two when POW2)
    const uint32_t rows = (uint32_t)(B * L);
    for (int i = threadIdx.x; i < R * H; i += 256) {
      const int h = POW2 ? i >> (31 - __clz(R)) : i / R, rl = i - h * R;
      const uint32_t row = row0 + rl;
      if (row < rows) {
        const uint32_t bu = pdiv<POW2>(row, (uint32_t)L, ix.sh_L);
        const int64_t ixo = ((int64_t)bu * H + h) * L + (row - bu * (uint32_t)L);
        P.Dsum[ixo] = s_D[rl * H + h];
        P.lse2[ixo] = P.f.lse[ixo] * 1.4426950408889634f;
      }
    }
  }
}

// ---------------------------------------------------------------------------------- main
constexpr int BW_BK = 128;  // keys per CTA
constexpr int BW_BQ = 128;  // queries per iteration

template <int CP, bool BIASS = false>
struct BwdSmem {
  // PTM (head dim <= 32): P^T lives in TMEM (the dV MMA reads its A operand from there), and
  // the freed 32 KB double-buffer the per-query-tile operands (Q, dO, lse, D), so the next
  // query tile is loaded while this one computes.  Head dim 64 keeps P^T in smem.
  // BIASS (msa_row's batch-shared full bias): the freed 32 KB hold the (key x query) bias tile
  // instead, prefetched with the Q/dO tile (single-buffered) rather than loaded from global
  // memory inside the softmax-backward loop.
  static constexpr bool PTM = CP <= 32;
  static constexpr int NB = (PTM && !BIASS) ? 2 : 1;        // query-tile operand buffers
  static constexpr uint32_t K = 0;                          // [key][d] K-major
  static constexpr uint32_t V = K + BW_BK * CP * 2;         // [key][d] K-major
  static constexpr uint32_t Q = V + BW_BK * CP * 2;         // NB x [query][d] K-major
  static constexpr uint32_t QD_BYTES = BW_BQ * CP * 2;
  static constexpr uint32_t DO = Q + NB * QD_BYTES;         // NB x [query][d] K-major
  static constexpr uint32_t PT = DO + NB * QD_BYTES;        // [key][query] K-major (!PTM)
  static constexpr uint32_t DST = PT + (PTM ? 0 : BW_BK * BW_BQ * 2);  // [key][query] K-major
  static constexpr uint32_t LSE = DST + BW_BK * BW_BQ * 2;  // NB x fp32 [128]
  static constexpr uint32_t DD = LSE + NB * BW_BQ * 4;      // NB x fp32 [128]
  static constexpr uint32_t KB = DD + NB * BW_BQ * 4;       // fp32 [2][128] per-key dbias partials
  static constexpr int BROW = BW_BQ + 8;                    // bias tile row (key): 136 bf16, conflict-free
  static constexpr uint32_t BT = KB + 2 * BW_BK * 4;        // [key][query] bias tile (BIASS)
  static constexpr uint32_t TOTAL = BT + (BIASS ? BW_BK * BROW * 2 : 0);
};

__device__ __forceinline__ void bw_tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
// D (+)= A[tmem] * B[smem]: A operand (M = 128 lanes, 2 bf16 per 32-bit column) in TMEM
__device__ __forceinline__ void bw_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int CP>
__device__ __forceinline__ void bw_load(uint32_t sdst, const bf16* base, int64_t row_stride, int row0, int nvalid,
                                        int c) {
  constexpr int CPR = CP / 8;
  for (int ch = threadIdx.x; ch < 128 * CPR; ch += 256) {
    const int r = ch / CPR, d = (ch % CPR) * 8;
    const bool ok = (r < nvalid) && (d < c);
    const bf16* src = ok ? base + (int64_t)(row0 + r) * row_stride + d : base;
    cp_async16(sdst + kmajor_off(r, d, 128), src, ok);
  }
}

// <= 128 registers, 256 TMEM columns, ~98 KB smem -> 2 CTAs (16 warps) per SM.
// A batch-shared bias (msa_row: dbias stride 0 over b) is handled by writing the
// scaled dS (bf16) per batch and reducing over batches in attn_dbias_reduce
// (deterministic, no atomics).
// MODE: 0 = no bias (msa_col), 1 = per-key bias (pair_row / pair_col), 2 = full bias shared
// over the batch with dS stored for the batch reduction (msa_row), 3 = generic full bias
// (fp32 atomics).  Specialised so the per-element loop carries no dead predicated paths.
template <int CP, int MODE>
__global__ void __launch_bounds__(256, 2) attn_bwd_kernel(AttnBwdParams P, int nkt, int dq_partial,
                                                          const __grid_constant__ BwdMaps maps, int tmaq) {
  pdl_wait();
  constexpr bool BIASS = MODE == 2 && CP <= 32;
  using SM = BwdSmem<CP, BIASS>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar1, bar2, bar3, tbar[2], bbar;
  __shared__ uint32_t tmem_sh;
  const uint32_t sb = smem_u32(smem);
  constexpr bool PTM = SM::PTM;
  constexpr bool DB = SM::NB == 2;  // double-buffered query-tile operands
  float* s_kb = reinterpret_cast<float*>(smem + SM::KB);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wq = warp & 3, wg = warp >> 2;
  const AttnParams& F = P.f;
  const int L = F.L, c = F.c, H = F.H;
  const int64_t Btot = P.B;
  const int kr = wq * 32 + lane;  // key row of this thread (TMEM lane)
  constexpr bool per_key_bias = MODE == 1;
  const bool db_per_key = MODE == 1 && P.dbias != nullptr;
  constexpr bool db_store = MODE == 2;  // batch-shared full bias -> dS workspace
  const int nqt = (L + BW_BQ - 1) / BW_BQ;
  // persistent CTAs walk the (batch, head, key tile) units; the first query tile of the next
  // unit (and its K/V) is prefetched under the TMEM drain of the current unit's last tile
  const int64_t units = Btot * H * nkt;

  if (warp == 0) tmem_alloc(&tmem_sh, 256);
  if (threadIdx.x == 0) {
    mbar_init(&bar1, 1);
    mbar_init(&bar2, 1);
    mbar_init(&tbar[0], 1);
    mbar_init(&tbar[1], 1);
    mbar_init(&bbar, 1);
    mbar_init(&bar3, 1);
    fence_mbar_init();
  }
  __syncthreads();  // the TMA path issues into tbar right below
  uint32_t t_par = 0;  // TMA path: completion parity of tbar[0] / tbar[1] in bits 0 / 1 (uniform over threads)
  uint32_t b_par = 0;  // TMA path, BIASS: completion parity of bbar (the bias tile's own barrier)
  // BIASS + TMA: the (key x query) bias tile has its own barrier and is issued as soon as the
  // previous tile's softmax-backward phase has read it (under that tile's dV/dK/dQ MMAs and TMEM
  // drain), not with the Q/dO tile after the MMAs: a phase trace showed the loop top waiting
  // 1-5.6 us per tile on it (profiles/r02_attn_bwd_msa_row_trace_before.txt)
  auto issue_bias = [&](int h, int k0, int q0) {
    mbar_expect_tx(&bbar, (uint32_t)(BW_BK * SM::BROW * 2));
    tma_ld3(sb + SM::BT, reinterpret_cast<uint64_t>(&maps.bt), q0, k0, h, smem_u32(&bbar));
  };
  const int64_t HC = (int64_t)H * c;
  // every per-tile operand is a cp.async copy (dO, D and lse*log2e come from the prep kernel)
  const bool vec_stats = (L & 3) == 0;
  auto issue_loads = [&](int64_t b, int h, int k0, int qt, bool with_kv, int buf) {
    const int q0 = qt * BW_BQ;
    const int64_t st0 = (b * H + h) * (int64_t)L + q0;
    const uint32_t lse_b = SM::LSE + buf * BW_BQ * 4, dd_b = SM::DD + buf * BW_BQ * 4;
    if (tmaq) {
      // one thread: K/V (first tile of a unit), Q, dO by tensor maps (64-byte swizzle), lse / D rows
      // by bulk copies; all of it completes on tbar[buf] (no per-thread cp.async address streams)
      if (threadIdx.x == 0) {
        const uint32_t tile = 128 * 32 * 2, vec = BW_BQ * 4;
        const int nq = L - q0 < BW_BQ ? L - q0 : BW_BQ;
        mbar_expect_tx(&tbar[buf], (with_kv ? 4 : 2) * tile + 2 * (uint32_t)nq * 4);
        const uint32_t br = smem_u32(&tbar[buf]);
        if (with_kv) {
          tma_ld4(sb + SM::K, reinterpret_cast<uint64_t>(&maps.k), 0, h, k0, (int)b, br);
          tma_ld4(sb + SM::V, reinterpret_cast<uint64_t>(&maps.v), 0, h, k0, (int)b, br);
        }
        tma_ld4(sb + SM::Q + buf * SM::QD_BYTES, reinterpret_cast<uint64_t>(&maps.q), 0, h, q0, (int)b, br);
        tma_ld4(sb + SM::DO + buf * SM::QD_BYTES, reinterpret_cast<uint64_t>(&maps.dO), 0, h, q0, (int)b, br);
        bulk_ld(sb + lse_b, P.lse2 + st0, (uint32_t)nq * 4, &tbar[buf]);
        bulk_ld(sb + dd_b, P.Dsum + st0, (uint32_t)nq * 4, &tbar[buf]);
        (void)vec;
      }
    } else {
      if (with_kv) {
        bw_load<CP>(sb + SM::K, F.k + b * F.k_sb + (int64_t)h * c, F.k_sl, k0, L - k0, c);
        bw_load<CP>(sb + SM::V, F.v + b * F.v_sb + (int64_t)h * c, F.v_sl, k0, L - k0, c);
      }
      bw_load<CP>(sb + SM::Q + buf * SM::QD_BYTES, F.q + b * F.q_sb + (int64_t)h * c, F.q_sl, q0, L - q0, c);
      bw_load<CP>(sb + SM::DO + buf * SM::QD_BYTES, P.dO + b * L * HC + (int64_t)h * c, HC, q0, L - q0, c);
    }
    if constexpr (BIASS) if (!tmaq) {  // transposed bias [h][key][query] (query-contiguous, L % 8 == 0)
      const bf16* bt = F.bias + (int64_t)h * F.bs1;
#pragma unroll
      for (int i = 0; i < BW_BK * (BW_BQ / 8) / 256; ++i) {
        const int ch = threadIdx.x + i * 256;
        const int r = ch >> 4, cq = (ch & 15) * 8;
        const bool ok = (k0 + r < L) && (q0 + cq < L);
        cp_async16(sb + SM::BT + r * (SM::BROW * 2) + cq * 2, ok ? bt + (int64_t)(k0 + r) * F.bs3 + q0 + cq : bt, ok);
      }
    }
    if (tmaq) {
      // lse / D were bulk-copied above
    } else if (vec_stats) {
      if (threadIdx.x < 2 * BW_BQ / 4) {
        const int t = threadIdx.x & (BW_BQ / 4 - 1);
        const bool ok = q0 + 4 * t < L;
        const float* src = threadIdx.x < BW_BQ / 4 ? P.lse2 : P.Dsum;
        cp_async16(sb + (threadIdx.x < BW_BQ / 4 ? lse_b : dd_b) + 16 * t, ok ? src + st0 + 4 * t : src, ok);
      }
    } else if (threadIdx.x < BW_BQ) {
      const bool ok = q0 + (int)threadIdx.x < L;
      reinterpret_cast<float*>(smem + lse_b)[threadIdx.x] = ok ? P.lse2[st0 + threadIdx.x] : 0.f;
      reinterpret_cast<float*>(smem + dd_b)[threadIdx.x] = ok ? P.Dsum[st0 + threadIdx.x] : 0.f;
    }
    cp_async_commit();
  };
  auto decode = [&](int64_t u, int64_t& b, int& h, int& kt) {
    kt = (int)(u % nkt);
    const int64_t t = u / nkt;
    h = (int)(t % H);
    b = t / H;
  };
  {
    int64_t b0;
    int h0, kt0;
    decode(blockIdx.x, b0, h0, kt0);
    if ((int64_t)blockIdx.x < units) {
      issue_loads(b0, h0, kt0 * BW_BK, 0, true, 0);
      if constexpr (BIASS) if (tmaq && threadIdx.x == 0) issue_bias(h0, kt0 * BW_BK, 0);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;
  const uint32_t t_lane = tmem + ((uint32_t)(wq * 32) << 16);
  // S^T [0,128) (PTM: P^T packed bf16 over it at wg*64 + part*8), dP^T [128,256); the
  // dV/dK/dQ products go where no operand of their own MMAs lives
  // PTM: dS^T packed bf16 over the dP^T columns already read (128 + wg*64 + part*8) is the A
  // operand of the dK MMA (TS: 32 KB less shared-memory operand traffic per tile); the dV / dK / dQ
  // products go to the columns neither packed operand occupies
  constexpr uint32_t T_S = 0, T_DP = 128;
  constexpr uint32_t T_DV = PTM ? 32 : 0, T_DK = PTM ? 96 : T_DV + CP, T_DQ = PTM ? 160 : T_DV + 2 * CP;

  constexpr uint32_t ID_SS = make_idesc_bf16(128, 128, 0, 0);  // S^T = K Q^T, dP^T = V dO^T
  constexpr uint32_t ID_KV = make_idesc_bf16(128, CP, 0, 1);   // dV = P^T dO, dK = dS^T Q  (B: MN-major view)
  constexpr uint32_t ID_Q = make_idesc_bf16(128, CP, 1, 1);    // dQ = dS K  (A and B: MN-major views)
  constexpr uint32_t LBO_ROWS = (128 / 8) * 128;               // 2048: next 8-k group of a 128-row K-major tile

#if EVO_EXP == 4 || EVO_EXP == 5
  if (blockIdx.x & 1) {  // experiment: offset the two co-resident CTAs by part of an iteration
    const long long t0 = clock64();
    while (clock64() - t0 < (EVO_EXP == 4 ? 1500 : 3000)) {
    }
  }
#endif
  int it = 0;
  uint32_t n_early = 0;  // bar3 phases (one per early_next tile; uniform over threads)
  bf16 kb_next = f2bf(0.f);  // per-key bias of the next unit (MODE 1)
  bool first_unit = true;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    int64_t b;
    int h, kt;
    decode(u, b, h, kt);
    const int k0 = kt * BW_BK;
    const int kj = k0 + kr;
    const bool kvalid = kj < L;
    float acc[CP];  // dV (warpgroup 0) or dK (warpgroup 1) of this key row, summed over query tiles
#pragma unroll
    for (int d = 0; d < CP; ++d) acc[d] = 0.f;
    float kbias = 0.f;
    if constexpr (per_key_bias) {
      if (first_unit) kb_next = kvalid ? F.bias[b * F.bs0 + (int64_t)h * F.bs1 + (int64_t)kj * F.bs3] : f2bf(0.f);
      kbias = bf2f(kb_next);  // loaded with this unit's prefetch, under the previous unit's drain
      first_unit = false;
    }
    const bf16* bias_col = nullptr;  // full bias: element (q, kj) at bias_col[q * bs2]
    if ((MODE == 2 || MODE == 3) && kvalid) bias_col = F.bias + b * F.bs0 + (int64_t)h * F.bs1 + (int64_t)kj * F.bs3;
    float* dbias_col = nullptr;
    if (P.dbias && kvalid) dbias_col = P.dbias + b * P.db0 + (int64_t)h * P.db1 + (int64_t)kj * P.db3;
    const int bs2 = (int)F.bs2;  // full-bias query stride (< 2^31)
    for (int qt = 0; qt < nqt; ++qt, ++it) {
      const int q0 = qt * BW_BQ;
      const int buf = DB ? (it & 1) : 0;
      // single-buffered tiles (msa_row's bias tile takes the second buffer's room): the next query
      // tile of the unit is loaded as soon as the dV / dK MMAs (its last readers) are done, under the
      // dQ MMAs, instead of after all of them
      const bool early_next = !DB && tmaq && qt + 1 < nqt;
      const uint32_t sQ = sb + SM::Q + buf * SM::QD_BYTES, sDO = sb + SM::DO + buf * SM::QD_BYTES;
      const float* s_lse = reinterpret_cast<const float*>(smem + SM::LSE + buf * BW_BQ * 4);
      const float* s_D = reinterpret_cast<const float*>(smem + SM::DD + buf * BW_BQ * 4);
      BTRACE(it * 8 + 0);
      cp_async_wait<0>();
      if (tmaq) {
        mbar_wait(&tbar[buf], (t_par >> buf) & 1u);
        t_par ^= 1u << buf;
        if constexpr (BIASS) {
          mbar_wait(&bbar, b_par);
          b_par ^= 1u;
        }
      }
      fence_async_smem();
      __syncthreads();
      BTRACE(it * 8 + 1);
      // double-buffered: the next query tile of this unit loads while this one computes (the
      // other buffer's last reader, the previous tile's MMAs, completed before this barrier)
      if (DB && qt + 1 < nqt) issue_loads(b, h, k0, qt + 1, false, buf ^ 1);
      if (threadIdx.x == 0) {
        tc_fence_after();
        // the previous tile's dS^T store must have read DST before this tile's softmax-backward
        // phase rewrites it; every thread passes bar1 (committed below) before writing DST
        if (db_store && tmaq) bulk_wait_read<0>();
#pragma unroll
        for (int kk = 0; kk < CP / 16; ++kk) {
          const uint32_t koff = kk * 2 * LBO_ROWS;
          if (tmaq) {
            mma_bf16(tmem + T_S, bw_sw64_k(sb + SM::K + kk * 32), bw_sw64_k(sQ + kk * 32), ID_SS, kk != 0);
            mma_bf16(tmem + T_DP, bw_sw64_k(sb + SM::V + kk * 32), bw_sw64_k(sDO + kk * 32), ID_SS, kk != 0);
          } else {
            mma_bf16(tmem + T_S, make_sdesc(sb + SM::K + koff, LBO_ROWS, 128), make_sdesc(sQ + koff, LBO_ROWS, 128),
                     ID_SS, kk != 0);
            mma_bf16(tmem + T_DP, make_sdesc(sb + SM::V + koff, LBO_ROWS, 128), make_sdesc(sDO + koff, LBO_ROWS, 128),
                     ID_SS, kk != 0);
          }
        }
        mma_commit(&bar1);
      }
      mbar_wait(&bar1, it & 1);
      tc_fence_after();
      BTRACE(it * 8 + 2);

      float kb_acc = 0.f;
#pragma unroll 1
      for (int part = 0; part < 4; ++part) {
        const int qc = wg * 64 + part * 16;  // query column offset inside the tile
        float s[16], dp[16];
        tmem_ld16(t_lane + T_S + qc, s);
        tmem_ld16(t_lane + T_DP + qc, dp);
        tmem_ld_wait();
        float pv[16], dsv[16];
        const bool all_valid = kvalid && q0 + qc + 16 <= L;
        float bv[16];
        if constexpr (BIASS) {  // this key row's 16 queries from the prefetched smem tile
#pragma unroll
          for (int e = 0; e < 16; e += 8) {
            uint32_t u0, u1, u2, u3;
            asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];\n" : "=r"(u0), "=r"(u1), "=r"(u2), "=r"(u3)
                         : "r"(sb + SM::BT + kr * (SM::BROW * 2) + (qc + e) * 2));
            unpack_bf16x2(u0, bv[e], bv[e + 1]); unpack_bf16x2(u1, bv[e + 2], bv[e + 3]);
            unpack_bf16x2(u2, bv[e + 4], bv[e + 5]); unpack_bf16x2(u3, bv[e + 6], bv[e + 7]);
          }
        } else if constexpr (MODE == 2) {  // transposed batch-shared bias: 16 consecutive queries per key
          if (bias_col) {
            const bf16* bp = bias_col + (q0 + qc);
#pragma unroll
            for (int e = 0; e < 16; e += 8) {
              if (q0 + qc + e < L) {
                const uint4 u = *reinterpret_cast<const uint4*>(bp + e);
                unpack_bf16x2(u.x, bv[e], bv[e + 1]); unpack_bf16x2(u.y, bv[e + 2], bv[e + 3]);
                unpack_bf16x2(u.z, bv[e + 4], bv[e + 5]); unpack_bf16x2(u.w, bv[e + 6], bv[e + 7]);
              } else {
#pragma unroll
                for (int t = 0; t < 8; ++t) bv[e + t] = 0.f;
              }
            }
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) bv[e] = 0.f;
          }
        } else if constexpr (MODE == 3) {
          if (bias_col) {
            const bf16* bp = bias_col + (q0 + qc) * bs2;
#pragma unroll
            for (int e = 0; e < 16; ++e) bv[e] = (q0 + qc + e < L) ? bf2f(bp[e * bs2]) : 0.f;
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) bv[e] = 0.f;
          }
        }
        float lse16[16], D16[16];
#pragma unroll
        for (int e = 0; e < 16; e += 4) {
          *reinterpret_cast<float4*>(lse16 + e) = *reinterpret_cast<const float4*>(s_lse + qc + e);
          *reinterpret_cast<float4*>(D16 + e) = *reinterpret_cast<const float4*>(s_D + qc + e);
        }
        // packed fp32x2 math (FFMA2 / FADD2 / FMUL2): half the issue slots of the scalar form
        const float2 sl2 = make_float2(F.scale_log2, F.scale_log2);
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          float2 x = make_float2(s[e], s[e + 1]);
          if constexpr (MODE == 1) x = __fadd2_rn(x, make_float2(kbias, kbias));
          if constexpr (MODE == 2 || MODE == 3) x = __fadd2_rn(x, make_float2(bv[e], bv[e + 1]));
          const float2 y = __ffma2_rn(x, sl2, make_float2(-lse16[e], -lse16[e + 1]));
          pv[e] = ex2f(y.x);
          pv[e + 1] = ex2f(y.y);
        }
        if (!all_valid) {
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (!(kvalid && q0 + qc + e < L)) pv[e] = 0.f;
        }
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          const float2 d = __fmul2_rn(make_float2(pv[e], pv[e + 1]),
                                      f2sub(make_float2(dp[e], dp[e + 1]), make_float2(D16[e], D16[e + 1])));
          dsv[e] = d.x;
          dsv[e + 1] = d.y;
        }
#if EVO_EXP == 1
#pragma unroll
        for (int e = 0; e < 16; ++e) { pv[e] = s[e]; dsv[e] = dp[e]; }
#endif
        if constexpr (MODE == 1) {
          float2 k2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int e = 0; e < 16; e += 2) k2 = __fadd2_rn(k2, make_float2(dsv[e], dsv[e + 1]));
          kb_acc += k2.x + k2.y;
        } else if constexpr (MODE == 3) {
          if (dbias_col) {
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (q0 + qc + e < L) atomicAdd(dbias_col + (int64_t)(q0 + qc + e) * P.db2, P.scale * dsv[e]);
          }
        }
        uint32_t dk[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) dk[e] = pack_bf16x2(dsv[2 * e], dsv[2 * e + 1]);
        if constexpr (PTM) {  // P^T over the S^T columns, dS^T over the dP^T columns this warp has read
          uint32_t pk[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) pk[e] = pack_bf16x2(pv[2 * e], pv[2 * e + 1]);
          bw_tmem_st8(t_lane + T_S + wg * 64 + part * 8, pk);
          bw_tmem_st8(t_lane + T_DP + wg * 64 + part * 8, dk);
        }
#pragma unroll
        for (int e = 0; e < 16; e += 8) {
          if constexpr (!PTM)
            st_shared_v4(sb + SM::PT + kmajor_off(kr, qc + e, 128), pack_bf16x2(pv[e], pv[e + 1]),
                         pack_bf16x2(pv[e + 2], pv[e + 3]), pack_bf16x2(pv[e + 4], pv[e + 5]),
                         pack_bf16x2(pv[e + 6], pv[e + 7]));
          st_shared_v4(sb + SM::DST + kmajor_off(kr, qc + e, 128), dk[e / 2], dk[e / 2 + 1], dk[e / 2 + 2],
                       dk[e / 2 + 3]);
        }
      }
      if (db_per_key) s_kb[wg * BW_BK + kr] = kb_acc;
      BTRACE(it * 8 + 3);

      if (PTM) tmem_st_wait();
      fence_async_smem();
      tc_fence_before();
      __syncthreads();
      if (db_per_key && wg == 0 && dbias_col) atomicAdd(dbias_col, P.scale * (s_kb[kr] + s_kb[BW_BK + kr]));
      if constexpr (BIASS) if (tmaq && threadIdx.x == 0) {  // every thread has read the bias tile
        if (qt + 1 < nqt) {
          issue_bias(h, k0, q0 + BW_BQ);
        } else if (u + gridDim.x < units) {
          int64_t nb;
          int nh, nkt_;
          decode(u + gridDim.x, nb, nh, nkt_);
          issue_bias(nh, nkt_ * BW_BK, 0);
        }
      }
      if (threadIdx.x == 0) {
        tc_fence_after();
#if EVO_EXP != 2
#pragma unroll
        for (int kk = 0; kk < BW_BQ / 16; ++kk) {
          const uint32_t aoff = kk * 2 * LBO_ROWS;
          const uint32_t boff = kk * 2 * 128;
          const uint64_t d_do = tmaq ? bw_sw64_mn(sDO + kk * 1024) : make_sdesc(sDO + boff, 128, LBO_ROWS);
          const uint64_t d_q = tmaq ? bw_sw64_mn(sQ + kk * 1024) : make_sdesc(sQ + boff, 128, LBO_ROWS);
          if constexpr (PTM) {  // queries [0,64) at columns [0,32), [64,128) at [64,96) of each operand
            const uint32_t ac = kk < 4 ? kk * 8 : 64 + (kk - 4) * 8;
            bw_mma_ts(tmem + T_DV, tmem + T_S + ac, d_do, ID_KV, kk != 0);
            bw_mma_ts(tmem + T_DK, tmem + T_DP + ac, d_q, ID_KV, kk != 0);
          } else {
            mma_bf16(tmem + T_DV, make_sdesc(sb + SM::PT + aoff, LBO_ROWS, 128), d_do, ID_KV, kk != 0);
            mma_bf16(tmem + T_DK, make_sdesc(sb + SM::DST + aoff, LBO_ROWS, 128), d_q, ID_KV, kk != 0);
          }
        }
        if (early_next) mma_commit(&bar3);  // dV / dK done: Q and dO are free
#pragma unroll
        for (int kk = 0; kk < BW_BK / 16; ++kk) {
          const uint32_t off = kk * 2 * 128;
          const uint64_t d_k = tmaq ? bw_sw64_mn(sb + SM::K + kk * 1024) : make_sdesc(sb + SM::K + off, 128, LBO_ROWS);
          mma_bf16(tmem + T_DQ, make_sdesc(sb + SM::DST + off, 128, LBO_ROWS), d_k, ID_Q, kk != 0);
        }
#endif
        mma_commit(&bar2);
        if (early_next) {  // the next query tile's Q / dO / lse / D load under the dQ MMAs
          mbar_wait(&bar3, n_early & 1);
          issue_loads(b, h, k0, qt + 1, false, 0);
        }
      }
      if (early_next) ++n_early;
      if (db_store && tmaq) {
        // (TMA store of the dS^T tile: issued after the next tile's loads, below)
      } else if constexpr (db_store) {
        // dS^T tile (unscaled bf16, canonical K-major [key][query]) -> workspace [b][h][key][query],
        // under the dV/dK/dQ MMAs (which only read the tile): all 8 smem reads of a thread first,
        // then its 8 16-byte stores (no register-reuse serialisation between load and store).
        // lane = (query group % 4, key % 8): each smem phase reads 128 contiguous bytes and each key
        // row gets 64 contiguous bytes per store (requires L % 8 == 0)
        bf16* wsb = P.dS + ((b * H + h) * (int64_t)L + k0) * L + q0;
        constexpr int NCP = (BW_BK * BW_BQ / 8) / 256;
        uint4 cv[NCP];
#pragma unroll
        for (int i = 0; i < NCP; ++i) {
          const int ch = threadIdx.x + i * 256;
          const int r = ((ch >> 5) & 15) * 8 + (ch & 7);
          const int g = (ch >> 9) * 4 + ((ch >> 3) & 3);
          cv[i] = *reinterpret_cast<const uint4*>(smem + SM::DST + (g * (BW_BK / 8) + (r >> 3)) * 128 + (r & 7) * 16);
        }
#pragma unroll
        for (int i = 0; i < NCP; ++i) {
          const int ch = threadIdx.x + i * 256;
          const int r = ((ch >> 5) & 15) * 8 + (ch & 7);
          const int g = (ch >> 9) * 4 + ((ch >> 3) & 3);
          if (k0 + r < L && q0 + g * 8 < L) *reinterpret_cast<uint4*>(wsb + (int64_t)r * L + g * 8) = cv[i];
        }
      }
      BTRACE(it * 8 + 4);
      mbar_wait(&bar2, it & 1);
      tc_fence_after();
      BTRACE(it * 8 + 5);
      // the tiles are free: prefetch the next (batch, query tile) while draining TMEM
      const bool last_q = qt + 1 == nqt;
      if (!last_q) {
        if (!DB && !early_next) issue_loads(b, h, k0, qt + 1, false, 0);
      } else if (u + gridDim.x < units) {
        int64_t nb;
        int nh, nkt_;
        decode(u + gridDim.x, nb, nh, nkt_);
#if EVO_EXP != 11
        issue_loads(nb, nh, nkt_ * BW_BK, 0, true, DB ? (buf ^ 1) : 0);
#endif
        if constexpr (per_key_bias) {
          const int nkj = nkt_ * BW_BK + kr;
          kb_next = nkj < L ? F.bias[nb * F.bs0 + (int64_t)nh * F.bs1 + (int64_t)nkj * F.bs3] : f2bf(0.f);
        }
      }
      if (db_store && tmaq && threadIdx.x == 0) {
        // dS^T tile -> workspace by one TMA tensor store (the map walks the canonical tile order),
        // issued AFTER the next tile's loads: a store queued ahead of them held them back by 1-3 us
        // per tile (phase trace); the tile is rewritten only after bulk_wait_read before the next
        // S/dP MMAs
        tma_st5(reinterpret_cast<uint64_t>(&maps.ws), sb + SM::DST, 0, 0, k0 / 8, q0 / 8, (int)(b * H + h));
        bulk_commit();
      }
      BTRACE(it * 8 + 7);
#if EVO_EXP != 3
      {
#pragma unroll
        for (int cc = 0; cc < CP; cc += 16) {
          float v[16];
          tmem_ld16(t_lane + (wg == 0 ? T_DV : T_DK) + cc, v);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 16; ++e) acc[cc + e] += v[e];
        }
        float w[CP / 2];
        if constexpr (CP == 16) tmem_ld8(t_lane + T_DQ + wg * 8, w);
        else if constexpr (CP == 32) tmem_ld16(t_lane + T_DQ + wg * 16, w);
        else tmem_ld32(t_lane + T_DQ + wg * 32, w);
        tmem_ld_wait();
        const int qq = q0 + kr;  // dQ: TMEM lane = query row
        if (qq < L) {
          if (dq_partial == 2) {  // one key tile: dQ is final, written as bf16 (no finish pass)
            bf16* dst = P.dq + b * P.dq_sb + (int64_t)qq * P.dq_sl + (int64_t)h * c + wg * (CP / 2);
            if (wg * (CP / 2) + CP / 2 <= c && (CP / 2) % 8 == 0) {
#pragma unroll
              for (int e = 0; e < CP / 2; e += 8) {
                uint4 u;
                u.x = pack_bf16x2(P.scale * w[e], P.scale * w[e + 1]);
                u.y = pack_bf16x2(P.scale * w[e + 2], P.scale * w[e + 3]);
                u.z = pack_bf16x2(P.scale * w[e + 4], P.scale * w[e + 5]);
                u.w = pack_bf16x2(P.scale * w[e + 6], P.scale * w[e + 7]);
                *reinterpret_cast<uint4*>(dst + e) = u;
              }
            } else {
#pragma unroll
              for (int e = 0; e < CP / 2; ++e)
                if (wg * (CP / 2) + e < c) dst[e] = f2bf(P.scale * w[e]);
            }
          } else if (dq_partial) {  // per-key-tile bf16 partial, summed in fp32 by the finish pass
            bf16* dst = reinterpret_cast<bf16*>(P.dQacc) + (((int64_t)kt * Btot + b) * L + qq) * HC + (int64_t)h * c +
                        wg * (CP / 2);
            if (wg * (CP / 2) + CP / 2 <= c && (CP / 2) % 8 == 0) {
#pragma unroll
              for (int e = 0; e < CP / 2; e += 8) {
                uint4 u;
                u.x = pack_bf16x2(P.scale * w[e], P.scale * w[e + 1]);
                u.y = pack_bf16x2(P.scale * w[e + 2], P.scale * w[e + 3]);
                u.z = pack_bf16x2(P.scale * w[e + 4], P.scale * w[e + 5]);
                u.w = pack_bf16x2(P.scale * w[e + 6], P.scale * w[e + 7]);
                *reinterpret_cast<uint4*>(dst + e) = u;
              }
            } else {
#pragma unroll
              for (int e = 0; e < CP / 2; ++e)
                if (wg * (CP / 2) + e < c) dst[e] = f2bf(P.scale * w[e]);
            }
          } else {
            float* dst = P.dQacc + (b * L + qq) * HC + (int64_t)h * c + wg * (CP / 2);
#pragma unroll
            for (int e = 0; e < CP / 2; ++e)
              if (wg * (CP / 2) + e < c) atomicAdd(dst + e, P.scale * w[e]);
          }
        }
      }
#endif
      BTRACE(it * 8 + 6);
      tc_fence_before();
      __syncthreads();
    }
    // dV (warpgroup 0) and dK (warpgroup 1) of batch b
    if (kvalid) {
      const float sc = wg == 0 ? 1.f : P.scale;
      bf16* dst = wg == 0 ? P.dv + b * P.dv_sb + (int64_t)kj * P.dv_sl + (int64_t)h * c
                          : P.dk + b * P.dk_sb + (int64_t)kj * P.dk_sl + (int64_t)h * c;
#pragma unroll
      for (int d = 0; d < CP; d += 8) {
        if (d < c) {
          uint4 wv;
          wv.x = pack_bf16x2(sc * acc[d], sc * acc[d + 1]);
          wv.y = pack_bf16x2(sc * acc[d + 2], sc * acc[d + 3]);
          wv.z = pack_bf16x2(sc * acc[d + 4], sc * acc[d + 5]);
          wv.w = pack_bf16x2(sc * acc[d + 6], sc * acc[d + 7]);
          *reinterpret_cast<uint4*>(dst + d) = wv;
        }
      }
    }
  }
  if (db_store && tmaq && threadIdx.x == 0) bulk_wait<0>();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

// dq = bf16(sum of the NP per-key-tile fp32 partials); all 2*NP loads of a thread in flight
#if EVO_EXP == 10 || EVO_EXP == 11
}  // namespace evo
extern "C" int evo_bwd_trace(void* dst) { return (int)cudaMemcpyFromSymbol(dst, evo::g_bwd_trace, sizeof(evo::g_bwd_trace)); }
namespace evo {
#endif
template <int NP>
__global__ void __launch_bounds__(256) attn_bwd_dq_finish(AttnBwdParams P, int64_t B, int sh_hc, int sh_l) {
  pdl_wait();
  const int L = P.f.L, H = P.f.H, c = P.f.c;
  const int64_t n = B * L * (int64_t)H * c;
  const int64_t n8 = n / 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * 8;
    const uint32_t eu = (uint32_t)e, hc = (uint32_t)(H * c);  // n < 2^31 (host-checked)
    // shifts when H*c and L are powers of two (sh >= 0): the emulated divisions cost more issue
    // slots than the element work
    const uint32_t rowu = sh_hc >= 0 ? eu >> sh_hc : eu / hc;
    const uint32_t bu = sh_l >= 0 ? rowu >> sh_l : rowu / (uint32_t)L;
    const int64_t col = eu - rowu * hc, b = bu, l = rowu - bu * (uint32_t)L;
    float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if constexpr (NP == 0) {  // one fp32 accumulator (atomics, > DQ_MAX_PARTS key tiles)
      const float4 x0 = __ldcs(reinterpret_cast<const float4*>(P.dQacc + e));
      const float4 x1 = __ldcs(reinterpret_cast<const float4*>(P.dQacc + e + 4));
      a[0] = x0.x; a[1] = x0.y; a[2] = x0.z; a[3] = x0.w; a[4] = x1.x; a[5] = x1.y; a[6] = x1.z; a[7] = x1.w;
    }
    const bf16* part = reinterpret_cast<const bf16*>(P.dQacc);
    uint4 raw[NP > 0 ? NP : 1];
#pragma unroll
    for (int p = 0; p < NP; ++p) raw[p] = __ldcs(reinterpret_cast<const uint4*>(part + p * n + e));
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      float v[8];
      unpack_bf16x2(raw[p].x, v[0], v[1]); unpack_bf16x2(raw[p].y, v[2], v[3]);
      unpack_bf16x2(raw[p].z, v[4], v[5]); unpack_bf16x2(raw[p].w, v[6], v[7]);
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] += v[k];
    }
    uint4 w;
    w.x = pack_bf16x2(a[0], a[1]); w.y = pack_bf16x2(a[2], a[3]);
    w.z = pack_bf16x2(a[4], a[5]); w.w = pack_bf16x2(a[6], a[7]);
    *reinterpret_cast<uint4*>(P.dq + b * P.dq_sb + l * P.dq_sl + col) = w;
  }
}

constexpr int DQ_MAX_PARTS = 4;  // <= 4 key tiles (L <= 512): per-tile dQ partials, plain stores

static int64_t ws_layout(int64_t B, int64_t L, int H, int c, int bias_batch_reduced, int64_t* off_dq, int64_t* off_D,
                         int64_t* off_lse2, int64_t* off_dS) {
  const int64_t n = B * L * (int64_t)H * c;
  const int64_t nkt = (L + BW_BK - 1) / BW_BK;
  const int64_t parts = nkt == 1 ? 0 : (nkt <= DQ_MAX_PARTS ? nkt : 1);
  const int64_t stats = ((B * H * L * 4 + 255) / 256) * 256;
  int64_t o1 = ((n * 2 + 255) / 256) * 256;
  // <= DQ_MAX_PARTS key tiles: bf16 partials; more: one fp32 atomic accumulator
  int64_t o2 = o1 + ((parts * n * (nkt <= DQ_MAX_PARTS ? 2 : 4) + 255) / 256) * 256;
  int64_t o3 = o2 + stats;
  int64_t o4 = o3 + stats;
  if (off_dq) *off_dq = o1;
  if (off_D) *off_D = o2;
  if (off_lse2) *off_lse2 = o3;
  if (off_dS) *off_dS = o4;
  // batch-shared bias: dS^T workspace [B][H][L][L] + the transposed bias [H][L][L]
  return o4 + (bias_batch_reduced ? ((B * H * L * L * 2 + 255) / 256) * 256 + ((H * L * L * 2 + 255) / 256) * 256 : 0);
}

int sm_count();

// tensor map of one per-tile operand: element (d, h, l, b) at base + b*sb + l*sl + h*c + d, box [32 d][1][128 l][1]
static bool bw_map(CUtensorMap* m, const void* base, int c, int H, int64_t L, int64_t B, int64_t sl, int64_t sb) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc || ((uintptr_t)base & 15) || (sl * 2) % 16 || (sb * 2) % 16 || sl <= 0 || sb <= 0) return false;
  cuuint64_t d[4] = {(cuuint64_t)c, (cuuint64_t)H, (cuuint64_t)L, (cuuint64_t)B};
  cuuint64_t s[3] = {(cuuint64_t)c * 2, (cuuint64_t)sl * 2, (cuuint64_t)sb * 2};
  cuuint32_t bx[4] = {32, 1, 128, 1}, es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), d, s, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// msa_row: the transposed bias [H][L][L] (box [136 q][128 keys], the padded smem rows) and the dS^T
// workspace [B*H][L][L] as 5-D (q % 8, key % 8, key / 8, q / 8, b*H + h) = the canonical tile order
static bool bw_bias_maps(BwdMaps* m, const void* bias_t, const void* ds, int H, int64_t L, int64_t B) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc || !bias_t || !ds || L % 8 || ((uintptr_t)bias_t & 15) || ((uintptr_t)ds & 15)) return false;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  {
    cuuint64_t d[3] = {(cuuint64_t)L, (cuuint64_t)L, (cuuint64_t)H};
    cuuint64_t s[2] = {(cuuint64_t)L * 2, (cuuint64_t)L * L * 2};
    cuuint32_t bx[3] = {136, 128, 1};
    if (enc(&m->bt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(bias_t), d, s, bx, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  cuuint64_t d[5] = {8, 8, (cuuint64_t)(L / 8), (cuuint64_t)(L / 8), (cuuint64_t)(B * H)};
  cuuint64_t s[4] = {(cuuint64_t)L * 2, (cuuint64_t)L * 16, 16, (cuuint64_t)L * L * 2};
  cuuint32_t bx[5] = {8, 8, 16, 16, 1};
  return enc(&m->ws, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(ds), d, s, bx, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int CP, int MODE>
static int launch_bwd_m(AttnBwdParams& p, int64_t B, int dq_partial, cudaStream_t st) {
  using SM = BwdSmem<CP, MODE == 2 && CP <= 32>;
  BwdMaps maps;
  memset(&maps, 0, sizeof(maps));
  static const bool tma_off = [] { const char* e = getenv("EVO_ATTN_BWD_NO_TMA"); return e && e[0] == '1'; }();
  const AttnParams& f = p.f;
  const int64_t HC = (int64_t)f.H * f.c;
  // TMA path: head dim exactly 32 (the 64-byte rows of the swizzled tiles) and 16-byte lse / D rows
  const int tmaq = !tma_off && CP == 32 && f.c == 32 && f.L % 4 == 0 &&
                   bw_map(&maps.q, f.q, f.c, f.H, f.L, B, f.q_sl, f.q_sb) &&
                   bw_map(&maps.k, f.k, f.c, f.H, f.L, B, f.k_sl, f.k_sb) &&
                   bw_map(&maps.v, f.v, f.c, f.H, f.L, B, f.v_sl, f.v_sb) &&
                   bw_map(&maps.dO, p.dO, f.c, f.H, f.L, B, HC, f.L * HC) &&
                   (MODE != 2 || bw_bias_maps(&maps, f.bias, p.dS, f.H, f.L, B));
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_kernel<CP, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SM::TOTAL);
    if (e != cudaSuccess) return cuda_status(e, "attn bwd attr");
    attr = true;
  }
  const int64_t nkt = (p.f.L + BW_BK - 1) / BW_BK;
  const int64_t units = B * p.f.H * nkt;
  // persistent: 2 CTAs per SM, units handed out round-robin
  const int64_t slots = (int64_t)sm_count() * 2;
  dim3 grid((unsigned)(units < slots ? units : slots));
  ::evo::pdl_launch(attn_bwd_kernel<CP, MODE>, grid, 256, SM::TOTAL, st, p, (int)nkt, dq_partial, maps, tmaq);
  EVO_LAUNCH_CHECK("attention bwd main");
  return EVO_OK;
}

template <int CP>
static int launch_bwd(AttnBwdParams& p, int64_t B, int dq_partial, cudaStream_t st) {
  if (!p.f.bias) return launch_bwd_m<CP, 0>(p, B, dq_partial, st);
  if (p.f.bs2 == 0) return launch_bwd_m<CP, 1>(p, B, dq_partial, st);
  if (p.dS) return launch_bwd_m<CP, 2>(p, B, dq_partial, st);
  return launch_bwd_m<CP, 3>(p, B, dq_partial, st);
}

}  // namespace evo

using namespace evo;

extern "C" int64_t evo_gated_attention_bwd_workspace(int64_t B, int64_t L, int H, int c, int bias_batch_reduced) {
  return ws_layout(B, L, H, c, bias_batch_reduced && L % 8 == 0, nullptr, nullptr, nullptr, nullptr);
}

extern "C" int evo_gated_attention_bwd(const EvoAttnBwdDesc* d, void* stream) {
  EVO_CHECK_ARG(d, EVO_ERR_ARG, "attention bwd: null descriptor");
  AttnBwdParams p;
  int rc = attn_params_from_desc(&d->f, p.f);
  if (rc) return rc;
  EVO_CHECK_ARG(d->f.o_raw && d->f.lse && d->dout && d->dq && d->dk && d->dv && d->dg && d->workspace, EVO_ERR_ARG,
                "attention bwd: null pointer (o_raw, lse, dout, dq, dk, dv, dg, workspace are required)");
  const int64_t B = d->f.B, L = d->f.L;
  const int H = d->f.H, c = d->f.c;
  EVO_CHECK_ARG((c & (c - 1)) == 0, EVO_ERR_SHAPE, "attention bwd: head dim must be 8, 16, 32 or 64 (got %d)", c);
  EVO_CHECK_ARG(B * L * H * c < (1LL << 31) && (int64_t)H * L * L < (1LL << 31), EVO_ERR_SHAPE,
                "attention bwd: B*L*H*c and H*L*L must be < 2^31 (32-bit index math)");
  int64_t off_dq, off_D, off_lse2, off_dS;
  // batch-shared full bias (msa_row): dS^T tiles to a workspace, reduced over the batch after
  // (16-byte tile copies need L % 8 == 0; otherwise the generic atomic path)
  const int batch_reduced = d->dbias && d->f.bias && d->dbias_s[0] == 0 && d->dbias_s[2] != 0 && L % 8 == 0;
  const int64_t need = ws_layout(B, L, H, c, batch_reduced, &off_dq, &off_D, &off_lse2, &off_dS);
  EVO_CHECK_ARG(d->workspace_bytes >= need, EVO_ERR_ARG, "attention bwd: workspace %lld < %lld bytes",
                (long long)d->workspace_bytes, (long long)need);
  const int64_t strides[] = {d->do_sb, d->do_sl, d->dq_sb, d->dq_sl, d->dk_sb, d->dk_sl, d->dv_sb, d->dv_sl,
                             d->dg_sb, d->dg_sl};
  for (int64_t s : strides) EVO_CHECK_ARG(s % 8 == 0, EVO_ERR_ALIGN, "attention bwd: strides must be multiples of 8");
  p.dout = (const bf16*)d->dout;
  p.do_sb = d->do_sb; p.do_sl = d->do_sl;
  p.dq = (bf16*)d->dq; p.dk = (bf16*)d->dk; p.dv = (bf16*)d->dv; p.dg = (bf16*)d->dg;
  p.dq_sb = d->dq_sb; p.dq_sl = d->dq_sl; p.dk_sb = d->dk_sb; p.dk_sl = d->dk_sl;
  p.dv_sb = d->dv_sb; p.dv_sl = d->dv_sl; p.dg_sb = d->dg_sb; p.dg_sl = d->dg_sl;
  p.dbias = d->dbias;
  p.db0 = d->dbias_s[0]; p.db1 = d->dbias_s[1]; p.db2 = d->dbias_s[2]; p.db3 = d->dbias_s[3];
  char* ws = (char*)d->workspace;
  p.dO = (bf16*)ws;
  p.dQacc = (float*)(ws + off_dq);
  p.Dsum = (float*)(ws + off_D);
  p.lse2 = (float*)(ws + off_lse2);
  p.dS = batch_reduced ? (bf16*)(ws + off_dS) : nullptr;
  // MODE 2 reads the batch-shared bias transposed ([h][key][query], queries contiguous)
  const bool bias_shared = batch_reduced && d->f.bias_s[0] == 0 && d->f.bias_s[3] == 1 && d->f.bias_s[1] % 8 == 0 &&
                           d->f.bias_s[2] % 8 == 0;
  if (batch_reduced && !bias_shared) p.dS = nullptr;  // generic atomic path (MODE 3)

  p.scale = d->f.scale;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nkt = (L + BW_BK - 1) / BW_BK;
  // 1 key tile: final bf16 dQ from the main kernel; <= 4: per-tile fp32 partials summed by the
  // finish pass; more: fp32 atomics into one accumulator
  const int dq_partial = nkt == 1 ? 2 : (nkt <= DQ_MAX_PARTS ? 1 : 0);
  p.B = B;
  if (!dq_partial) {
    cudaError_t e = cudaMemsetAsync(p.dQacc, 0, (size_t)(B * L * H * c) * 4, st);
    if (e != cudaSuccess) return cuda_status(e, "attention bwd memset");
  }
  {
    const int64_t rows = B * L;
    const int64_t pairs = rows * (H * c / 8), per_cta = 8 * PREP_PASSES * 32;
    const unsigned g = (unsigned)((pairs + per_cta - 1) / per_cta);
    auto lg = [](int64_t v) { int k = 0; while ((int64_t(1) << k) < v) ++k; return k; };
    const PrepIdx ix{(uint32_t)(H * c / 8), (uint32_t)L, (uint32_t)c, lg(H * c / 8), lg(L), lg(c)};
    const bool pow2 = (int64_t(1) << ix.sh_nch) == H * c / 8 && (int64_t(1) << ix.sh_L) == L &&
                      (int64_t(1) << ix.sh_c) == c;
    const bool staged = per_cta % (H * c / 8) == 0;
    if (staged && pow2) ::evo::pdl_launch(attn_bwd_prep<true, true>, g, 256, 0, st, p, B, ix);
    else if (staged) ::evo::pdl_launch(attn_bwd_prep<true, false>, g, 256, 0, st, p, B, ix);
    else if (pow2) ::evo::pdl_launch(attn_bwd_prep<false, true>, g, 256, 0, st, p, B, ix);
    else ::evo::pdl_launch(attn_bwd_prep<false, false>, g, 256, 0, st, p, B, ix);
    EVO_LAUNCH_CHECK("attention bwd prep");
  }
  if (p.dS) {
    bf16* bias_t = (bf16*)(ws + off_dS + ((B * H * L * L * 2 + 255) / 256) * 256);
    dim3 tg((unsigned)((L + 31) / 32), (unsigned)((L + 31) / 32), (unsigned)H);
    ::evo::pdl_launch(attn_bias_transpose, tg, 256, 0, st, p.f.bias, p.f.bs1, p.f.bs2, bias_t, (int)L);
    EVO_LAUNCH_CHECK("attention bwd bias transpose");
    p.f.bias = bias_t;
    p.f.bs0 = 0; p.f.bs1 = L * L; p.f.bs2 = 1; p.f.bs3 = L;
  }
  if (c <= 16) rc = launch_bwd<16>(p, B, dq_partial, st);
  else if (c <= 32) rc = launch_bwd<32>(p, B, dq_partial, st);
  else rc = launch_bwd<64>(p, B, dq_partial, st);
  if (rc) return rc;
  if (p.dS) {
    static const bool r32 = getenv("EVO_DBIAS_REDUCE32") != nullptr;  // A/B switch: the 32-query tiles
    if (L % 64 == 0 && !r32) {  // 128-byte rows: 32.7 -> 26-27.5 us per call at the training shape (ncu)
      const dim3 g2((unsigned)(L / 64), (unsigned)((L + 31) / 32), (unsigned)H);
      ::evo::pdl_launch(attn_dbias_reduce64, g2, 512, 0, st, p.dS, p.dbias, B, H, L, p.db1, p.db2, p.db3, p.scale);
    } else {
      const dim3 g2((unsigned)((L + 31) / 32), (unsigned)((L + 31) / 32), (unsigned)H);
      ::evo::pdl_launch(attn_dbias_reduce, g2, 256, 0, st, p.dS, p.dbias, B, H, L, p.db1, p.db2, p.db3, p.scale);
    }
    EVO_LAUNCH_CHECK("attention bwd dbias reduce");
  }
  if (dq_partial == 2) return EVO_OK;
  int64_t n8 = B * L * H * c / 8;
  int64_t g = (n8 + 255) / 256, cap = (int64_t)sm_count() * 16;
  const unsigned gf = (unsigned)(g < cap ? g : cap);
  auto lg2 = [](int64_t v) { int k = 0; while ((int64_t(1) << k) < v) ++k; return (int64_t(1) << k) == v ? k : -1; };
  const int sh_hc = lg2((int64_t)H * c), sh_l = lg2(L);
  switch (dq_partial ? (int)nkt : 0) {  // 0: fp32 atomic accumulator; 2..4: bf16 per-tile partials
    case 0: ::evo::pdl_launch(attn_bwd_dq_finish<0>, gf, 256, 0, st, p, B, sh_hc, sh_l); break;
    case 2: ::evo::pdl_launch(attn_bwd_dq_finish<2>, gf, 256, 0, st, p, B, sh_hc, sh_l); break;
    case 3: ::evo::pdl_launch(attn_bwd_dq_finish<3>, gf, 256, 0, st, p, B, sh_hc, sh_l); break;
    default: ::evo::pdl_launch(attn_bwd_dq_finish<4>, gf, 256, 0, st, p, B, sh_hc, sh_l); break;
  }
  EVO_LAUNCH_CHECK("attention bwd finish");
  return EVO_OK;
}
