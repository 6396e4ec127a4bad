// Gated multi-head attention with bias on tcgen05 (replaces the per-head loop of
// _attention_core, evoformer.py:173-198, for msa_row / msa_col / pair_row / pair_col).
//
// One CTA (4 warps, 128 threads) owns 128 queries of one (batch, head) and streams
// the keys in tiles of 64 (flash-style online softmax, so N_r = 4096 never
// materialises a logit matrix).  <= 128 registers, 128 TMEM columns and ~34 KB of
// shared memory per CTA -> 4 CTAs (16 warps) per SM hide each other's latency:
//   S   = [Q | 1] [K | b]^T       tcgen05.mma M=128 N=64 -> TMEM cols [0,64) (fp32); a per-key
//                                 bias b (pair_row / pair_col) rides in an extra K group
//   s   = S * scale (+ full bias)  thread r owns query row r (tcgen05.ld 32x32b), running
//   p   = exp2(s - m)              max in registers (no shuffles)
//   P  -> TMEM cols [0,32) as bf16 pairs over S (tcgen05.st) - never touches smem
//   O_t = P [V | 1]                tcgen05.mma with the A operand in TMEM, N = CP + 8 ->
//                                 TMEM cols [64, 64+CP+8): column CP is the row sum of P
//   O  += O_t, l += O_t[CP]        in registers, rescaled by the running-max correction
// Epilogue: o = O / l, out = sigmoid(g) * o (gate on raw x, G2), log-sum-exp saved.
// K/V tiles are double-buffered with cp.async; several CTAs per SM overlap the
// MMA of one CTA with the softmax of another.
#include "attn.cuh"
#include "tma.cuh"
#include <cstdlib>
#include <cstring>


namespace evo {

constexpr int ATT_BQ = 128;
constexpr int ATT_BK = 64;   // keys per tile: S = 64 TMEM columns, P = 16 KB
constexpr float LOG2E = 1.4426950408889634f;


template <int CP>
struct AttnSmem {
  static constexpr int CQ = CP + 16;  // Q / K K-extent: data + [1 | per-key bias] group + zero group
  static constexpr int CV = CP + 8;   // V N-extent: data + [1, 0 x 7] (row sums of P)
  static constexpr uint32_t Q = 0, Q_BYTES = ATT_BQ * CQ * 2;
  static constexpr uint32_t KT = Q + Q_BYTES;                  // 2 stages
  static constexpr uint32_t VT = KT + 2 * ATT_BK * CQ * 2;     // 2 stages
  static constexpr uint32_t TOTAL = VT + 2 * ATT_BK * CV * 2;
  static constexpr uint32_t K_BYTES = ATT_BK * CQ * 2, V_BYTES = ATT_BK * CV * 2;
  // full (per query and key) bias tiles, 2 stages, rows padded to 72 elements (conflict-free
  // 16-byte row reads): only with the FB variant
  static constexpr int BROW = ATT_BK + 8;
  static constexpr uint32_t BS = TOTAL, BS_BYTES = ATT_BQ * BROW * 2;
  static constexpr uint32_t TOTAL_FB = BS + 2 * BS_BYTES;
  // gate rows of the unit's queries for the epilogue (non-FB variant only: FB needs the room)
  static constexpr uint32_t GT = TOTAL, GT_BYTES = ATT_BQ * CP * 2;
  static constexpr uint32_t TOTAL_G = GT + GT_BYTES;
};

// 128 query rows x 64 keys of a full bias into smem (rows padded to BROW): 4 rows of 128
// contiguous bytes per warp instruction
template <int BROW>
__device__ __forceinline__ void att_load_bias(uint32_t sdst, const bf16* base, int64_t row_stride, int q0, int k0,
                                              int L) {
#pragma unroll
  for (int it = 0; it < ATT_BQ * 8 / 128; ++it) {
    const int ch = threadIdx.x + it * 128;
    const int rr = ch >> 3, cc = (ch & 7) * 8;
    const bool ok = (q0 + rr < L) && (k0 + cc < L);
    const bf16* src = ok ? base + (int64_t)(q0 + rr) * row_stride + k0 + cc : base;
    cp_async16(sdst + rr * (BROW * 2) + (ch & 7) * 16, src, ok);
  }
}

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
// keys x CP tile stored MN-major over d (the PV B operand: N = d, K = key; N extent NV)
template <int CP, int NV>
__device__ __forceinline__ void att_load_v(uint32_t sdst, const bf16* base, int64_t row_stride, int row0,
                                           int nrows_valid, int c) {
  constexpr int CPR = CP / 8;
#pragma unroll
  for (int it = 0; it < ATT_BK * CPR / 128; ++it) {
    const int ch = threadIdx.x + it * 128;
    const int r = ch / CPR, d = (ch % CPR) * 8;
    const bool ok = (r < nrows_valid) && (d < c);
    const bf16* src = ok ? base + (int64_t)(row0 + r) * row_stride + d : base;
    cp_async16(sdst + mnmajor_off(d, r, NV), src, ok);
  }
}
__device__ __forceinline__ void att_tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void att_tmem_ld8(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void att_tmem_st8(uint32_t taddr, const float* v) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
// O (+)= P[tmem] * V[smem]^T: A operand (M = 128 lanes, 2 bf16 per 32-bit column) in TMEM
__device__ __forceinline__ void att_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
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

#ifndef EVO_EXP
#define EVO_EXP 0
#endif
#if EVO_EXP == 5
__device__ long long g_fwd_trace[4096];
#define FTR(i)                                                                              \
  do {                                                                                      \
    if (blockIdx.x == 0 && threadIdx.x == 0 && (i) < 4096) evo::g_fwd_trace[(i)] = clock64(); \
  } while (0)
#else
#define FTR(i) (void)0
#endif
int sm_count();

// TMA path (head dim 32): tensor maps whose boxes land exactly in the canonical (SWIZZLE_NONE)
// operand layouts - Q / K [k/8][row/8][row%8][k%8] data groups, V as [d/8][key/8][key%8][d%8]
// (the row-sum group d/8 = 4 stays a constant block after the data), the full-bias tile with its
// padded 72-key rows and the gate rows - so one thread issues a unit's / a tile's loads
struct AttnFwdMaps {
  CUtensorMap q, k, v, bias, g;
};
// V (TMA layout): byte offset of element (key, d) in a stage
__device__ __forceinline__ uint32_t vt_off(int key, int d) {
  return (uint32_t)(((d >> 3) * (ATT_BK / 8) + (key >> 3)) * 128 + (key & 7) * 16 + (d & 7) * 2);
}

// FB: full bias staged through smem with the K/V tiles (msa_row: [1, H, L, L] shared over the
// batch, so the tile loads hit L2) instead of 16-byte global loads after the S wait.
//
// Persistent: each CTA walks units u = (batch, head, query tile) with stride gridDim.x.  The
// K/V stage and the mbarrier phases follow a CTA-wide tile counter, so the last key tile of a
// unit already prefetches the next unit's first K/V tile, and the next unit's Q follows as
// soon as this unit's last S MMA has read Q: the next unit's load latency hides under this
// unit's last softmax and epilogue.
// VAR: 0 = no bias (gate rows prefetched into smem for the epilogue), 1 = per-key bias (4 = the same at
// 3 CTAs/SM with register-prefetched gate rows, for rows of <= 512 keys),
// 2 = full bias staged through smem (FB), 3 = generic full bias (strided global loads)
template <int CP, int VAR>
__global__ void __launch_bounds__(128, CP == 64 ? 2 : ((VAR == 2 || VAR == 4 || EVO_EXP == 1) ? 3 : 4)) attn_fwd_kernel(
    AttnParams P, int nunits, const __grid_constant__ AttnFwdMaps maps, int tmaq) {
  pdl_wait();
  // The epilogue's gate rows are fetched early, with the unit's last tile, so the epilogue does not
  // wait on a DRAM load (a tile trace showed a 4.5-5.2K clk epilogue per unit, ~30 % of it, with the
  // gate loaded there; profiles/r02_attn_fwd_tile_trace.txt): GS (no bias) into smem; GR (the smem-staged
  // full-bias variant, 3 CTAs/SM: registers to spare) into registers (msa_row fwd 58.3 -> 54.6 us).  The
  // per-key-bias variant (4 CTAs/SM at its register limit) keeps the epilogue load: the smem gate
  // tile, registers and an L1 prefetch all measured 3-7 % slower there (spills)
  constexpr bool FB = VAR == 2, GS = VAR == 0, GR = VAR == 2 || VAR == 4;
  using SM = AttnSmem<CP>;
  constexpr int CQ = SM::CQ, CV = SM::CV;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_s, bar_o, kv_full[2], q_full, g_full;
  __shared__ uint32_t tmem_sh;
  const uint32_t sb = smem_u32(smem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int L = P.L, c = P.c, H = P.H;
  const int nqt = (L + ATT_BQ - 1) / ATT_BQ;
  const int r = warp * 32 + lane;  // query row inside the tile
  const bool per_key_bias = VAR == 1 || VAR == 4;
  constexpr uint32_t ONE_BF16 = 0x3F80u;
  const int nkt = (L + ATT_BK - 1) / ATT_BK;

  constexpr uint32_t TCOLS = 64 + CV <= 128 ? 128 : 256;
  if (warp == 0) tmem_alloc(&tmem_sh, TCOLS);
  if (threadIdx.x == 0) {
    mbar_init(&bar_s, 1);
    mbar_init(&bar_o, 1);
    mbar_init(&kv_full[0], 1);
    mbar_init(&kv_full[1], 1);
    mbar_init(&q_full, 1);
    mbar_init(&g_full, 1);
    fence_mbar_init();
  }
  __syncthreads();  // the TMA path issues into these barriers in the prologue

  struct Unit {
    int q0, h;
    int64_t b;
  };
  auto decode = [&](int u) {
    Unit t;
    const int qt = u % nqt, rest = u / nqt;
    t.q0 = qt * ATT_BQ;
    t.h = rest % H;
    t.b = rest / H;
    return t;
  };
  auto kbase = [&](const Unit& t) { return P.k + t.b * P.k_sb + (int64_t)t.h * c; };
  auto vbase = [&](const Unit& t) { return P.v + t.b * P.v_sb + (int64_t)t.h * c; };
  auto kbias_of = [&](const Unit& t) {
    return per_key_bias ? reinterpret_cast<const unsigned short*>(P.bias + t.b * P.bs0 + (int64_t)t.h * P.bs1)
                        : nullptr;
  };
  auto bfull_of = [&](const Unit& t) { return FB ? P.bias + t.b * P.bs0 + (int64_t)t.h * P.bs1 : nullptr; };

  // TMA issue (thread 0): a K/V (+ full-bias) tile into a stage, a unit's Q, a unit's gate rows
  auto tma_kv = [&](const Unit& t, int k0, int st) {
    const uint32_t bytes = 2u * ATT_BK * CP * 2 + (FB ? (uint32_t)(ATT_BQ * SM::BROW * 2) : 0u);
    mbar_expect_tx(&kv_full[st], bytes);
    const uint32_t br = smem_u32(&kv_full[st]);
    tma_ld5(sb + SM::KT + st * SM::K_BYTES, reinterpret_cast<uint64_t>(&maps.k), 0, 0, k0 / 8, t.h * (CP / 8),
            (int)t.b, br);
    tma_ld5(sb + SM::VT + st * SM::V_BYTES, reinterpret_cast<uint64_t>(&maps.v), 0, 0, k0 / 8, t.h * (CP / 8),
            (int)t.b, br);
    if (FB)
      tma_ld4(sb + SM::BS + st * SM::BS_BYTES, reinterpret_cast<uint64_t>(&maps.bias), k0, t.q0, t.h,
              P.bs0 == 0 ? 0 : (int)t.b, br);
  };
  auto tma_q = [&](const Unit& t) {
    mbar_expect_tx(&q_full, (uint32_t)(ATT_BQ * CP * 2));
    tma_ld5(sb + SM::Q, reinterpret_cast<uint64_t>(&maps.q), 0, 0, t.q0 / 8, t.h * (CP / 8), (int)t.b,
            smem_u32(&q_full));
  };
  auto tma_g = [&](const Unit& t) {
    mbar_expect_tx(&g_full, (uint32_t)(ATT_BQ * CP * 2));
    tma_ld4(sb + SM::GT, reinterpret_cast<uint64_t>(&maps.g), 0, t.h, t.q0, (int)t.b, smem_u32(&g_full));
  };
  uint32_t ui = 0;  // CTA-local unit counter: q_full / g_full parity

  int u = blockIdx.x;
  if (u >= nunits) {  // (grid <= nunits by construction)
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem_sh, TCOLS);
    return;
  }
  Unit cur = decode(u);
  // prologue: Q and tile 0 of the first unit into Q buffer 0 / stage 0
  if (tmaq) {
    if (threadIdx.x == 0) {
      tma_q(cur);
      tma_kv(cur, 0, 0);
    }
  } else {
    att_load_kmajor<CP, ATT_BQ>(sb + SM::Q, P.q + cur.b * P.q_sb + (int64_t)cur.h * c, P.q_sl, cur.q0, L - cur.q0, c);
    att_load_kmajor<CP, ATT_BK>(sb + SM::KT, kbase(cur), P.k_sl, 0, L, c);
    att_load_v<CP, CV>(sb + SM::VT, vbase(cur), P.v_sl, 0, L, c);
    if (FB) att_load_bias<SM::BROW>(sb + SM::BS, bfull_of(cur), P.bs2, cur.q0, 0, L);
  }
  cp_async_commit();
  // constant parts of the augmented operands (Q, both K/V stages): Q rows
  // [.. | 1 or 0, 0 x 7 | 0 x 8], K rows' zero group (the bias group is written per tile),
  // V rows' [1, 0 x 7] row-sum column
  st_shared_v4(sb + SM::Q + kmajor_off(r, CP, ATT_BQ), per_key_bias ? ONE_BF16 : 0u, 0u, 0u, 0u);
  st_shared_v4(sb + SM::Q + kmajor_off(r, CP + 8, ATT_BQ), 0u, 0u, 0u, 0u);
  {
    const int st = r / ATT_BK, kr = r % ATT_BK;  // 128 threads = 2 stages x 64 keys
    st_shared_v4(sb + SM::KT + st * SM::K_BYTES + kmajor_off(kr, CP + 8, ATT_BK), 0u, 0u, 0u, 0u);
    st_shared_v4(sb + SM::VT + st * SM::V_BYTES + (tmaq ? vt_off(kr, CP) : mnmajor_off(CP, kr, CV)), ONE_BF16, 0u,
                 0u, 0u);
    if (st == 0)
      st_shared_v4(sb + SM::KT + kmajor_off(kr, CP, ATT_BK),
                   (per_key_bias && kr < L) ? (uint32_t)kbias_of(cur)[(int64_t)kr * P.bs3] : 0u, 0u, 0u, 0u);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;
  const uint32_t t_row = tmem + ((uint32_t)(warp * 32) << 16);

  constexpr uint32_t IDESC_S = make_idesc_bf16(128, ATT_BK, 0, 0);
  constexpr uint32_t IDESC_O = make_idesc_bf16(128, CV, 0, 1);
  constexpr uint32_t T_O = 64;  // O and its row sum (column CP) accumulate in TMEM [64, 64 + CV)
  const int ksteps = per_key_bias ? CQ / 16 : CP / 16;

  uint32_t gt = 0;  // CTA-wide tile counter: K/V stage = gt & 1, mbarrier phase parity = gt & 1
  while (u < nunits) {
    const int nu = u + gridDim.x;
    const bool has_next = nu < nunits;
    const Unit nxt = decode(has_next ? nu : u);
    const int q0 = cur.q0, h = cur.h;
    const int64_t b = cur.b;
    const int qi = q0 + r;
    const bf16* kb = kbase(cur);
    const bf16* vb = vbase(cur);
    const unsigned short* kbias = kbias_of(cur);
    const bf16* bfull = bfull_of(cur);
    float m_run = -INFINITY;  // running max, scaled log2 units
    uint4 greg[GR ? CP / 8 : 1];  // GR: the gate rows of this thread's query (loaded with the last tile)
    const bf16* brow = nullptr;
    if (VAR == 3 && qi < L) brow = P.bias + b * P.bs0 + (int64_t)h * P.bs1 + (int64_t)qi * P.bs2;
    uint32_t nb = 0;  // next tile's per-key bias (threads 0..63), stored with its K tile

    for (int j = 0; j < nkt; ++j, ++gt) {
      const int k0 = j * ATT_BK;
      const int st = gt & 1;
      FTR(gt * 8 + 0);
      cp_async_wait<0>();
      if (tmaq) {
        mbar_wait(&kv_full[st], (gt >> 1) & 1);
        if (j == 0) mbar_wait(&q_full, ui & 1);
      }
      fence_async_smem();
      __syncthreads();
      FTR(gt * 8 + 1);
      // prefetch into the other stage (its MMAs finished last iteration): this unit's next
      // K/V tile, or on the last tile the next unit's first K/V tile
      const uint32_t kdst = sb + SM::KT + (st ^ 1) * SM::K_BYTES, vdst = sb + SM::VT + (st ^ 1) * SM::V_BYTES;
      if (j + 1 < nkt) {
        if (tmaq) {
          if (threadIdx.x == 0) tma_kv(cur, k0 + ATT_BK, st ^ 1);
        } else {
          att_load_kmajor<CP, ATT_BK>(kdst, kb, P.k_sl, k0 + ATT_BK, L - k0 - ATT_BK, c);
          att_load_v<CP, CV>(vdst, vb, P.v_sl, k0 + ATT_BK, L - k0 - ATT_BK, c);
          if (FB) att_load_bias<SM::BROW>(sb + SM::BS + (st ^ 1) * SM::BS_BYTES, bfull, P.bs2, q0, k0 + ATT_BK, L);
        }
        if (per_key_bias && threadIdx.x < ATT_BK) {
          const int k = k0 + ATT_BK + threadIdx.x;
          nb = k < L ? (uint32_t)kbias[(int64_t)k * P.bs3] : 0u;
        }
      } else if (has_next) {
        if (tmaq) {
          if (threadIdx.x == 0) tma_kv(nxt, 0, st ^ 1);
        } else {
          att_load_kmajor<CP, ATT_BK>(kdst, kbase(nxt), P.k_sl, 0, L, c);
          att_load_v<CP, CV>(vdst, vbase(nxt), P.v_sl, 0, L, c);
          if (FB) att_load_bias<SM::BROW>(sb + SM::BS + (st ^ 1) * SM::BS_BYTES, bfull_of(nxt), P.bs2, nxt.q0, 0, L);
        }
        if (per_key_bias && threadIdx.x < ATT_BK)
          nb = (int)threadIdx.x < L ? (uint32_t)kbias_of(nxt)[(int64_t)threadIdx.x * P.bs3] : 0u;
      }
      cp_async_commit();
      if (GS && j + 1 == nkt) {  // this unit's gate rows
        if (tmaq) {
          if (threadIdx.x == 0) tma_g(cur);
        } else if (qi < L) {  // (own row: no barrier needed)
          const bf16* gsrc = P.g + b * P.g_sb + (int64_t)qi * P.g_sl + (int64_t)h * c;
#pragma unroll
          for (int d = 0; d < CP; d += 8)
            if (d < c) cp_async16(sb + SM::GT + r * (CP * 2) + d * 2, gsrc + d, true);
        }
      }
      if (GS) cp_async_commit();
      if (GR && j + 1 == nkt && qi < L) {  // gate rows into registers, consumed by the epilogue
        const bf16* gsrc = P.g + b * P.g_sb + (int64_t)qi * P.g_sl + (int64_t)h * c;
#pragma unroll
        for (int d = 0; d < CP; d += 8)
          if (d < c) greg[d / 8] = *reinterpret_cast<const uint4*>(gsrc + d);
      }

      if (threadIdx.x == 0) {
        // S overwrites the columns the previous tile's P was read from: its PV must be complete
        if (gt > 0) mbar_wait(&bar_o, (gt - 1) & 1);
        tc_fence_after();
        for (int kk = 0; kk < ksteps; ++kk) {
          uint64_t ad = make_sdesc(sb + SM::Q + kk * 2 * (128 / 8) * 128, (128 / 8) * 128, 128);
          uint64_t bd = make_sdesc(sb + SM::KT + st * SM::K_BYTES + kk * 2 * (ATT_BK / 8) * 128, (ATT_BK / 8) * 128,
                                   128);
          mma_bf16(tmem, ad, bd, IDESC_S, kk != 0);
        }
        mma_commit(&bar_s);
      }
      // bar_s completes after S, which was issued after the previous PV completed: O is stable
      mbar_wait(&bar_s, gt & 1);
      FTR(gt * 8 + 2);
      tc_fence_after();
      if (j + 1 == nkt && has_next) {  // Q is free: this unit's last S MMA has completed
        if (tmaq) {
          if (threadIdx.x == 0) tma_q(nxt);
        } else {
          att_load_kmajor<CP, ATT_BQ>(sb + SM::Q, P.q + nxt.b * P.q_sb + (int64_t)nxt.h * c, P.q_sl, nxt.q0,
                                      L - nxt.q0, c);
          cp_async_commit();
        }
      }

      float s[ATT_BK];
#pragma unroll
      for (int cc = 0; cc < ATT_BK; cc += 32) tmem_ld32(t_row + cc, s + cc);
      tmem_ld_wait();

      // full bias (before the scale, G1); keys >= L masked on the last tile only
      const bool full_tile = k0 + ATT_BK <= L;
      if (FB) {
        const uint32_t brs = sb + SM::BS + st * SM::BS_BYTES + r * (SM::BROW * 2);
#pragma unroll
        for (int kk = 0; kk < ATT_BK; kk += 8) {
          uint32_t u0, u1, u2, u3;
          asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];\n" : "=r"(u0), "=r"(u1), "=r"(u2), "=r"(u3)
                       : "r"(brs + kk * 2));
          float t[8];
          unpack_bf16x2(u0, t[0], t[1]); unpack_bf16x2(u1, t[2], t[3]);
          unpack_bf16x2(u2, t[4], t[5]); unpack_bf16x2(u3, t[6], t[7]);
#pragma unroll
          for (int e = 0; e < 8; ++e) s[kk + e] += t[e];
        }
      } else if (brow) {
        if (P.bias_vec && full_tile) {
#pragma unroll
          for (int kk = 0; kk < ATT_BK; kk += 8) {
            uint4 w = *reinterpret_cast<const uint4*>(brow + k0 + kk);
            float t[8];
            unpack_bf16x2(w.x, t[0], t[1]); unpack_bf16x2(w.y, t[2], t[3]);
            unpack_bf16x2(w.z, t[4], t[5]); unpack_bf16x2(w.w, t[6], t[7]);
#pragma unroll
            for (int e = 0; e < 8; e += 2) {  // FADD2
              const float2 r = __fadd2_rn(make_float2(s[kk + e], s[kk + e + 1]), make_float2(t[e], t[e + 1]));
              s[kk + e] = r.x;
              s[kk + e + 1] = r.y;
            }
          }
        } else {
#pragma unroll
          for (int kk = 0; kk < ATT_BK; ++kk)
            if (k0 + kk < L) s[kk] += bf2f(brow[(int64_t)(k0 + kk) * P.bs3]);
        }
      }
      if (!full_tile) {
#pragma unroll
        for (int kk = 0; kk < ATT_BK; ++kk)
          if (k0 + kk >= L) s[kk] = -INFINITY;
      }
      float m8[8];  // row max: 8 chains of three-input max (FMNMX3)
#pragma unroll
      for (int e = 0; e < 8; ++e) m8[e] = fmax3f(s[e], s[e + 8], s[e + 16]);
#pragma unroll
      for (int kk = 24; kk + 16 <= ATT_BK; kk += 16) {
#pragma unroll
        for (int e = 0; e < 8; ++e) m8[e] = fmax3f(m8[e], s[kk + e], s[kk + 8 + e]);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) m8[e] = fmaxf(m8[e], s[ATT_BK - 8 + e]);
      const float mxs = P.scale_log2 * fmax3f(fmax3f(m8[0], m8[1], m8[2]), fmax3f(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
      // lazy rescale: O (and l) in TMEM are rescaled only when a row's max grows by > 2^8
      // (warp-uniform: TMEM loads/stores are warp-collective); P <= 2^8 is exact enough in bf16
      const bool grow = mxs > m_run + 8.0f;
      if (__any_sync(0xffffffffu, grow)) {
        const float m_new = grow ? mxs : m_run;
        if (j > 0) {
          const float f = ex2f(m_run - m_new);
#pragma unroll
          for (int cc = 0; cc < CV; cc += 8) {
            float v[8];
            att_tmem_ld8(t_row + T_O + cc, v);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] *= f;
            att_tmem_st8(t_row + T_O + cc, v);
          }
        }
        m_run = m_new;
      }
      const float mref = m_run == -INFINITY ? 0.f : m_run;
      // P over S in TMEM columns [0, 32): this thread's row of S was read above
#pragma unroll
      for (int half = 0; half < 2; ++half) {  // 16 packed columns at a time (register budget)
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int kk = half * 32 + 2 * e;
          const float2 y = __ffma2_rn(make_float2(s[kk], s[kk + 1]), make_float2(P.scale_log2, P.scale_log2),
                                      make_float2(-mref, -mref));  // FFMA2
          pk[e] = pack_bf16x2(ex2f(y.x), ex2f(y.y));
        }
        tmem_st16(t_row + half * 16, reinterpret_cast<const float*>(pk));
      }
      // the next tile's per-key bias into its K tile's bias group (stage st^1, loaded above)
      if (per_key_bias && threadIdx.x < ATT_BK && (j + 1 < nkt || has_next))
        st_shared_v4(sb + SM::KT + (st ^ 1) * SM::K_BYTES + kmajor_off(threadIdx.x, CP, ATT_BK), nb, 0u, 0u, 0u);
      tmem_st_wait();
      FTR(gt * 8 + 3);
      tc_fence_before();
      __syncthreads();
      FTR(gt * 8 + 4);
      if (threadIdx.x == 0) {
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < ATT_BK / 16; ++kk) {
          const uint64_t bd =
              tmaq ? make_sdesc(sb + SM::VT + st * SM::V_BYTES + kk * 2 * 128, 128, (ATT_BK / 8) * 128)
                   : make_sdesc(sb + SM::VT + st * SM::V_BYTES + kk * 2 * (CV / 8) * 128, (CV / 8) * 128, 128);
          att_mma_ts(tmem + T_O, tmem + kk * 8, bd, IDESC_O, (j > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&bar_o);
      }
    }
    // O and l of this row (the next unit's first PV overwrites O only after the __syncthreads
    // at the top of its first tile, which every thread reaches after these TMEM loads)
    FTR((gt - 1) * 8 + 5);
    mbar_wait(&bar_o, (gt - 1) & 1);
    FTR((gt - 1) * 8 + 6);
    tc_fence_after();
    float o_acc[CV];
#pragma unroll
    for (int cc = 0; cc < CV; cc += 8) att_tmem_ld8(t_row + T_O + cc, o_acc + cc);
    tmem_ld_wait();
    tc_fence_before();
    const float l_run = o_acc[CP];

    if (GS) {  // the gate group: only the next unit's Q group may still be in flight
      if (tmaq) {
        mbar_wait(&g_full, ui & 1);
      } else if (has_next) {
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
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
          uint4 w0;
          if constexpr (GR) {
            w0 = greg[d / 8];
          } else if constexpr (!GS) {
            w0 = *reinterpret_cast<const uint4*>(gp + d);
          } else {
            asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];\n" : "=r"(w0.x), "=r"(w0.y), "=r"(w0.z), "=r"(w0.w)
                         : "r"(sb + SM::GT + r * (CP * 2) + d * 2));
          }
          unpack_bf16x2(w0.x, gv[0], gv[1]); unpack_bf16x2(w0.y, gv[2], gv[3]);
          unpack_bf16x2(w0.z, gv[4], gv[5]); unpack_bf16x2(w0.w, gv[6], gv[7]);
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
      if (P.lse) P.lse[(b * P.H + h) * (int64_t)L + qi] = (m_run + log2f(l_run)) * 0.6931471805599453f;
    }
    FTR((gt - 1) * 8 + 7);
    u = nu;
    cur = nxt;
    ++ui;
  }

  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, TCOLS);
}

static bool a16(const void* p) { return ((uintptr_t)p & 15) == 0; }

static bool fwd_map5(CUtensorMap* m, const void* base, int H, int64_t L, int64_t B, int64_t sl, int64_t sb, bool v) {
  // Q / K: (d%8, row%8, row/8, d/8 over all heads, b) box [8][8][rows/8][4][1];  V: (d%8, key%8, key/8, d/8, b)
  // with the boxes ordered so the smem image is [d/8][key/8][key%8][d%8]
  EncodeTiledFn enc = encode_tiled();
  if (!enc || ((uintptr_t)base & 15) || (sl * 2) % 16 || (sb * 2) % 16) return false;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  if (!v) {
    cuuint64_t d[5] = {8, 8, (cuuint64_t)((L + 7) / 8), (cuuint64_t)(H * 4), (cuuint64_t)B};
    cuuint64_t s[4] = {(cuuint64_t)sl * 2, (cuuint64_t)sl * 16, 16, (cuuint64_t)sb * 2};
    cuuint32_t bx[5] = {8, 8, 16, 4, 1};  // Q box; K tiles use the first 8 row groups (set below)
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), d, s, bx, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  cuuint64_t d[5] = {8, 8, (cuuint64_t)((L + 7) / 8), (cuuint64_t)(H * 4), (cuuint64_t)B};
  cuuint64_t s[4] = {(cuuint64_t)sl * 2, (cuuint64_t)sl * 16, 16, (cuuint64_t)sb * 2};
  cuuint32_t bx[5] = {8, 8, 8, 4, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), d, s, bx, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int CP, int VAR>
static int launch_attn_fwd_v(const AttnParams& p, int64_t B, cudaStream_t st) {
  using SM = AttnSmem<CP>;
  constexpr bool FB = VAR == 2;
  constexpr uint32_t bytes = FB ? SM::TOTAL_FB : (VAR == 0 ? SM::TOTAL_G : SM::TOTAL);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel<CP, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return cuda_status(e, "attn fwd attr");
    attr = true;
  }
  // resident CTAs per SM: the launch bound (registers; TMEM 4 x 128 columns) or what fits in
  // 228 KB of shared memory (1 KB reserved per CTA), whichever is smaller.  The persistent grid
  // is exactly one wave: measured, a grid above the resident count is slower (uneven tails).
  constexpr int occ_lb = CP == 64 ? 2 : ((FB || VAR == 4 || EVO_EXP == 1) ? 3 : 4);
  constexpr int occ_sm = (int)((228u * 1024u) / (bytes + 1024u + 64u));
  static int occ = occ_lb < occ_sm ? occ_lb : occ_sm;
  if (EVO_EXP == 2) {
    if (const char* ev = getenv("EVO_FWD_OCC")) occ = atoi(ev);
  }
  const int64_t nunits = (int64_t)((p.L + ATT_BQ - 1) / ATT_BQ) * p.H * B;
  EVO_CHECK_ARG(nunits < (1ll << 31), EVO_ERR_SHAPE, "attention fwd: too many (batch, head, query tile) units");
  const int64_t cap = (int64_t)occ * sm_count();
  AttnFwdMaps maps;
  memset(&maps, 0, sizeof(maps));
  static const bool tma_off = [] { const char* e = getenv("EVO_ATTN_FWD_NO_TMA"); return e && e[0] == '1'; }();
  // rows more than 1 MB apart (the column variants at N_r >= 2048: every 16-byte box row of a tile in
  // another 2 MB page) measured slower through TMA than through per-thread cp.async (pair_col at N_r =
  // 2048: 2.3x; msa_col at 400 KB and pair_col at 800 KB are faster through TMA), so those keep cp.async
  const bool near_rows = p.q_sl * 2 <= (1 << 20) && p.k_sl * 2 <= (1 << 20) && p.v_sl * 2 <= (1 << 20);
  int tmaq = !tma_off && near_rows && CP == 32 && p.c == 32 && p.L % 8 == 0 && fwd_map5(&maps.q, p.q, p.H, p.L, B, p.q_sl, p.q_sb, false) &&
             fwd_map5(&maps.k, p.k, p.H, p.L, B, p.k_sl, p.k_sb, false) &&
             fwd_map5(&maps.v, p.v, p.H, p.L, B, p.v_sl, p.v_sb, true);
  if (tmaq) {  // K tiles: 64 rows (8 row groups); V box written in the [d/8][key/8][key%8][d%8] order
    EncodeTiledFn enc = encode_tiled();
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    {
      cuuint64_t d[5] = {8, 8, (cuuint64_t)(p.L / 8), (cuuint64_t)(p.H * 4), (cuuint64_t)B};
      cuuint64_t s[4] = {(cuuint64_t)p.k_sl * 2, (cuuint64_t)p.k_sl * 16, 16, (cuuint64_t)p.k_sb * 2};
      cuuint32_t bx[5] = {8, 8, 8, 4, 1};
      tmaq = enc(&maps.k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<bf16*>(p.k), d, s, bx, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    if (tmaq) {  // V: dims reordered (d%8, key%8, key/8, d/8, b) -> smem [d/8][key/8][key%8][d%8]
      cuuint64_t d[5] = {8, 8, (cuuint64_t)(p.L / 8), (cuuint64_t)(p.H * 4), (cuuint64_t)B};
      cuuint64_t s[4] = {(cuuint64_t)p.v_sl * 2, (cuuint64_t)p.v_sl * 16, 16, (cuuint64_t)p.v_sb * 2};
      cuuint32_t bx[5] = {8, 8, 8, 4, 1};
      tmaq = enc(&maps.v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<bf16*>(p.v), d, s, bx, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    if (tmaq && FB) {  // full bias [b?][h][q][key]: box [72 keys][128 q] = the padded smem rows
      cuuint64_t d[4] = {(cuuint64_t)p.L, (cuuint64_t)p.L, (cuuint64_t)p.H, (cuuint64_t)(p.bs0 == 0 ? 1 : B)};
      cuuint64_t s[3] = {(cuuint64_t)p.bs2 * 2, (cuuint64_t)p.bs1 * 2,
                         (cuuint64_t)(p.bs0 == 0 ? p.bs1 * p.H : p.bs0) * 2};
      cuuint32_t bx[4] = {(cuuint32_t)SM::BROW, ATT_BQ, 1, 1};
      tmaq = p.bs3 == 1 && (p.bs2 * 2) % 16 == 0 && (p.bs1 * 2) % 16 == 0 && (p.bs0 * 2) % 16 == 0 &&
             enc(&maps.bias, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<bf16*>(p.bias), d, s, bx, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    if (tmaq && VAR == 0) {  // gate rows [b][l][h*c]: box [32 d][1 h][128 l][1 b]
      cuuint64_t d[4] = {32, (cuuint64_t)p.H, (cuuint64_t)p.L, (cuuint64_t)B};
      cuuint64_t s[3] = {64, (cuuint64_t)p.g_sl * 2, (cuuint64_t)p.g_sb * 2};
      cuuint32_t bx[4] = {32, 1, ATT_BQ, 1};
      tmaq = (p.g_sl * 2) % 16 == 0 && (p.g_sb * 2) % 16 == 0 && a16(p.g) &&
             enc(&maps.g, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<bf16*>(p.g), d, s, bx, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
  }
  ::evo::pdl_launch(attn_fwd_kernel<CP, VAR>, (unsigned)(nunits < cap ? nunits : cap), 128, bytes, st, p, (int)nunits, maps, tmaq);
  EVO_LAUNCH_CHECK("attention fwd");
  return EVO_OK;
}

template <int CP>
static int launch_attn_fwd(const AttnParams& p, int64_t B, int flags, cudaStream_t st) {
  if (!p.bias) return launch_attn_fwd_v<CP, 0>(p, B, st);
  // per-key bias: up to 512 keys the 3-CTA/SM form with register-prefetched gate rows (VAR 4: pair_row /
  // pair_col forward 50.3 / 51.2 -> 48.4 / 48.8 us at the training shape); longer rows keep 4 CTAs/SM
  // (VAR 1: at N_r = 1024 / 2048 the 3-CTA form measured 9-10 % slower)
  if (p.bs2 == 0) return p.L <= 512 ? launch_attn_fwd_v<CP, 4>(p, B, st) : launch_attn_fwd_v<CP, 1>(p, B, st);
  // a full bias is staged through smem with the K/V tiles unless EVO_ATTN_NO_BIAS_SMEM
  if (!(flags & EVO_ATTN_NO_BIAS_SMEM) && p.bias_vec) return launch_attn_fwd_v<CP, 2>(p, B, st);
  return launch_attn_fwd_v<CP, 3>(p, B, st);
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
constexpr int kWsMinLen = 4096;  // measured: faster than attn_fwd_kernel from N_r = 4096 on (per-key/no bias)
}  // namespace evo

#if EVO_EXP == 5
extern "C" int evo_fwd_trace(void* dst) { return (int)cudaMemcpyFromSymbol(dst, evo::g_fwd_trace, sizeof(evo::g_fwd_trace)); }
#endif
extern "C" int evo_gated_attention_fwd(const EvoAttnDesc* d, void* stream) {
  AttnParams p;
  int rc = attn_params_from_desc(d, p);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int flags = d->flags;
  EVO_CHECK_ARG((flags & ~(EVO_ATTN_FORCE_WS | EVO_ATTN_FORCE_FLASH | EVO_ATTN_NO_BIAS_SMEM)) == 0 &&
                    (flags & (EVO_ATTN_FORCE_WS | EVO_ATTN_FORCE_FLASH)) != (EVO_ATTN_FORCE_WS | EVO_ATTN_FORCE_FLASH),
                EVO_ERR_ARG, "attention fwd: bad flags 0x%x", flags);
  // the full (per query and key) bias path of the warp-specialised kernel measured slower
  const bool ws_auto = p.L >= kWsMinLen && (!p.bias || p.bs2 == 0);
  if ((flags & EVO_ATTN_FORCE_WS) || (ws_auto && !(flags & EVO_ATTN_FORCE_FLASH))) {
    if (p.c <= 16) return launch_attn_fwd_ws<16>(p, d->B, st);
    if (p.c <= 32) return launch_attn_fwd_ws<32>(p, d->B, st);
    return launch_attn_fwd_ws<64>(p, d->B, st);
  }
  if (p.c <= 16) return launch_attn_fwd<16>(p, d->B, flags, st);
  if (p.c <= 32) return launch_attn_fwd<32>(p, d->B, flags, st);
  return launch_attn_fwd<64>(p, d->B, flags, st);
}
