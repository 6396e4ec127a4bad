// Warp-specialised forward of the gated attention for long sequences (N_r >= 512), the
// long-sequence inference path of _attention_core (evoformer.py:173-198).  Same math and
// outputs as attn_fwd_kernel (attention.cu); different schedule:
//
//   CTA = 256 queries (two 128-query tiles) of one (batch, head); 1 CTA per SM, 11 warps:
//     warps 0-3   softmax warpgroup 0 (query tile 0, thread = query row = TMEM lane)
//     warps 4-7   softmax warpgroup 1 (query tile 1)
//     warp  8/10  MMA issuers of warpgroup 0/1 (one lane each): S_w = Q_w K_j^T, O_w += P_w V_j;
//                 one issuer per warpgroup so neither waits on the other's softmax
//     warp  9     loader: cp.async K/V (+ per-key bias) ring of WS_NS stages, completion
//                 tracked by cp.async.mbarrier.arrive.noinc
//   The two warpgroups take turns on the exponential phase (named barriers 1/2, ping-pong):
//   one warpgroup's TMEM load, row max and P store run under the other's MUFU work
//   (in-kernel clock trace: tile period 2039 -> 1791 clk; profiles/r02_ws_pingpong_trace.txt).
//   K/V tiles (64 keys) are loaded once and shared by both query tiles.  S is double
//   buffered per warpgroup in TMEM and P (bf16) is written back over S in TMEM and read from
//   there by the PV MMA (A operand in tensor memory), so the tensor core works
//   on tile j+1 while the warpgroups run the softmax of tile j, and the two warpgroups
//   interleave on the MUFU/FMA pipes.  O accumulates in TMEM; a row's O is rescaled (TMEM
//   load-scale-store, warp-uniform) only when its running max grows by more than 2^8, so the
//   common case does no O traffic at all (P <= 2^8 stays exact enough in bf16 and l is fp32).
//
// Two pieces of softmax arithmetic ride on the tensor core instead of the FP32/ALU pipes:
//   * a per-key bias (pair_row / pair_col) is an extra K-dimension group of the S product:
//     Q is augmented with a column of ones and each K row with its key's bias, so
//     S = [Q | 1] [K | b]^T = QK^T + b with no per-element bias add (G1: before the scale);
//   * the row sums l = sum_k P[q,k] are an extra N column of the PV product: V is augmented
//     with a column of ones, so O[:, CP] = P 1 accumulates (and is rescaled) with O.
//
// TMEM (512 cols): S[w][buf] at (2w+buf)*64, O[w] (CP + 8 cols, column CP = l) at 256 + w*128.
// mbarrier phases are tracked per buffer so a waiter can never be lapped (see comments).
#include "attn.cuh"

#ifndef EVO_EXP
#define EVO_EXP 0
#endif

namespace evo {

#if EVO_EXP == 12
__device__ long long g_ws_trace[3 * 4096];
#define WTRACE(slot, i)                                                                         \
  do {                                                                                          \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (i) < 4096) g_ws_trace[(slot) * 4096 + (i)] = clock64(); \
  } while (0)
#else
#define WTRACE(slot, i) (void)0
#endif

constexpr int WS_BQ = 128;
constexpr int WS_BK = 64;
constexpr int WS_THREADS = 352;
constexpr float WS_RESCALE = 8.0f;

  // log2 units: rescale O when the max grows by > 2^8

template <int CP>
struct WsSmem {
  // K/V ring depth: deep enough to cover an L2/DRAM round trip (~3 tiles of softmax time)
  static constexpr int NS = CP <= 32 ? 8 : 4;
  static constexpr int CQ = CP + 16;  // Q / K K-extent: CP data + [1 | bias] group + zero group
  static constexpr int CV = CP + 8;   // V N-extent: CP data + [1, 0..0] (row sums)
  static constexpr uint32_t Q = 0;                                  // 2 x [128][CQ] K-major
  static constexpr uint32_t K = Q + 2 * WS_BQ * CQ * 2;             // NS x [64][CQ] K-major
  static constexpr uint32_t V = K + NS * WS_BK * CQ * 2;         // NS x [64 keys][CV] MN-major over d
  static constexpr uint32_t TOTAL = V + NS * WS_BK * CV * 2;  // (P lives in TMEM, over S)
  static constexpr uint32_t Q_BYTES = WS_BQ * CQ * 2, K_BYTES = WS_BK * CQ * 2, V_BYTES = WS_BK * CV * 2;
};

__device__ __forceinline__ void ws_arrive(uint64_t* bar) {
  asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void ws_cp_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void ws_tmem_ld8(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void ws_tmem_st8(uint32_t taddr, const float* v) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]^T: the A operand (M = 128 lanes, K packed 2 bf16 per 32-bit
// column) is read from tensor memory - P never leaves TMEM
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
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
__device__ __forceinline__ void ws_tmem_st32(uint32_t taddr, const uint32_t* r) {
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

// O row (NC fp32 columns, row sum included) scaled in place: warp-collective TMEM load/store
template <int NC>
__device__ __forceinline__ void ws_scale_o(uint32_t taddr, float f) {
#pragma unroll
  for (int cc = 0; cc < NC; cc += 8) {
    float v[8];
    ws_tmem_ld8(taddr + cc, v);
    tmem_ld_wait();
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] *= f;
    ws_tmem_st8(taddr + cc, v);
  }
  tmem_st_wait();
}

template <int CP>
__global__ void __launch_bounds__(WS_THREADS, 1) attn_fwd_ws_kernel(AttnParams P) {
  pdl_wait();
  using SM = WsSmem<CP>;
  constexpr int CQ = SM::CQ, CV = SM::CV, WS_NS = SM::NS;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t q_full, kv_full[WS_NS], kv_empty[WS_NS], s_full[2][2], p_full[2][2], o_done[2][2];
  __shared__ uint32_t tmem_sh;
  const uint32_t sb = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = blockIdx.x * (2 * WS_BQ);
  const int h = blockIdx.y;
  const int64_t b = blockIdx.z;
  const int L = P.L, c = P.c;
  const int nkt = (L + WS_BK - 1) / WS_BK;
  const bool per_key_bias = P.bias && P.bs2 == 0;
  const uint32_t ONE_BF16 = 0x3F80u;  // bf16(1.0) in the low half of a 32-bit word

  if (warp == 8) tmem_alloc(&tmem_sh, 512);
  if (threadIdx.x == 0) {
    // loader arrivals: 32 cp.async completions (noinc) + 32 plain arrivals for its st.shared
    mbar_init(&q_full, 64);
    for (int s = 0; s < WS_NS; ++s) {
      mbar_init(&kv_full[s], 64);
      mbar_init(&kv_empty[s], 2);  // one PV commit per warpgroup
    }
    for (int w = 0; w < 2; ++w)
      for (int i = 0; i < 2; ++i) {
        mbar_init(&s_full[w][i], 1);
        mbar_init(&p_full[w][i], WS_BQ);
        mbar_init(&o_done[w][i], 1);
      }
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;

  const bf16* qb = P.q + b * P.q_sb + (int64_t)h * c;
  const bf16* kb = P.k + b * P.k_sb + (int64_t)h * c;
  const bf16* vb = P.v + b * P.v_sb + (int64_t)h * c;

  if (warp == 9) {
    // ------------------------------------------------------------------ loader
    constexpr int CPR = CP / 8;  // 16-byte data chunks per row
#pragma unroll 1
    for (int ch = lane; ch < 2 * WS_BQ * CPR; ch += 32) {
      const int w = ch / (WS_BQ * CPR), r = (ch / CPR) % WS_BQ, d = (ch % CPR) * 8;
      const int qi = q0 + w * WS_BQ + r;
      const bool ok = qi < L && d < c;
      cp_async16(sb + SM::Q + w * SM::Q_BYTES + kmajor_off(r, d, WS_BQ), ok ? qb + (int64_t)qi * P.q_sl + d : qb,
                 ok);
    }
    ws_cp_arrive(&q_full);
    // constant parts of the augmented operands (never overwritten by the tile loads):
    //   Q rows: [.. | 1 (per-key bias) or 0, 0 x 7 | 0 x 8];  K rows: [.. | b_k, 0 x 7 | 0 x 8]
    //   (the b_k group is rewritten per tile);  V rows: [.. | 1, 0 x 7] (row sums)
    const uint32_t qone = per_key_bias ? ONE_BF16 : 0u;
#pragma unroll 1
    for (int r = lane; r < 2 * WS_BQ; r += 32) {
      const uint32_t base = sb + SM::Q + (r / WS_BQ) * SM::Q_BYTES;
      st_shared_v4(base + kmajor_off(r % WS_BQ, CP, WS_BQ), qone, 0u, 0u, 0u);
      st_shared_v4(base + kmajor_off(r % WS_BQ, CP + 8, WS_BQ), 0u, 0u, 0u, 0u);
    }
#pragma unroll 1
    for (int r = lane; r < WS_NS * WS_BK; r += 32) {
      const uint32_t kbase = sb + SM::K + (r / WS_BK) * SM::K_BYTES;
      st_shared_v4(kbase + kmajor_off(r % WS_BK, CP, WS_BK), 0u, 0u, 0u, 0u);
      st_shared_v4(kbase + kmajor_off(r % WS_BK, CP + 8, WS_BK), 0u, 0u, 0u, 0u);
      // V MN-major [k/8][n/8][k%8][n%8]: the 8 n-columns CP..CP+7 of key row k are one 16-byte run
      st_shared_v4(sb + SM::V + (r / WS_BK) * SM::V_BYTES + mnmajor_off(CP, r % WS_BK, CV), ONE_BF16, 0u, 0u, 0u);
    }
    fence_async_smem();
    ws_arrive(&q_full);
    const bf16* kbias = per_key_bias ? P.bias + b * P.bs0 + (int64_t)h * P.bs1 : nullptr;
    // per-key bias values are read one tile ahead (plain loads) and stored with the tile
    uint16_t nb[WS_BK / 32];
    auto load_bias = [&](int k0) {
#pragma unroll
      for (int it = 0; it < WS_BK / 32; ++it) {
        const int k = k0 + lane + it * 32;
        nb[it] = (per_key_bias && k < L) ? __ldg(reinterpret_cast<const unsigned short*>(kbias) + (int64_t)k * P.bs3)
                                         : (uint16_t)0;
      }
    };
    load_bias(0);
#pragma unroll 1
    for (int j = 0; j < nkt; ++j) {
      const int s = j % WS_NS;
      // slot s last held tile j - NS: its PV commit is completion #(j/NS - 1) of kv_empty[s]
      if (j >= WS_NS) mbar_wait(&kv_empty[s], ((j / WS_NS) - 1) & 1);
      const int k0 = j * WS_BK;
#pragma unroll
      for (int it = 0; it < WS_BK * CPR / 32; ++it) {
        const int ch = lane + it * 32;
        const int r = ch / CPR, d = (ch % CPR) * 8;
        const bool ok = k0 + r < L && d < c;
        cp_async16(sb + SM::K + s * SM::K_BYTES + kmajor_off(r, d, WS_BK), ok ? kb + (int64_t)(k0 + r) * P.k_sl + d : kb,
                   ok);
        cp_async16(sb + SM::V + s * SM::V_BYTES + mnmajor_off(d, r, CV), ok ? vb + (int64_t)(k0 + r) * P.v_sl + d : vb,
                   ok);
      }
      ws_cp_arrive(&kv_full[s]);
      if (per_key_bias) {
#pragma unroll
        for (int it = 0; it < WS_BK / 32; ++it)
          st_shared_v4(sb + SM::K + s * SM::K_BYTES + kmajor_off(lane + it * 32, CP, WS_BK), (uint32_t)nb[it], 0u, 0u,
                       0u);
        fence_async_smem();
        if (j + 1 < nkt) load_bias(k0 + WS_BK);
      }
      ws_arrive(&kv_full[s]);
    }
    cp_async_wait<0>();
  } else if (warp == 8 || warp == 10) {
    // ------------------------------------------------------------------ MMA issuers
    const int w = warp == 8 ? 0 : 1;
    if (lane == 0) {
      constexpr uint32_t IDESC_S = make_idesc_bf16(128, WS_BK, 0, 0);
      constexpr uint32_t IDESC_O = make_idesc_bf16(128, CV, 0, 1);
      const int ksteps = per_key_bias ? CQ / 16 : CP / 16;
      mbar_wait(&q_full, 0);
      fence_async_smem();
      for (int j = 0; j <= nkt; ++j) {
        if (j < nkt) {
          const int s = j % WS_NS, buf = j & 1;
          mbar_wait(&kv_full[s], (j / WS_NS) & 1);
          if (w == 0) WTRACE(2, j * 8 + 0);
          fence_async_smem();
          // S[w][buf] last held P_{j-2} (written over S_{j-2}), read by PV_{j-2}: completion
          // #((j-2)/2) of o_done[w][buf]; the softmax read of S_{j-2} preceded its p_full
          if (j >= 2) mbar_wait(&o_done[w][buf], ((j - 2) >> 1) & 1);
          if (w == 0) WTRACE(2, j * 8 + 1);
          tc_fence_after();
          for (int kk = 0; kk < ksteps; ++kk) {
            const uint64_t ad = make_sdesc(sb + SM::Q + w * SM::Q_BYTES + kk * 2 * (WS_BQ / 8) * 128,
                                           (WS_BQ / 8) * 128, 128);
            const uint64_t bd = make_sdesc(sb + SM::K + s * SM::K_BYTES + kk * 2 * (WS_BK / 8) * 128,
                                           (WS_BK / 8) * 128, 128);
            mma_bf16(tmem + (2 * w + buf) * WS_BK, ad, bd, IDESC_S, kk != 0);
          }
          mma_commit(&s_full[w][buf]);
        }
        if (j >= 1) {
          const int jj = j - 1, s = jj % WS_NS, buf = jj & 1;
          mbar_wait(&p_full[w][buf], (jj >> 1) & 1);
          if (w == 0) WTRACE(2, jj * 8 + 2);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < WS_BK / 16; ++kk) {  // A = P_jj in TMEM: 16 keys per 8 columns
            const uint64_t bd = make_sdesc(sb + SM::V + s * SM::V_BYTES + kk * 2 * (CV / 8) * 128, (CV / 8) * 128, 128);
            mma_bf16_ts(tmem + 256 + w * 128, tmem + (2 * w + buf) * WS_BK + kk * 8, bd, IDESC_O,
                        (jj > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&o_done[w][buf]);
          mma_commit(&kv_empty[s]);  // this warpgroup is done with K_jj (S_jj) and V_jj
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------------ softmax warpgroups
    const int w = warp >> 2;
    const int r = (warp & 3) * 32 + lane;
    const int qi = q0 + w * WS_BQ + r;
    const uint32_t t_lane = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const uint32_t t_o = t_lane + 256 + w * 128;
    const bf16* brow = nullptr;
    if (P.bias && !per_key_bias && qi < L) brow = P.bias + b * P.bs0 + (int64_t)h * P.bs1 + (int64_t)qi * P.bs2;
    const float sl2 = P.scale_log2;
    float m_run = -INFINITY;  // running max in scaled log2 units
    if (w == 1) named_bar_arrive(1, 256);  // warpgroup 0 takes the first turn

    for (int j = 0; j < nkt; ++j) {
      const int buf = j & 1;
      const int k0 = j * WS_BK;
      // full-bias row segment: issue the loads before waiting on the tensor core
      float bv[WS_BK];
      if (brow) {
        if (P.bias_vec && k0 + WS_BK <= L) {
#pragma unroll
          for (int kk = 0; kk < WS_BK; kk += 8) {
            const uint4 u = *reinterpret_cast<const uint4*>(brow + k0 + kk);
            unpack_bf16x2(u.x, bv[kk], bv[kk + 1]); unpack_bf16x2(u.y, bv[kk + 2], bv[kk + 3]);
            unpack_bf16x2(u.z, bv[kk + 4], bv[kk + 5]); unpack_bf16x2(u.w, bv[kk + 6], bv[kk + 7]);
          }
        } else {
#pragma unroll
          for (int kk = 0; kk < WS_BK; ++kk) bv[kk] = k0 + kk < L ? bf2f(brow[(int64_t)(k0 + kk) * P.bs3]) : 0.f;
        }
      }
      if ((threadIdx.x & 127) == 0) WTRACE(w, j * 8 + 0);
      mbar_wait(&s_full[w][buf], (j >> 1) & 1);
      if ((threadIdx.x & 127) == 0) WTRACE(w, j * 8 + 1);
      tc_fence_after();
      float sv[WS_BK];
      tmem_ld32(t_lane + (2 * w + buf) * WS_BK, sv);
      tmem_ld32(t_lane + (2 * w + buf) * WS_BK + 32, sv + 32);
      tmem_ld_wait();
      if ((threadIdx.x & 127) == 0) WTRACE(w, j * 8 + 2);

      if (brow) {
#pragma unroll
        for (int kk = 0; kk < WS_BK; ++kk) sv[kk] += bv[kk];
      }
      if (k0 + WS_BK > L) {
#pragma unroll
        for (int kk = 0; kk < WS_BK; ++kk)
          if (k0 + kk >= L) sv[kk] = -INFINITY;
      }
      // row max as a tree (8 independent chains): a serial chain of dependent max ops is
      // latency-bound with only two softmax warps per scheduler
      // (three-input max: 36 FMNMX3 for 64 keys)
      float m8[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) m8[e] = fmax3f(sv[e], sv[e + 8], sv[e + 16]);
#pragma unroll
      for (int kk = 24; kk + 16 <= WS_BK; kk += 16) {
#pragma unroll
        for (int e = 0; e < 8; ++e) m8[e] = fmax3f(m8[e], sv[kk + e], sv[kk + 8 + e]);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) m8[e] = fmaxf(m8[e], sv[WS_BK - 8 + e]);
      const float mx = fmax3f(fmax3f(m8[0], m8[1], m8[2]), fmax3f(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
      const float mxs = mx * sl2;
      // lazy rescale: a row whose max grew by more than 2^8 rescales its O row (and its row
      // sum, column CP) - warp-uniform because TMEM loads/stores are warp-collective
      const bool grow = mxs > m_run + WS_RESCALE;
      if (__any_sync(0xffffffffu, grow)) {
        const float m_new = grow ? mxs : m_run;
        if (j > 0) {
          // every PV up to j-1 must have landed in O: PV_{j-1} is completion #((j-1)/2) of
          // o_done[w][(j-1)&1]; the next one on that barrier needs P_{j+1} (not yet written)
          mbar_wait(&o_done[w][(j - 1) & 1], ((j - 1) >> 1) & 1);
          tc_fence_after();
          ws_scale_o<CV>(t_o, ex2f(m_run - m_new));
          tc_fence_before();
        }
        m_run = m_new;
      }
      if ((threadIdx.x & 127) == 0) WTRACE(w, j * 8 + 3);
      // ping-pong: the two warpgroups take turns on the exp phase (the MUFU pipe), so one
      // warpgroup's TMEM round trips and row max run under the other's exponentials
      named_bar_sync(1 + w, 256);
      if ((threadIdx.x & 127) == 0) WTRACE(w, j * 8 + 6);
      const float mref = m_run == -INFINITY ? 0.f : m_run;
      // P_j (bf16, 2 keys per 32-bit column) overwrites S_j in TMEM columns [0, 32) of the
      // buffer: this thread's row was read above, and S_{j+2} will not be issued into the
      // buffer before PV_j (which reads P_j) completes
      uint32_t pk[WS_BK / 2];
#pragma unroll
      for (int kk = 0; kk < WS_BK; kk += 2)
      {
        const float2 y = __ffma2_rn(make_float2(sv[kk], sv[kk + 1]), make_float2(sl2, sl2), make_float2(-mref, -mref));
        pk[kk / 2] = pack_bf16x2(ex2f(y.x), ex2f(y.y));
      }
      if ((threadIdx.x & 127) == 0) WTRACE(w, j * 8 + 4);
      ws_tmem_st32(t_lane + (2 * w + buf) * WS_BK, pk);
      if (w == 0 || j + 1 < nkt) named_bar_arrive(2 - w, 256);  // hand the turn over
      tmem_st_wait();
      tc_fence_before();
      ws_arrive(&p_full[w][buf]);
      if ((threadIdx.x & 127) == 0) WTRACE(w, j * 8 + 5);
    }
    // epilogue: the last PV (j = nkt-1) is completion #((nkt-1)/2) of o_done[w][(nkt-1)&1]
    mbar_wait(&o_done[w][(nkt - 1) & 1], ((nkt - 1) >> 1) & 1);
    tc_fence_after();
    float ov[CV];
#pragma unroll
    for (int cc = 0; cc < CV; cc += 8) ws_tmem_ld8(t_o + cc, ov + cc);
    tmem_ld_wait();
    const float l_run = ov[CP];
    if (qi < L) {
      const float inv = rcpf(l_run);
      const bf16* gp = P.g + b * P.g_sb + (int64_t)qi * P.g_sl + (int64_t)h * c;
      bf16* og = P.og + b * P.o_sb + (int64_t)qi * P.o_sl + (int64_t)h * c;
      bf16* orw = P.orw ? P.orw + b * P.r_sb + (int64_t)qi * P.r_sl + (int64_t)h * c : nullptr;
#pragma unroll
      for (int d = 0; d < CP; d += 8) {
        if (d < c) {
          float o[8], gv[8];
          const uint4 u = *reinterpret_cast<const uint4*>(gp + d);
          unpack_bf16x2(u.x, gv[0], gv[1]); unpack_bf16x2(u.y, gv[2], gv[3]);
          unpack_bf16x2(u.z, gv[4], gv[5]); unpack_bf16x2(u.w, gv[6], gv[7]);
#pragma unroll
          for (int e = 0; e < 8; ++e) o[e] = ov[d + e] * inv;
          if (orw) {
            uint4 wv;
            wv.x = pack_bf16x2(o[0], o[1]); wv.y = pack_bf16x2(o[2], o[3]);
            wv.z = pack_bf16x2(o[4], o[5]); wv.w = pack_bf16x2(o[6], o[7]);
            *reinterpret_cast<uint4*>(orw + d) = wv;
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) o[e] *= sigmoidf_(gv[e]);
          uint4 wv;
          wv.x = pack_bf16x2(o[0], o[1]); wv.y = pack_bf16x2(o[2], o[3]);
          wv.z = pack_bf16x2(o[4], o[5]); wv.w = pack_bf16x2(o[6], o[7]);
          *reinterpret_cast<uint4*>(og + d) = wv;
        }
      }
      if (P.lse) P.lse[(b * P.H + h) * (int64_t)L + qi] = (m_run + log2f(l_run)) * 0.6931471805599453f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc(tmem, 512);
}

// used by evo_gated_attention_fwd (attention.cu) for long sequences
template <int CP>
int launch_attn_fwd_ws(const AttnParams& p, int64_t B, cudaStream_t st) {
  using SM = WsSmem<CP>;
  static size_t attr_bytes = 0;
  const size_t smem = SM::TOTAL;
  if (smem > (size_t)attr_bytes) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_ws_kernel<CP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "attn fwd ws attr");
    attr_bytes = smem;
  }
  dim3 grid((unsigned)((p.L + 2 * WS_BQ - 1) / (2 * WS_BQ)), (unsigned)p.H, (unsigned)B);
  ::evo::pdl_launch(attn_fwd_ws_kernel<CP>, grid, WS_THREADS, smem, st, p);
  EVO_LAUNCH_CHECK("attention fwd (warp-specialised)");
  return EVO_OK;
}
#if EVO_EXP == 12
extern "C" int evo_ws_trace(void* dst) { return (int)cudaMemcpyFromSymbol(dst, g_ws_trace, sizeof(g_ws_trace)); }
#endif
template int launch_attn_fwd_ws<16>(const AttnParams&, int64_t, cudaStream_t);
template int launch_attn_fwd_ws<32>(const AttnParams&, int64_t, cudaStream_t);
template int launch_attn_fwd_ws<64>(const AttnParams&, int64_t, cudaStream_t);

}  // namespace evo
