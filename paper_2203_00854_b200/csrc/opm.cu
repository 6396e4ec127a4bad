// Fused OuterProductMean forward (evoformer.py:243-255):
//
//   y[i,j,c] = sum_{p,q} o[i,j,p,q] W_o[p*P+q, c],   o[i,j,p,q] = alpha * sum_s a[s,i,p] b[s,j,q]
//
// as two back-to-back tcgen05 GEMMs per tile, so o ([I, J, P, P]: 134 MB at N_r = 256, 34 GB at
// N_r = 4096) never goes to HBM unless the caller asks for it (training saves it for the backward).
//
// Tile = 32 i x 8 j = 256 (i, j) pairs, two sub-tiles s = 0, 1 of 4 j each that share every a and
// W_o load (half the L2 -> SM bytes per pair of a 128-pair tile; the kernel is bound by that
// stream).  The P = 32 outer-product channels are walked in 8 chunks of 4 p:
//   GEMM1_s  acc1_s[(p_l, i_l)][(j_l, q)] = sum_s aT[p][s][i] b[s][j][q]   M = 4p x 32i, N = 4j x 32q, K = N_s
//          (a is stored transposed, [p][s][i], so i is the MN-contiguous dim of the A operand and a
//          TMEM lane holds one (p, i) row: lanes of a warp are 32 different i)
//   convert_s  TMEM -> registers -> alpha, bf16 -> shared memory as the A operand of GEMM2, rows =
//          pairs (j_l*32 + i_l), K = (p_l, q), 128-byte swizzle (the 8 lanes of a quarter-warp hit
//          8 different rows -> 8 different 16-byte bank groups: conflict-free)
//   GEMM2_s  y_s[(j_l, i_l)][c] += o_chunk_s . W_o[chunk rows][c]           M = 128 pairs, N = Hz, K = 4p x 32q
// TMEM: acc1_0, acc1_1 (128 columns each), y_0, y_1 (Hz each).  The MMA issue order
// G1_0(c) G1_1(c) | G2_0(c) G1_0(c+1) | G2_1(c) G1_1(c+1) | ... keeps the tensor pipe busy while
// the two converter groups drain the other sub-tile's accumulator.  a and W_o chunks stream
// through 64-row (16 KB) TMA granule rings; b is loaded per sub-tile and released as soon as that
// sub-tile's last GEMM1 has read it.
//
// Warp roles (512 threads, 1 CTA per SM, persistent over tiles):
//   warp 0      TMA producer (a granules, b sub-tiles, W_o granules)
//   warp 1      MMA issuer
//   warp 2      TMEM allocator
//   warps 4-7   converter of sub-tile 0, warps 8-11 of sub-tile 1 (lane quarter = warp % 4);
//               optional TMA store of the o chunk (training keeps o for the backward)
//   warps 12-15 y epilogue (TMEM -> bf16 rows of y)
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tma.cuh"

namespace evo {

int sm_count();

namespace {

constexpr int OPM_THREADS = 512;
constexpr int OPM_SMAX = 128;                   // sequences held per tile (K of GEMM1)
#ifndef EVO_EXP
#define EVO_EXP 0
#endif
constexpr int NA = EVO_EXP == 1 ? 3 : EVO_EXP == 2 ? 2 : 4;  // a granule ring: [128 rows (p_l, i_l)][64 s] = 16 KB
constexpr int NW = EVO_EXP == 1 ? 3 : EVO_EXP == 2 ? 4 : 2;  // W_o granule ring: [Hz/64 atoms][64 k][64 c] (16 KB)
constexpr uint32_t AG_BYTES = 128 * 64 * 2;
constexpr uint32_t B1_BYTES = 2 * 128 * 64 * 2;  // one sub-tile's b: <= 2 granules of [128 rows (j_l, q)][64 s]
constexpr uint32_t A2_BYTES = 128 * 128 * 2;      // 128 pairs x 128 k (two 64-k swizzle columns)

#if EVO_EXP == 3
__device__ unsigned long long g_opm_trace[4096];
__device__ __forceinline__ void trace(int idx) {
  if (blockIdx.x == 0 && idx < 4096) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_opm_trace[idx] = t;
  }
}
#define TRACE(i) trace(i)
#else
#define TRACE(i) (void)0
#endif
#if EVO_EXP == 4
__device__ long long g_opmb_trace[4096];
#define BTR(i)                                                          \
  do {                                                                  \
    if (blockIdx.x == 0 && (i) < 4096) g_opmb_trace[(i)] = clock64();   \
  } while (0)
#else
#define BTR(i) (void)0
#endif

struct OpmArgs {
  int I, J, S;
  int tiles_i, tiles;
  float alpha;
  bf16* y;
  int64_t y_ld;
  int save_o;
  int dbg;  // experiment switches (EVO_OPM_DBG): 1 no convert, 2 no GEMM2, 4 no GEMM1
};

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;  // 2 = SWIZZLE_128B, 4 = SWIZZLE_64B
  return d;
}

struct Ring {  // producer/consumer position in an mbarrier ring of n slots
  int slot = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void next(int n) {
    if (++slot == n) {
      slot = 0;
      phase ^= 1;
    }
  }
};

template <int HZ>
__global__ void __launch_bounds__(OPM_THREADS, 1)
    opm_fused_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmO, OpmArgs g) {
  pdl_wait();
  constexpr uint32_t WG_BYTES = HZ * 64 * 2;  // W_o granule: 64 k rows x HZ c
  constexpr uint32_t W_ATOM = HZ >= 64 ? 8192 : 4096;  // one 64-c (32-c) swizzle column of a granule
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t a_full[NA], a_empty[NA], w_full[NW], w_empty[NW], b_full[2], b_empty[2], acc_full[2],
      acc_empty[2], o_full[2], o_empty[2], y_full[2], y_empty[2];
  __shared__ uint32_t tmem_sh;

  const uint32_t sbase = smem_u32(smem);
  const uint32_t sA1 = sbase, sB1 = sA1 + NA * AG_BYTES, sA2 = sB1 + 2 * B1_BYTES, sB2 = sA2 + 2 * A2_BYTES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = g.S;
  const int NG = (S + 63) / 64;  // 64-sequence granules per chunk (the TMA zero-fills s >= S)
  constexpr int NCH = 8;           // P = 32 in chunks of 4

  if (threadIdx.x == 0) {
    for (int i = 0; i < NA; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 2);
    }
    for (int i = 0; i < NW; ++i) {
      mbar_init(&w_full[i], 1);
      mbar_init(&w_empty[i], 2);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 128);
      mbar_init(&o_full[i], 128);
      mbar_init(&o_empty[i], 1);
      mbar_init(&y_full[i], 1);
      mbar_init(&y_empty[i], 128);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(&tmem_sh, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;  // acc1_s at columns s*128, y_s at 256 + s*HZ

  if (warp == 0 || warp == 2) {
    // ------------------------------------------------------------ TMA producers: warp 0 a + b, warp 2 W_o
    // (separate threads, so a stalled W_o ring never holds back the next chunk's a granules)
    if (lane == 0) {
      const uint64_t ma = reinterpret_cast<uint64_t>(&tmA), mb = reinterpret_cast<uint64_t>(&tmB),
                     mw = reinterpret_cast<uint64_t>(&tmW);
      Ring r;
      int it = 0;
      for (int t = blockIdx.x; t < g.tiles; t += gridDim.x, ++it) {
        const int i0 = (t % g.tiles_i) * 32, j0 = (t / g.tiles_i) * 8;
        for (int c = 0; c < NCH; ++c) {
          if (warp == 0) {
            for (int kg = 0; kg < NG; ++kg) {
              mbar_wait(&a_empty[r.slot], r.phase ^ 1);
              TRACE((it * NCH + c) * 16 + kg);
              mbar_expect_tx(&a_full[r.slot], AG_BYTES);
              tma_ld3(sA1 + r.slot * AG_BYTES, ma, kg * 64, i0, c * 4, smem_u32(&a_full[r.slot]));
              r.next(NA);
            }
            if (c == 0) {  // this tile's b, per sub-tile (released by that sub-tile's last GEMM1)
              for (int s = 0; s < 2; ++s) {
                mbar_wait(&b_empty[s], (it & 1) ^ 1);
                mbar_expect_tx(&b_full[s], (uint32_t)NG * AG_BYTES);
                for (int kg = 0; kg < NG; ++kg)
                  tma_ld3(sB1 + s * B1_BYTES + kg * AG_BYTES, mb, kg * 64, 0, j0 + 4 * s, smem_u32(&b_full[s]));
              }
            }
          } else {
            for (int wg = 0; wg < 2; ++wg) {
              mbar_wait(&w_empty[r.slot], r.phase ^ 1);
              TRACE((it * NCH + c) * 16 + 2 + wg);
              mbar_expect_tx(&w_full[r.slot], WG_BYTES);
              tma_ld3(sB2 + r.slot * WG_BYTES, mw, 0, c * 128 + wg * 64, 0, smem_u32(&w_full[r.slot]));
              r.next(NW);
            }
          }
        }
      }
    }
  } else if (warp == 1 || warp == 3) {
    // ------------------------------------------------------------ MMA issuers: warp 1 -> sub-tile 0, warp 3 -> 1
    // (one issuing thread per sub-tile halves the barrier traffic each thread waits on; the shared a / W_o
    // granules are released by both: their empty barriers count 2 commits)
    const int s = warp >> 1;
    constexpr uint32_t IDESC1 = make_idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t IDESC2 = make_idesc_bf16(128, HZ, 0, 1);
    Ring ra, rw;  // consumer positions in the a / W_o rings
    uint32_t acc_ph = 0, o_ph = 0, y_ph = 0;
    const uint32_t acc = tmem + s * 128, yacc = tmem + 256 + s * HZ, b1s = sB1 + s * B1_BYTES;
    int it = 0;
    for (int t = blockIdx.x; t < g.tiles; t += gridDim.x, ++it) {
      mbar_wait(&b_full[s], it & 1);
      for (int c = 0; c <= NCH; ++c) {
        if (c < NCH) {  // GEMM1 of chunk c
          mbar_wait(&acc_empty[s], acc_ph ^ 1);
          acc_ph ^= 1;
          for (int kg = 0; kg < NG; ++kg) {
            mbar_wait(&a_full[ra.slot], ra.phase);
            tc_fence_after();
            if (lane == 0) {
              const uint32_t a1 = sA1 + ra.slot * AG_BYTES, b1 = b1s + kg * AG_BYTES;
              if (!(g.dbg & 4)) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  mma_bf16(acc, sdesc(a1 + kk * 32, 16, 1024, 2), sdesc(b1 + kk * 32, 16, 1024, 2), IDESC1,
                           (kg | kk) != 0);
              }
              mma_commit(&a_empty[ra.slot]);
            }
            __syncwarp();
            ra.next(NA);
          }
          if (lane == 0) {
            mma_commit(&acc_full[s]);
            if (c == NCH - 1) mma_commit(&b_empty[s]);
          }
          __syncwarp();
        }
        if (c > 0) {  // GEMM2 of chunk c-1 (its conversion overlapped GEMM1 of chunk c)
          const int cc = c - 1;
          if (cc == 0) {
            mbar_wait(&y_empty[s], y_ph ^ 1);
            y_ph ^= 1;
          }
          mbar_wait(&o_full[s], o_ph);
          o_ph ^= 1;
          for (int wg = 0; wg < 2; ++wg) {
            mbar_wait(&w_full[rw.slot], rw.phase);
            tc_fence_after();
            if (lane == 0) {
              const uint32_t a2 = sA2 + s * A2_BYTES + wg * 16384, b2 = sB2 + rw.slot * WG_BYTES;
              if (!(g.dbg & 2)) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                  const uint64_t ad = sdesc(a2 + kk * 32, 16, 1024, 2);
                  const uint64_t bd =
                      HZ >= 64 ? sdesc(b2 + kk * 2048, W_ATOM, 1024, 2) : sdesc(b2 + kk * 1024, W_ATOM, 512, 4);
                  mma_bf16(yacc, ad, bd, IDESC2, (cc | wg | kk) != 0);
                }
              }
              mma_commit(&w_empty[rw.slot]);
            }
            __syncwarp();
            rw.next(NW);
          }
          if (lane == 0) {
            mma_commit(&o_empty[s]);
            if (cc == NCH - 1) mma_commit(&y_full[s]);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ------------------------------------------------------------ converters: acc1_s -> o chunk (bf16, swizzled)
    const int s = (warp - 4) >> 2;
    const int q = warp & 3;  // TMEM lane quarter = p_l of this warp's rows; lane = i_l
    const int et = threadIdx.x - 128 - 128 * s;
    uint32_t ph = 0;
    int tcount = 0;
    for (int t = blockIdx.x; t < g.tiles; t += gridDim.x, ++tcount) {
      const int i0 = (t % g.tiles_i) * 32, j0 = (t / g.tiles_i) * 8 + 4 * s;
      for (int c = 0; c < NCH; ++c, ph ^= 1) {
        mbar_wait(&acc_full[s], ph);
        tc_fence_after();
        const int tb = (tcount * NCH + c) * 16;
        if (et == 0) TRACE(tb + 9 + 2 * s);
        if (g.save_o) {  // the TMA store of the previous chunk must have read the buffer
          if (et == 0) bulk_wait_read<0>();
          named_sync(1 + s, 128);
        }
        mbar_wait(&o_empty[s], ph ^ 1);
        const uint32_t a2 = sA2 + s * A2_BYTES + (q >> 1) * 16384;
        if (!(g.dbg & 1)) {
#pragma unroll
          for (int jp = 0; jp < 4; jp += 2) {  // two 32-column TMEM loads in flight per wait
            float v[64];
            tmem_ld32(tmem + s * 128 + ((uint32_t)(q * 32) << 16) + jp * 32, v);
            tmem_ld32(tmem + s * 128 + ((uint32_t)(q * 32) << 16) + jp * 32 + 32, v + 32);
            tmem_ld_wait();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int m2 = (jp + h) * 32 + lane;
              const uint32_t row = a2 + m2 * 128;
#pragma unroll
              for (int t4 = 0; t4 < 4; ++t4) {
                const int ch = ((q & 1) * 4 + t4) ^ (m2 & 7);
                const float* w = v + h * 32 + t4 * 8;
                st_shared_v4(row + ch * 16, pack_bf16x2(g.alpha * w[0], g.alpha * w[1]),
                             pack_bf16x2(g.alpha * w[2], g.alpha * w[3]), pack_bf16x2(g.alpha * w[4], g.alpha * w[5]),
                             pack_bf16x2(g.alpha * w[6], g.alpha * w[7]));
              }
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&acc_empty[s]);
        fence_async_smem();
        mbar_arrive(&o_full[s]);
        if (et == 0) TRACE(tb + 10 + 2 * s);
        if (g.save_o) {
          named_sync(1 + s, 128);
          if (et == 0) {
            const uint64_t mo = reinterpret_cast<uint64_t>(&tmO);
            tma_st3(mo, sA2 + s * A2_BYTES, c * 128, i0, j0);
            tma_st3(mo, sA2 + s * A2_BYTES + 16384, c * 128 + 64, i0, j0);
            bulk_commit();
          }
        }
      }
    }
    if (g.save_o && et == 0) bulk_wait<0>();
  } else if (warp >= 12) {
    // ------------------------------------------------------------ y epilogue: TMEM -> bf16 rows
    const int q = warp & 3;  // lane quarter = j_l within the sub-tile; lane = i_l
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < g.tiles; t += gridDim.x, ph ^= 1) {
      const int i0 = (t % g.tiles_i) * 32, j0 = (t / g.tiles_i) * 8;
      for (int s = 0; s < 2; ++s) {
        mbar_wait(&y_full[s], ph);
        tc_fence_after();
        bf16* yrow = g.y + ((int64_t)(i0 + lane) * g.J + (j0 + 4 * s + q)) * g.y_ld;
#pragma unroll
        for (int c0 = 0; c0 < HZ; c0 += 32) {
          float v[32];
          tmem_ld32(tmem + 256 + s * HZ + ((uint32_t)(q * 32) << 16) + c0, v);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; e += 8)
            *reinterpret_cast<uint4*>(yrow + c0 + e) =
                make_uint4(pack_bf16x2(v[e], v[e + 1]), pack_bf16x2(v[e + 2], v[e + 3]),
                           pack_bf16x2(v[e + 4], v[e + 5]), pack_bf16x2(v[e + 6], v[e + 7]));
        }
        tc_fence_before();
        mbar_arrive(&y_empty[s]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// x [S*R][ld] (rows (s, r)), channels col0 .. col0+P (and col0+P .. col0+2P when out_b) ->
// out[r][p][s]: one CTA per residue r; the [S][P] slab is staged in shared memory so the global
// reads are 16-byte row chunks and the writes 16-byte runs of 8 sequences.
__global__ void __launch_bounds__(256) opm_transpose_kernel(const bf16* __restrict__ x, int64_t ld, int64_t col0, int S,
                                                            int R, int P, bf16* __restrict__ out_a,
                                                            bf16* __restrict__ out_b) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t tsm[];
  bf16* t = reinterpret_cast<bf16*>(tsm);  // [S][CW + 8] (CW = P or 2P channels)
  const int r = blockIdx.x;
  const int CW = out_b ? 2 * P : P, pitch = CW + 8;
  const int cpr = CW / 8;  // 16-byte chunks per row
  for (int ch = threadIdx.x; ch < S * cpr; ch += blockDim.x) {
    const int sq = ch / cpr, c8 = (ch % cpr) * 8;
    const uint4 v = *reinterpret_cast<const uint4*>(x + ((int64_t)sq * R + r) * ld + col0 + c8);
    *reinterpret_cast<uint4*>(t + sq * pitch + c8) = v;
  }
  __syncthreads();
  const int sc_n = (S + 7) / 8;
  for (int ch = threadIdx.x; ch < sc_n * CW; ch += blockDim.x) {
    const int sc = ch / CW, p = ch % CW;  // consecutive threads: consecutive channels (no bank conflicts)
    bf16* dst = (p < P ? out_a : out_b) + ((int64_t)r * P + (p % P)) * S + sc * 8;
    if (sc * 8 + 8 <= S) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const bf16 lo = t[(sc * 8 + 2 * e) * pitch + p], hi = t[(sc * 8 + 2 * e + 1) * pitch + p];
        w[e] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
      }
      *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      for (int e = 0; sc * 8 + e < S; ++e) dst[e] = t[(sc * 8 + e) * pitch + p];
    }
  }
}


// ===================================================================================== backward
// Gradients of the OPM factors without materialising do[i,j,p,q] = sum_c dy[i,j,c] W_o[pq,c]:
//
//   da[s,i,p] = alpha sum_{j,q} b[s,j,q] do[i,j,p,q]        db[s,j,q] = alpha sum_{i,p} a[s,i,p] do[i,j,p,q]
//
// are the same contraction with the roles of (i, p, a) and (j, q, b) exchanged, so one kernel runs
// both (the caller swaps the tensor maps).  In da's terms: a unit = (32 x-rows [i], 4 p of a chunk,
// a range of y [j]); per step of 4 y (128 (y, x) pairs):
//   GEMM_A   D_A[(y_l, x_l)][(p_l, q)] = dy[(x, y)][c] . W[(p_l, q)][c]^T        M = 128 pairs, N = 128, K = Hz
//   convert  D_A -> bf16 shared memory, rows (p_l, x_l), K = (y_l, q) (128-byte swizzle, conflict-free)
//   GEMM_B   acc[(p_l, x_l)][s] += A_B . other[y][q][s]^T                        M = 128, N = N_s, K = 128
// acc stays in TMEM over the unit's y range and leaves as fp32 partials [split][x][p][s];
// opm_bwd_finish sums the splits in order, scales by alpha and writes the factor gradient in the
// projection's row layout (or the rank-major layout a DAP reduce-scatter takes).
constexpr int OB_THREADS = 384;
constexpr uint32_t OB_T = 128 * 64 * 2;  // one 128-row x 64-element swizzle column: 16 KB

struct OpmBwdArgs {
  int X, Y, S, units_x, units, nsplit, ysteps_per_split, hz_halves;
  float* part;  // [nsplit][X][P][128] fp32
};

__global__ void __launch_bounds__(OB_THREADS, 1)
    opm_bwd_contract_kernel(const __grid_constant__ CUtensorMap tmDY, const __grid_constant__ CUtensorMap tmW,
                            const __grid_constant__ CUtensorMap tmO, OpmBwdArgs g) {
  pdl_wait();
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t w_full, w_empty, dy_full[2], dy_empty[2], ot_full[2], ot_empty[2], da_full[2], da_empty[2],
      ab_full[2], ab_empty[2], acc_full, acc_empty;
  __shared__ uint32_t tmem_sh;
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sW = sbase, sDY = sW + 2 * OB_T, sOT = sDY + 4 * OB_T, sAB = sOT + 4 * OB_T;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int HH = g.hz_halves;  // Hz / 64: K of GEMM_A in 64-element swizzle columns

  if (threadIdx.x == 0) {
    mbar_init(&w_full, 1);
    mbar_init(&w_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&dy_full[i], 1);
      mbar_init(&dy_empty[i], 1);
      mbar_init(&ot_full[i], 1);
      mbar_init(&ot_empty[i], 1);
      mbar_init(&da_full[i], 1);
      mbar_init(&da_empty[i], 128);
      mbar_init(&ab_full[i], 128);
      mbar_init(&ab_empty[i], 1);
    }
    mbar_init(&acc_full, 1);
    mbar_init(&acc_empty, 128);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(&tmem_sh, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;  // D_A[b] at b*128, acc at 256

  auto decode = [&](int u, int& x0, int& p0, int& sp) {
    x0 = (u % g.units_x) * 32;
    const int r = u / g.units_x;
    p0 = (r % 8) * 4;
    sp = r / 8;
  };
  auto ysteps = [&](int sp) {
    const int y_total = g.Y / 4, lo = sp * g.ysteps_per_split;
    const int hi = lo + g.ysteps_per_split < y_total ? lo + g.ysteps_per_split : y_total;
    return hi > lo ? hi - lo : 0;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t mdy = reinterpret_cast<uint64_t>(&tmDY), mw = reinterpret_cast<uint64_t>(&tmW),
                     mo = reinterpret_cast<uint64_t>(&tmO);
      int st = 0, it = 0;
      for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
        int x0, p0, sp;
        decode(u, x0, p0, sp);
        const int n = ysteps(sp), y0 = sp * g.ysteps_per_split * 4;
        mbar_wait(&w_empty, (it & 1) ^ 1);
        mbar_expect_tx(&w_full, HH * OB_T);
        for (int hh = 0; hh < HH; ++hh) tma_ld3(sW + hh * OB_T, mw, hh * 64, 0, p0, smem_u32(&w_full));
        for (int t = 0; t < n; ++t, ++st) {
          const int b = st & 1;
          const uint32_t ph = ((st >> 1) & 1) ^ 1;
          const int yb = y0 + t * 4;
          mbar_wait(&dy_empty[b], ph);
          mbar_expect_tx(&dy_full[b], HH * OB_T);
          for (int hh = 0; hh < HH; ++hh)
            tma_ld3(sDY + (2 * b + hh) * OB_T, mdy, hh * 64, x0, yb, smem_u32(&dy_full[b]));
          mbar_wait(&ot_empty[b], ph);
          mbar_expect_tx(&ot_full[b], 2 * OB_T);
          for (int sh = 0; sh < 2; ++sh)
            tma_ld3(sOT + (2 * b + sh) * OB_T, mo, sh * 64, 0, yb, smem_u32(&ot_full[b]));
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t IDA = make_idesc_bf16(128, 128, 0, 0);  // dy (K-major) x W (K-major)
    constexpr uint32_t IDB = make_idesc_bf16(128, 128, 0, 1);  // A_B (K-major) x other (MN-major over s)
    int st = 0, it = 0;
    for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
      int x0, p0, sp;
      decode(u, x0, p0, sp);
      const int n = ysteps(sp);
      mbar_wait(&w_full, it & 1);
      for (int t = 0; t <= n; ++t) {
        if (t < n) {  // GEMM_A of step t
          const int s_ = st + t, b = s_ & 1;
          if (lane == 0) BTR(s_ * 8 + 0);
          mbar_wait(&dy_full[b], (s_ >> 1) & 1);
          if (lane == 0) BTR(s_ * 8 + 1);
          mbar_wait(&da_empty[b], ((s_ >> 1) & 1) ^ 1);
          if (lane == 0) BTR(s_ * 8 + 2);
          tc_fence_after();
          if (lane == 0) {
            for (int kk = 0; kk < 4 * HH; ++kk) {
              const uint32_t off = (kk >> 2) * OB_T + (kk & 3) * 32;
              mma_bf16(tmem + b * 128, sdesc(sDY + 2 * b * OB_T + off, 16, 1024, 2), sdesc(sW + off, 16, 1024, 2),
                       IDA, kk != 0);
            }
            mma_commit(&dy_empty[b]);
            mma_commit(&da_full[b]);
            if (t == n - 1) mma_commit(&w_empty);
          }
          __syncwarp();
        }
        if (t > 0) {  // GEMM_B of step t-1 (its conversion overlapped GEMM_A of step t)
          const int s_ = st + t - 1, b = s_ & 1;
          if (lane == 0) BTR(s_ * 8 + 3);
          if (t == 1) mbar_wait(&acc_empty, (it & 1) ^ 1);
          mbar_wait(&ab_full[b], (s_ >> 1) & 1);
          if (lane == 0) BTR(s_ * 8 + 4);
          mbar_wait(&ot_full[b], (s_ >> 1) & 1);
          if (lane == 0) BTR(s_ * 8 + 5);
          tc_fence_after();
          if (lane == 0) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint64_t ad = sdesc(sAB + (2 * b + (kk >> 2)) * OB_T + (kk & 3) * 32, 16, 1024, 2);
              const uint64_t bd = sdesc(sOT + 2 * b * OB_T + kk * 2048, OB_T, 1024, 2);
              mma_bf16(tmem + 256, ad, bd, IDB, (t > 1 || kk > 0) ? 1u : 0u);
            }
            mma_commit(&ab_empty[b]);
            mma_commit(&ot_empty[b]);
            if (t == n) mma_commit(&acc_full);
          }
          __syncwarp();
        }
      }
      if (n == 0 && lane == 0) mma_commit(&w_empty);
      st += n;
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ converter: D_A -> A_B
    const int yq = warp & 3;  // lane quarter = y_l of the pairs; lane = x_l
    int st = 0;
    for (int u = blockIdx.x; u < g.units; u += gridDim.x) {
      int x0, p0, sp;
      decode(u, x0, p0, sp);
      const int n = ysteps(sp);
      for (int t = 0; t < n; ++t, ++st) {
        const int b = st & 1;
        const uint32_t ph = (st >> 1) & 1;
        mbar_wait(&da_full[b], ph);
        tc_fence_after();
        mbar_wait(&ab_empty[b], ph ^ 1);
        if (threadIdx.x == 128) BTR(st * 8 + 6);
        const uint32_t ab = sAB + (2 * b + (yq >> 1)) * OB_T;
#pragma unroll
        for (int pp = 0; pp < 4; pp += 2) {
          float v[64];
          tmem_ld32(tmem + b * 128 + ((uint32_t)(yq * 32) << 16) + pp * 32, v);
          tmem_ld32(tmem + b * 128 + ((uint32_t)(yq * 32) << 16) + pp * 32 + 32, v + 32);
          tmem_ld_wait();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = (pp + h) * 32 + lane;  // row (p_l, x_l)
            const uint32_t row = ab + r * 128;
#pragma unroll
            for (int t4 = 0; t4 < 4; ++t4) {
              const int ch = ((yq & 1) * 4 + t4) ^ (r & 7);
              const float* w = v + h * 32 + t4 * 8;
              st_shared_v4(row + ch * 16, pack_bf16x2(w[0], w[1]), pack_bf16x2(w[2], w[3]), pack_bf16x2(w[4], w[5]),
                           pack_bf16x2(w[6], w[7]));
            }
          }
        }
        tc_fence_before();
        if (threadIdx.x == 128) BTR(st * 8 + 7);
        mbar_arrive(&da_empty[b]);
        fence_async_smem();
        mbar_arrive(&ab_full[b]);
      }
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------------ epilogue: acc -> fp32 partials
    const int pq = warp & 3;  // lane quarter = p_l; lane = x_l
    int it = 0;
    for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
      int x0, p0, sp;
      decode(u, x0, p0, sp);
      const int n = ysteps(sp);
      float* dst = g.part + (((int64_t)sp * g.X + x0 + lane) * 32 + p0 + pq) * 128;
      if (n == 0) {  // an empty y range contributes zeros
        for (int c0 = 0; c0 < 128; c0 += 4) *reinterpret_cast<float4*>(dst + c0) = make_float4(0.f, 0.f, 0.f, 0.f);
        continue;
      }
      mbar_wait(&acc_full, it & 1);
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 32) {
        float v[32];
        tmem_ld32(tmem + 256 + ((uint32_t)(pq * 32) << 16) + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; e += 4)
          *reinterpret_cast<float4*>(dst + c0 + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
      }
      tc_fence_before();
      mbar_arrive(&acc_empty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// out(s, x, p) = alpha * sum_split part[split][x][p][s]  for s < S: one CTA per x, the [P][S] slab
// transposed through shared memory; out element (s, x, p) at
//   out + s*o_ss + (x / x_split)*o_sr + (x % x_split)*o_sx + p   (bf16 or fp32)
template <typename TO>
__global__ void __launch_bounds__(256) opm_bwd_finish(const float* __restrict__ part, int nsplit, int X, int S,
                                                      float alpha, TO* __restrict__ out, int64_t o_ss, int64_t o_sr,
                                                      int64_t o_sx, int x_split) {
  pdl_wait();
  __shared__ float t[32][129];
  const int x = blockIdx.x;
  // the [32 p][128 s] slab: 4 float4 per thread and split, every load of a thread in flight
  float4 acc[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k < nsplit) {
      const float4* src = reinterpret_cast<const float4*>(part + ((int64_t)k * X + x) * 32 * 128);
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(src + threadIdx.x + u * 256);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc[u].x += v[u].x; acc[u].y += v[u].y; acc[u].z += v[u].z; acc[u].w += v[u].w;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = (threadIdx.x + u * 256) * 4, p = i >> 7, sq = i & 127;
    t[p][sq] = alpha * acc[u].x;
    t[p][sq + 1] = alpha * acc[u].y;
    t[p][sq + 2] = alpha * acc[u].z;
    t[p][sq + 3] = alpha * acc[u].w;
  }
  __syncthreads();
  TO* base = out + (int64_t)(x / x_split) * o_sr + (int64_t)(x % x_split) * o_sx;
  for (int i = threadIdx.x; i < S * 32; i += 256) {  // lanes = consecutive p: coalesced rows
    const int sq = i >> 5, p = i & 31;
    stf<TO>(base + (int64_t)sq * o_ss + p, t[p][sq]);
  }
}

bool encode(CUtensorMap* map, const void* ptr, int nd, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
            const cuuint32_t* box, CUtensorMapSwizzle sw) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return false;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, (cuuint32_t)nd, const_cast<void*>(ptr), dims, strides_bytes, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int HZ>
int launch(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tw, const CUtensorMap& to, const OpmArgs& a,
           cudaStream_t st) {
  constexpr size_t smem = NA * AG_BYTES + 2 * B1_BYTES + 2 * A2_BYTES + NW * (size_t)HZ * 64 * 2;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(opm_fused_kernel<HZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "opm_fused attr");
    attr = true;
  }
  const int grid = a.tiles < sm_count() ? a.tiles : sm_count();
  ::evo::pdl_launch(opm_fused_kernel<HZ>, grid, OPM_THREADS, smem, st, ta, tb, tw, to, a);
  EVO_LAUNCH_CHECK("opm_fused launch");
  return EVO_OK;
}

}  // namespace
}  // namespace evo

#if EVO_EXP == 4
extern "C" int evo_opmb_trace(void* dst) { return (int)cudaMemcpyFromSymbol(dst, evo::g_opmb_trace, sizeof(evo::g_opmb_trace)); }
#endif
#if EVO_EXP == 3
extern "C" int evo_opm_trace(void* dst) { return (int)cudaMemcpyFromSymbol(dst, evo::g_opm_trace, sizeof(evo::g_opm_trace)); }
#endif

extern "C" int evo_opm_fused_supported(int64_t I, int64_t J, int64_t S, int64_t P, int64_t Hz) {
  return P == 32 && S >= 8 && S <= evo::OPM_SMAX && S % 8 == 0 && I >= 32 && I % 32 == 0 && J >= 8 && J % 8 == 0 &&
         (Hz == 32 || Hz == 64 || Hz == 128);
}

extern "C" int evo_opm_fused_fwd(const void* a_t, const void* b_t, const void* w_o, void* y, int64_t y_ld, void* o_save,
                                 int64_t I, int64_t J, int64_t S, int64_t P, int64_t Hz, float alpha, void* stream) {
  using namespace evo;
  EVO_CHECK_ARG(a_t && b_t && w_o && y, EVO_ERR_ARG, "opm_fused_fwd: null operand");
  EVO_CHECK_ARG(evo_opm_fused_supported(I, J, S, P, Hz), EVO_ERR_SHAPE,
                "opm_fused_fwd: unsupported extents I=%lld J=%lld S=%lld P=%lld Hz=%lld (needs P=32, S%%8==0 and "
                "S<=128, I%%32==0, J%%8==0, Hz in {32,64,128})",
                (long long)I, (long long)J, (long long)S, (long long)P, (long long)Hz);
  EVO_CHECK_ARG((((uintptr_t)a_t | (uintptr_t)b_t | (uintptr_t)w_o | (uintptr_t)o_save | (uintptr_t)y) & 15) == 0 &&
                    y_ld % 8 == 0,
                EVO_ERR_ALIGN, "opm_fused_fwd: operands must be 16-byte aligned");
  CUtensorMap ta, tb, tw, to;
  memset(&to, 0, sizeof(to));
  {  // a [i][p][s]: box [64 s][32 i][4 p] -> rows (p_l, i_l), 128-byte swizzle (s >= S zero-filled)
    cuuint64_t d[3] = {(cuuint64_t)S, (cuuint64_t)I, (cuuint64_t)P};
    cuuint64_t st[2] = {(cuuint64_t)(P * S * 2), (cuuint64_t)(S * 2)};
    cuuint32_t bx[3] = {64, 32, 4};
    EVO_CHECK_ARG(encode(&ta, a_t, 3, d, st, bx, CU_TENSOR_MAP_SWIZZLE_128B), EVO_ERR_ARG, "opm_fused_fwd: a map");
  }
  {  // b [j][q][s]: box [64 s][32 q][4 j] -> rows (j_l, q)
    cuuint64_t d[3] = {(cuuint64_t)S, (cuuint64_t)P, (cuuint64_t)J};
    cuuint64_t st[2] = {(cuuint64_t)(S * 2), (cuuint64_t)(P * S * 2)};
    cuuint32_t bx[3] = {64, 32, 4};
    EVO_CHECK_ARG(encode(&tb, b_t, 3, d, st, bx, CU_TENSOR_MAP_SWIZZLE_128B), EVO_ERR_ARG, "opm_fused_fwd: b map");
  }
  {  // W_o [P*P][Hz]: [c_lo 64][k 64][c_hi] granules, 128-byte swizzle (Hz = 32: 64-byte rows)
    if (Hz >= 64) {
      cuuint64_t d[3] = {64, (cuuint64_t)(P * P), (cuuint64_t)(Hz / 64)};
      cuuint64_t st[2] = {(cuuint64_t)Hz * 2, 128};
      cuuint32_t bx[3] = {64, 64, (cuuint32_t)(Hz / 64)};
      EVO_CHECK_ARG(encode(&tw, w_o, 3, d, st, bx, CU_TENSOR_MAP_SWIZZLE_128B), EVO_ERR_ARG, "opm_fused_fwd: W map");
    } else {
      cuuint64_t d[3] = {32, (cuuint64_t)(P * P), 1};
      cuuint64_t st[2] = {64, (cuuint64_t)(P * P) * 64};
      cuuint32_t bx[3] = {32, 64, 1};
      EVO_CHECK_ARG(encode(&tw, w_o, 3, d, st, bx, CU_TENSOR_MAP_SWIZZLE_64B), EVO_ERR_ARG, "opm_fused_fwd: W map");
    }
  }
  if (o_save) {  // o [i][j][P*P]: box [64 k][32 i][4 j] (rows j_l*32 + i_l), 128-byte swizzle
    cuuint64_t d[3] = {(cuuint64_t)(P * P), (cuuint64_t)I, (cuuint64_t)J};
    cuuint64_t st[2] = {(cuuint64_t)J * P * P * 2, (cuuint64_t)P * P * 2};
    cuuint32_t bx[3] = {64, 32, 4};
    EVO_CHECK_ARG(encode(&to, o_save, 3, d, st, bx, CU_TENSOR_MAP_SWIZZLE_128B), EVO_ERR_ARG, "opm_fused_fwd: o map");
  }
  OpmArgs a;
  a.I = (int)I;
  a.J = (int)J;
  a.S = (int)S;
  a.tiles_i = (int)(I / 32);
  a.tiles = (int)((I / 32) * (J / 8));
  a.alpha = alpha;
  a.y = static_cast<bf16*>(y);
  a.y_ld = y_ld;
  a.save_o = o_save != nullptr;
  { static const int dbg = [] { const char* e = getenv("EVO_OPM_DBG"); return e ? atoi(e) : 0; }(); a.dbg = dbg; }
  cudaStream_t st = (cudaStream_t)stream;
  if (Hz == 128) return launch<128>(ta, tb, tw, to, a, st);
  if (Hz == 64) return launch<64>(ta, tb, tw, to, a, st);
  return launch<32>(ta, tb, tw, to, a, st);
}

extern "C" int evo_opm_transpose(const void* x, int64_t ld, int64_t col0, int64_t S, int64_t R, int64_t P, void* out_a,
                                 void* out_b, void* stream) {
  using namespace evo;
  EVO_CHECK_ARG(x && out_a, EVO_ERR_ARG, "opm_transpose: null operand");
  EVO_CHECK_ARG(S >= 1 && R >= 1 && P >= 8 && P % 8 == 0 && ld % 8 == 0 && col0 % 8 == 0 &&
                    col0 + (out_b ? 2 : 1) * P <= ld && S * R < (1LL << 31),
                EVO_ERR_SHAPE, "opm_transpose: bad extents");
  EVO_CHECK_ARG((((uintptr_t)x | (uintptr_t)out_a | (uintptr_t)out_b) & 15) == 0 && S % 8 == 0, EVO_ERR_ALIGN,
                "opm_transpose: 16-byte alignment and S %% 8 == 0 required");
  const size_t smem = (size_t)S * ((out_b ? 2 : 1) * P + 8) * 2;
  EVO_CHECK_ARG(smem <= 200 * 1024, EVO_ERR_SHAPE, "opm_transpose: slab too large");
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(opm_transpose_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return cuda_status(e, "opm_transpose attr");
    attr = true;
  }
  ::evo::pdl_launch(opm_transpose_kernel, (unsigned)R, 256, smem, (cudaStream_t)stream, 
      static_cast<const bf16*>(x), ld, col0, (int)S, (int)R, (int)P, static_cast<bf16*>(out_a), static_cast<bf16*>(out_b));
  EVO_LAUNCH_CHECK("opm_transpose launch");
  return EVO_OK;
}

extern "C" int evo_opm_bwd_supported(int64_t I, int64_t J, int64_t S, int64_t P, int64_t Hz) {
  return P == 32 && S >= 8 && S <= 128 && S % 8 == 0 && I >= 32 && I % 32 == 0 && J >= 32 && J % 32 == 0 &&
         (Hz == 64 || Hz == 128);
}

// role 0: da (x = i over a's rows, y = j, other = b_t);  role 1: db (x = j, y = i, other = a_t, W with
// (p, q) exchanged)
static int opm_bwd_one(int role, const void* dy, int64_t ldy, const void* w_o, const void* other_t, int64_t X,
                       int64_t Y, int64_t S, int64_t Hz, float alpha, void* out, int out_f32, int64_t o_ss,
                       int64_t o_sr, int64_t o_sx, int64_t x_split, float* part, int nsplit, cudaStream_t st) {
  using namespace evo;
  CUtensorMap tdy, tw, to;
  const int64_t I = role == 0 ? X : Y, J = role == 0 ? Y : X;
  {  // dy (i, j, c) at (i*J + j)*ldy + c: dims {c, x, y}, box [64 c][32 x][4 y] -> rows (y_l, x_l)
    const int64_t sx = role == 0 ? J * ldy : ldy, sy = role == 0 ? ldy : J * ldy;
    cuuint64_t d[3] = {(cuuint64_t)Hz, (cuuint64_t)X, (cuuint64_t)Y};
    cuuint64_t s[2] = {(cuuint64_t)sx * 2, (cuuint64_t)sy * 2};
    cuuint32_t bx[3] = {64, 32, 4};
    EVO_CHECK_ARG(encode(&tdy, dy, 3, d, s, bx, CU_TENSOR_MAP_SWIZZLE_128B), EVO_ERR_ARG, "opm_bwd: dy map");
    (void)I;
  }
  {  // W rows (chunk-dim index, inner index): da (p, q) -> row p*32+q; db (q, p) -> row p*32+q
    const int64_t s_in = role == 0 ? Hz : 32 * Hz, s_ch = role == 0 ? 32 * Hz : Hz;
    cuuint64_t d[3] = {(cuuint64_t)Hz, 32, 32};
    cuuint64_t s[2] = {(cuuint64_t)s_in * 2, (cuuint64_t)s_ch * 2};
    cuuint32_t bx[3] = {64, 32, 4};
    EVO_CHECK_ARG(encode(&tw, w_o, 3, d, s, bx, CU_TENSOR_MAP_SWIZZLE_128B), EVO_ERR_ARG, "opm_bwd: W map");
  }
  {  // other [y][q][s]: box [64 s][32 q][4 y]
    cuuint64_t d[3] = {(cuuint64_t)S, 32, (cuuint64_t)Y};
    cuuint64_t s[2] = {(cuuint64_t)S * 2, (cuuint64_t)32 * S * 2};
    cuuint32_t bx[3] = {64, 32, 4};
    EVO_CHECK_ARG(encode(&to, other_t, 3, d, s, bx, CU_TENSOR_MAP_SWIZZLE_128B), EVO_ERR_ARG, "opm_bwd: other map");
  }
  OpmBwdArgs a;
  a.X = (int)X;
  a.Y = (int)Y;
  a.S = (int)S;
  a.units_x = (int)(X / 32);
  a.nsplit = nsplit;
  a.ysteps_per_split = (int)((Y / 4 + nsplit - 1) / nsplit);
  a.units = a.units_x * 8 * nsplit;
  a.hz_halves = (int)(Hz / 64);
  a.part = part;
  constexpr size_t smem = 2 * OB_T + 4 * OB_T + 4 * OB_T + 4 * OB_T;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(opm_bwd_contract_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "opm_bwd attr");
    attr = true;
  }
  const int grid = a.units < sm_count() ? a.units : sm_count();
  ::evo::pdl_launch(opm_bwd_contract_kernel, grid, OB_THREADS, smem, st, tdy, tw, to, a);
  EVO_LAUNCH_CHECK("opm_bwd contract launch");
  if (out_f32)
    ::evo::pdl_launch(opm_bwd_finish<float>, (unsigned)X, 256, 0, st, part, nsplit, (int)X, (int)S, alpha, static_cast<float*>(out),
                                                       o_ss, o_sr, o_sx, (int)x_split);
  else
    ::evo::pdl_launch(opm_bwd_finish<bf16>, (unsigned)X, 256, 0, st, part, nsplit, (int)X, (int)S, alpha, static_cast<bf16*>(out),
                                                      o_ss, o_sr, o_sx, (int)x_split);
  EVO_LAUNCH_CHECK("opm_bwd finish launch");
  return EVO_OK;
}

extern "C" int64_t evo_opm_bwd_workspace(int64_t X) { return 4 * X * 32 * 128 * 4; }

extern "C" int evo_opm_bwd_factor(int role, const void* dy, int64_t ldy, const void* w_o, const void* other_t,
                                  int64_t X, int64_t Y, int64_t S, int64_t P, int64_t Hz, float alpha, void* out,
                                  int out_f32, int64_t o_ss, int64_t o_sr, int64_t o_sx, int64_t x_split,
                                  void* workspace, int64_t ws_bytes, void* stream) {
  using namespace evo;
  EVO_CHECK_ARG(role == 0 || role == 1, EVO_ERR_ARG, "opm_bwd_factor: role must be 0 (da) or 1 (db)");
  EVO_CHECK_ARG(dy && w_o && other_t && out && workspace, EVO_ERR_ARG, "opm_bwd_factor: null operand");
  EVO_CHECK_ARG(evo_opm_bwd_supported(role == 0 ? X : Y, role == 0 ? Y : X, S, P, Hz), EVO_ERR_SHAPE,
                "opm_bwd_factor: unsupported extents X=%lld Y=%lld S=%lld P=%lld Hz=%lld", (long long)X, (long long)Y,
                (long long)S, (long long)P, (long long)Hz);
  EVO_CHECK_ARG(ws_bytes >= evo_opm_bwd_workspace(X) && ldy % 8 == 0 && x_split >= 1, EVO_ERR_ARG,
                "opm_bwd_factor: workspace too small or bad strides");
  EVO_CHECK_ARG((((uintptr_t)dy | (uintptr_t)w_o | (uintptr_t)other_t | (uintptr_t)workspace) & 15) == 0,
                EVO_ERR_ALIGN, "opm_bwd_factor: operands must be 16-byte aligned");
  // y splits so the units (x blocks x 8 p-chunks x splits) fill one wave
  // ONE wave: a second partial wave would double the time of the CTAs it lands on
  int ns = (int)(sm_count() / (X / 32 * 8));
  if (ns > 4) ns = 4;
  while (ns > 1 && (Y / 4) / ns < 4) --ns;
  return opm_bwd_one(role, dy, ldy, w_o, other_t, X, Y, S, Hz, alpha, out, out_f32, o_ss, o_sr, o_sx, x_split,
                     static_cast<float*>(workspace), ns < 1 ? 1 : ns, (cudaStream_t)stream);
}
