// Batched bf16 GEMM on 5th-generation tensor cores (tcgen05, fp32 accumulators in TMEM).
//
//   C[b] = alpha * A[b] . B[b]^T + beta * C[b]      A:[M,K]  B:[N,K]  C:[M,N]
//
// Used for the dense contractions of the Evoformer block:
//   * triangle multiplicative update einsums (evoformer.py:276 "ikh,jkh->ijh",
//     evoformer.py:283 "kih,kjh->ijh") - batch = channel h, M = N = K = N_r;
//   * the outer-product-mean contraction (evoformer.py:253 "sip,sjq->ijpq") -
//     M = N_r*p, N = N_r*p, K = N_s, written straight into the [i][j][p][q] layout;
//   * all of their backward products.
//
// Design: 128-thread CTA, tile 128 x BN x 64, STAGES-deep cp.async ring into
// canonical (SWIZZLE_NONE) UMMA layouts; one elected thread issues
// tcgen05.mma (M=128, N=BN, K=16) and commits each stage to an mbarrier that
// gates the reuse of that stage's shared memory; the 4 warps then drain the
// TMEM accumulator (tcgen05.ld 32x32b) in the epilogue.  Operands may be K-major
// or MN-major (instruction-descriptor major bits), so no transpose copies are
// ever made.  Addressing is 2-level per dim (see EvoMat in include/evo.h).
#include <cstdlib>

#include "common.cuh"
#include "tma.cuh"

#include <cstdlib>
#include <cstring>

namespace evo {

int sm_count();

struct MatArg {
  const char* ptr;
  int64_t bs;                 // batch stride (elements)
  uint32_t split0, split1;
  uint32_t mul0, sh0, mul1, sh1;  // magic numbers: i / split = umulhi(i, mul) >> sh (mul = 0: split 1)
  int64_t hi0, lo0, hi1, lo1;
};

// round-up magic-number division, exact for dividends < 2^31 (all indices are)
__device__ __forceinline__ uint32_t fdiv(uint32_t n, uint32_t mul, uint32_t sh) {
  return mul == 0 ? n : (__umulhi(n, mul) >> sh);
}

__device__ __forceinline__ int64_t mat_off(const MatArg& m, uint32_t i0, uint32_t i1) {
  uint32_t q0 = fdiv(i0, m.mul0, m.sh0), r0 = i0 - q0 * m.split0;
  uint32_t q1 = fdiv(i1, m.mul1, m.sh1), r1 = i1 - q1 * m.split1;
  return (int64_t)q0 * m.hi0 + (int64_t)r0 * m.lo0 + (int64_t)q1 * m.hi1 + (int64_t)r1 * m.lo1;
}

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;

// load one ROWS x 64 operand tile (bf16) into a canonical layout; 128 threads
template <int ROWS, bool MN>
__device__ __forceinline__ void load_tile(uint32_t sdst, const MatArg& m, const char* base, uint32_t r0,
                                          uint32_t k0, uint32_t R, uint32_t K) {
  constexpr int CHUNKS = ROWS * GEMM_BK / 8;  // 16-byte chunks
#pragma unroll
  for (int it = 0; it < CHUNKS / 128; ++it) {
    int ch = threadIdx.x + it * 128;
    uint32_t r, k, soff;
    if (!MN) {  // 8 chunks (64 k) per row
      r = ch >> 3;
      k = (ch & 7) * 8;
      soff = kmajor_off(r, k, ROWS);
    } else {    // ROWS/8 chunks per k
      k = ch / (ROWS / 8);
      r = (ch % (ROWS / 8)) * 8;
      soff = mnmajor_off(r, k, ROWS);
    }
    bool pred = (r0 + r < R) && (k0 + k < K);
    const char* src = base;
    if (pred) src = base + mat_off(m, r0 + r, k0 + k) * 2;
    cp_async16(sdst + soff, src, pred);
  }
}

// split-K: blockIdx.z = batch * splits + split; with ws != nullptr each split writes its
// fp32 partial tile densely to ws[(split * batch + b)][M][N] and bgemm_splitk_reduce
// applies alpha/beta and the output addressing.
template <int BN, bool A_MN, bool B_MN, int STAGES, typename TC>
__global__ void __launch_bounds__(128) bgemm_kernel(MatArg A, MatArg B, MatArg C, uint32_t M, uint32_t N,
                                                    uint32_t K, float alpha, float beta, int c_mode, int splits,
                                                    float* __restrict__ ws) {
  pdl_wait();
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[STAGES];
  __shared__ uint32_t tmem_base_sh;

  constexpr uint32_t A_BYTES = GEMM_BM * GEMM_BK * 2;
  constexpr uint32_t B_BYTES = BN * GEMM_BK * 2;
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sA = sbase, sB = sbase + STAGES * A_BYTES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t m0 = blockIdx.y * GEMM_BM, n0 = blockIdx.x * BN;
  const int64_t bz = blockIdx.z / splits;
  const int split = blockIdx.z % splits;
  const char* Abase = A.ptr + bz * A.bs * 2;
  const char* Bbase = B.ptr + bz * B.bs * 2;

  if (warp == 0) tmem_alloc(&tmem_base_sh, BN < 32 ? 32 : BN);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&mbar[s], 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  const int KT_all = (K + GEMM_BK - 1) / GEMM_BK;
  const int KT_per = (KT_all + splits - 1) / splits;
  const int kt0 = split * KT_per;
  const int KT = (KT_all - kt0 < KT_per ? KT_all - kt0 : KT_per);  // >= 1 by construction
  constexpr uint32_t IDESC = make_idesc_bf16(GEMM_BM, BN, A_MN, B_MN);

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) {
      load_tile<GEMM_BM, A_MN>(sA + s * A_BYTES, A, Abase, m0, (kt0 + s) * GEMM_BK, M, K);
      load_tile<BN, B_MN>(sB + s * B_BYTES, B, Bbase, n0, (kt0 + s) * GEMM_BK, N, K);
    }
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    const int pf = kt + STAGES - 1;
    if (pf < KT) {
      const int ps = pf % STAGES;
      if (kt >= 1) mbar_wait(&mbar[ps], ((kt - 1) / STAGES) & 1);  // MMA kt-1 released stage ps
      load_tile<GEMM_BM, A_MN>(sA + ps * A_BYTES, A, Abase, m0, (kt0 + pf) * GEMM_BK, M, K);
      load_tile<BN, B_MN>(sB + ps * B_BYTES, B, Bbase, n0, (kt0 + pf) * GEMM_BK, N, K);
    }
    cp_async_commit();
    cp_async_wait<STAGES - 1>();
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      const int s = kt % STAGES;
#pragma unroll
      for (int kk = 0; kk < GEMM_BK / 16; ++kk) {
        uint64_t ad = make_sdesc(sA + s * A_BYTES + kk * 2 * (GEMM_BM / 8) * 128, (GEMM_BM / 8) * 128, 128);
        uint64_t bd = make_sdesc(sB + s * B_BYTES + kk * 2 * (BN / 8) * 128, (BN / 8) * 128, 128);
        mma_bf16(tmem, ad, bd, IDESC, (kt | kk) != 0);
      }
      mma_commit(&mbar[s]);
    }
    __syncwarp();
  }

  mbar_wait(&mbar[(KT - 1) % STAGES], ((KT - 1) / STAGES) & 1);
  tc_fence_after();

  // ---------------- epilogue: TMEM -> registers -> (smem staging) -> global
  const uint32_t row = m0 + warp * 32 + lane;
  const bool row_ok = row < M;
  char* Cbase = const_cast<char*>(C.ptr) + bz * C.bs * (int64_t)sizeof(TC);
  if (c_mode == 1 && ws == nullptr) {
    // stage the alpha-scaled tile in the (now idle) pipeline buffers, row pitch padded by
    // 16 bytes (conflict-free 16-byte stores), then write 16-byte chunks with consecutive
    // threads on consecutive chunks of a row: full-sector, coalesced row segments.
    constexpr int PITCH = BN * (int)sizeof(TC) + 16;
    uint8_t* stile = smem;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
      tmem_ld_wait();
      uint8_t* dst = stile + (warp * 32 + lane) * PITCH + c0 * (int)sizeof(TC);
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        if constexpr (sizeof(TC) == 2) {
          *reinterpret_cast<uint4*>(dst + j * 2) =
              make_uint4(pack_bf16x2(alpha * v[j], alpha * v[j + 1]), pack_bf16x2(alpha * v[j + 2], alpha * v[j + 3]),
                         pack_bf16x2(alpha * v[j + 4], alpha * v[j + 5]), pack_bf16x2(alpha * v[j + 6], alpha * v[j + 7]));
        } else {
          *reinterpret_cast<float4*>(dst + j * 4) =
              make_float4(alpha * v[j], alpha * v[j + 1], alpha * v[j + 2], alpha * v[j + 3]);
          *reinterpret_cast<float4*>(dst + j * 4 + 16) =
              make_float4(alpha * v[j + 4], alpha * v[j + 5], alpha * v[j + 6], alpha * v[j + 7]);
        }
      }
    }
    __syncthreads();
    constexpr int CPR = BN * (int)sizeof(TC) / 16;  // 16-byte chunks per tile row
    constexpr int EPC = 16 / (int)sizeof(TC);        // elements per chunk
    for (int ch = threadIdx.x; ch < GEMM_BM * CPR; ch += 128) {
      const int r = ch / CPR, cc = ch % CPR;
      const uint32_t grow = m0 + r, gcol = n0 + cc * EPC;
      if (grow >= M || gcol >= N) continue;
      const uint32_t qr = fdiv(grow, C.mul0, C.sh0), rr = grow - qr * C.split0;
      const uint32_t qc = fdiv(gcol, C.mul1, C.sh1), rc = gcol - qc * C.split1;
      TC* p = reinterpret_cast<TC*>(Cbase) + (int64_t)qr * C.hi0 + (int64_t)rr * C.lo0 + (int64_t)qc * C.hi1 + rc;
      uint4 val = *reinterpret_cast<const uint4*>(stile + r * PITCH + cc * 16);
      if (beta != 0.f) {
        const TC* sv = reinterpret_cast<const TC*>(&val);
        uint4 outv;
        TC* ov = reinterpret_cast<TC*>(&outv);
#pragma unroll
        for (int e = 0; e < EPC; ++e) stf<TC>(ov + e, ldf<TC>(sv + e) + beta * ldf<TC>(p + e));
        val = outv;
      }
      *reinterpret_cast<uint4*>(p) = val;
    }
  } else {
    int64_t roff = 0;
    if (row_ok) {
      uint32_t q = fdiv(row, C.mul0, C.sh0), r = row - q * C.split0;
      roff = (int64_t)q * C.hi0 + (int64_t)r * C.lo0;
    }
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
      tmem_ld_wait();
      if (!row_ok) continue;
      if (ws != nullptr) {  // split-K partial, dense fp32 [M][N]
        float* wrow = ws + ((int64_t)(split * (gridDim.z / splits) + bz) * M + row) * N;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const uint32_t col = n0 + c0 + j;
          if (col + 4 <= N) *reinterpret_cast<float4*>(wrow + col) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          else
            for (int e = 0; e < 4; ++e)
              if (col + e < N) wrow[col + e] = v[j + e];
        }
        continue;
      }
      TC* crow = reinterpret_cast<TC*>(Cbase) + roff;
#pragma unroll
      for (int j = 0; j < 32; ++j) {  // generic addressing (e.g. rows contiguous: coalesced per column)
        uint32_t col = n0 + c0 + j;
        if (col >= N) break;
        uint32_t q = fdiv(col, C.mul1, C.sh1), r = col - q * C.split1;
        TC* p = crow + (int64_t)q * C.hi1 + (int64_t)r * C.lo1;
        float o = alpha * v[j];
        if (beta != 0.f) o += beta * ldf<TC>(p);
        stf<TC>(p, o);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, BN < 32 ? 32 : BN);
}

// C = alpha * sum_split ws[split] + beta * C   (output addressing of C; 8 elements per thread
// along whichever C dimension is contiguous)
template <typename TC>
__global__ void __launch_bounds__(256) bgemm_splitk_reduce(const float* __restrict__ ws, MatArg C, uint32_t M,
                                                           uint32_t N, int64_t batch, int splits, float alpha,
                                                           float beta, int rows_contig) {
  pdl_wait();
  const int64_t MN = (int64_t)M * N;
  const int64_t n8 = batch * MN / 8;
  char* Cbase = const_cast<char*>(C.ptr);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b, r0, c0;
    if (rows_contig) {  // 8 consecutive rows of one column
      const int64_t per_b = MN / 8;
      b = i / per_b;
      const int64_t t = i % per_b;
      c0 = t / (M / 8);
      r0 = (t % (M / 8)) * 8;
    } else {            // 8 consecutive columns of one row
      const int64_t per_b = MN / 8;
      b = i / per_b;
      const int64_t t = i % per_b;
      r0 = t / (N / 8);
      c0 = (t % (N / 8)) * 8;
    }
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int s = 0; s < splits; ++s) {
      const float* w = ws + ((int64_t)s * batch + b) * MN;
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += rows_contig ? w[(r0 + e) * N + c0] : w[r0 * N + c0 + e];
    }
    TC* cb = reinterpret_cast<TC*>(Cbase) + b * C.bs;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t r = (uint32_t)(rows_contig ? r0 + e : r0), c = (uint32_t)(rows_contig ? c0 : c0 + e);
      const uint32_t qr = fdiv(r, C.mul0, C.sh0), rr = r - qr * C.split0, qc = fdiv(c, C.mul1, C.sh1), rc = c - qc * C.split1;
      TC* p = cb + (int64_t)qr * C.hi0 + (int64_t)rr * C.lo0 + (int64_t)qc * C.hi1 + (int64_t)rc * C.lo1;
      float o = alpha * acc[e];
      if (beta != 0.f) o += beta * ldf<TC>(p);
      stf<TC>(p, o);
    }
  }
}


// =====================================================================================
// Warp-specialised persistent variant (the default path):
//   warps 0..3  producers: cp.async ring of STAGES (A,B) k-tiles, completion signalled with
//               cp.async.mbarrier.arrive.noinc on full[stage] (128 arrivals)
//   warp 4      MMA issuer: waits full[stage], issues tcgen05.mma into one of two TMEM
//               accumulators, tcgen05.commit -> empty[stage]; after the last k-tile of a
//               tile, commit -> tmem_full[buf]
//   warps 5..8  epilogue: wait tmem_full[buf], TMEM -> regs -> smem staging -> coalesced
//               16-byte global stores (or split-K fp32 partials), arrive tmem_empty[buf]
// The CTA loops over tiles (tile += gridDim.x), so the loads and MMAs of tile t+1 run
// under the epilogue of tile t.
// =====================================================================================
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ int64_t off_dim0(const MatArg& m, uint32_t i) {
  uint32_t q = fdiv(i, m.mul0, m.sh0);
  return (int64_t)q * m.hi0 + (int64_t)(i - q * m.split0) * m.lo0;
}
__device__ __forceinline__ int64_t off_dim1(const MatArg& m, uint32_t i) {
  uint32_t q = fdiv(i, m.mul1, m.sh1);
  return (int64_t)q * m.hi1 + (int64_t)(i - q * m.split1) * m.lo1;
}

// ROWS x 64 operand tile loader for the 128 producer threads.  The row (M/N) part of every
// address is computed once per output tile, the K part once per k-tile, so the inner loop
// is one add + one cp.async per 16-byte chunk.
template <int ROWS, bool MN>
struct TileLoader {
  static constexpr int IT = ROWS / 16;  // chunks per thread per k-tile
  int64_t roff[MN ? 1 : IT];            // element offset of the row part, -1 = out of range

  // K-major thread map: lane = (k chunk of a pair, row of 16); warp w owns k chunks 2w, 2w+1.
  // Global: 32 contiguous bytes (one sector) per row; smem: each half-warp writes 256
  // contiguous bytes (two core matrices) -> conflict-free 16-byte cp.async stores.
  static __device__ __forceinline__ int krow(int tid) { return tid & 15; }
  static __device__ __forceinline__ int kcol(int tid) { return ((tid >> 5) * 2 + ((tid >> 4) & 1)) * 8; }
  __device__ __forceinline__ void setup(const MatArg& m, uint32_t r0, uint32_t R, int tid) {
    if constexpr (!MN) {
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const uint32_t r = r0 + krow(tid) + it * 16;
        roff[it] = r < R ? off_dim0(m, r) : -1;
      }
    } else {
      const uint32_t r = r0 + (tid % (ROWS / 8)) * 8;
      roff[0] = r < R ? off_dim0(m, r) : -1;
    }
  }
  // smem offsets: chunk it sits a constant stride after chunk 0 (16 rows = 2 core-matrix
  // rows for K-major; KSTEP k = KSTEP/8 core-matrix columns = 2048 B for MN-major)
  __device__ __forceinline__ void load(uint32_t sdst, const MatArg& m, const char* base, uint32_t k0, uint32_t K,
                                       int tid) const {
    if constexpr (!MN) {
      const int k = kcol(tid);
      const uint32_t kk = k0 + k;
      const bool kok = kk < K;
      const int64_t koff = kok ? off_dim1(m, kk) : 0;
      const uint32_t s0 = sdst + kmajor_off(krow(tid), k, ROWS);
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const bool pred = kok && roff[it] >= 0;
        cp_async16(s0 + it * 256, pred ? base + (roff[it] + koff) * 2 : base, pred);
      }
    } else {
      constexpr int KSTEP = 128 / (ROWS / 8);
      const int kb = tid / (ROWS / 8);
      const uint32_t s0 = sdst + mnmajor_off((tid % (ROWS / 8)) * 8, kb, ROWS);
      const bool rok = roff[0] >= 0;
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const uint32_t kk = k0 + kb + it * KSTEP;
        const bool pred = rok && kk < K;
        cp_async16(s0 + it * 2048, pred ? base + (roff[0] + off_dim1(m, kk)) * 2 : base, pred);
      }
    }
  }
};

// ---------------------------------------------------------------- TMA (K-major operands)
// A / B tiles arrive by cp.async.bulk.tensor with the 128-byte swizzle: BM (BN) rows of 64
// bf16 = 128 B each, 8-row atoms of 1 KB.  One elected producer thread per stage instead of
// 128 threads x 12 cp.async with per-chunk address arithmetic.
// How the producer addresses one operand's tensor map.  The map's dims are, in order: the
// contiguous dim (K for K-major, rows for MN-major) as [lo] or [lo = 32, hi], the other dim
// as [lo] or [lo = split, hi], then [batch] (MatArg's two-level addressing, e.g. the OPM
// [i][j][p][q] layout, maps onto dims of the tensor map).
struct TmaOp {
  int c2;       // contiguous dim in 32-element runs (64-byte swizzle)
  int chi;      // the map has a contiguous-hi dim (placed after the other dim): the whole stage
                // tile is ONE box; otherwise one box per 64-row atom (MN-major, ragged rows)
  int cw;       // contiguous-lo width of the map (32 or 64, or the full extent when !chi)
  int o2;       // other dim two-level
  int split_o;
};
// issue the box whose contiguous-dim start is cs and other-dim start is os (coordinates stay in
// registers: the producer is a single thread, so no local-memory coordinate arrays).  Maps are
// always >= 3-D (a unit batch dim is kept for 1-level operands).
__device__ __forceinline__ void tma_issue(const TmaOp& op, uint32_t dst, const CUtensorMap* map, int cs, int os, int b,
                                          uint64_t* bar) {
  // map dims: [c_lo, o_lo, (o_hi), (c_hi), batch]
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  const uint32_t br = smem_u32(bar);
  const int cl = op.chi ? cs % op.cw : cs, ch = op.chi ? cs / op.cw : 0;
  const int ol = op.o2 ? os % op.split_o : os, oh = op.o2 ? os / op.split_o : 0;
  if (!op.o2 && !op.chi) tma_ld3(dst, m, cl, ol, b, br);
  else if (!op.o2) tma_ld4(dst, m, cl, ol, ch, b, br);
  else if (!op.chi) tma_ld4(dst, m, cl, ol, oh, b, br);
  else tma_ld5(dst, m, cl, ol, oh, ch, b, br);
}

// MN-major SWIZZLE_128B descriptor: tile = (rows/64) TMA boxes of [64 k][64 mn] (8 KB each);
// LBO = 8 KB (next 64-element MN atom), SBO = 1 KB (next 8 k rows)
__device__ __forceinline__ uint64_t make_sdesc_sw128_mn(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(8192 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// K-major SWIZZLE_128B descriptor: LBO = 16 B (unused within the atom), SBO = 1 KB (8 rows)
__device__ __forceinline__ uint64_t make_sdesc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;  // version
  d |= (uint64_t)2 << 61;  // layout SWIZZLE_128B
  return d;
}
// SWIZZLE_64B variants for operands whose contiguous dim comes in 32-element (64 B) runs:
// K-major: [rows][32 k] blocks, 8-row atoms of 512 B (SBO); MN-major: [64 k][32 mn] atoms
// of 4 KB (LBO) with 8 k rows = 512 B (SBO)
__device__ __forceinline__ uint64_t make_sdesc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;  // layout SWIZZLE_64B
  return d;
}
__device__ __forceinline__ uint64_t make_sdesc_sw64_mn(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(4096 >> 4) << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}
// descriptor of K-step kk (16 k) of an operand tile of `rows` rows at `base`
__device__ __forceinline__ uint64_t tma_desc(bool mn, bool sw64, uint32_t base, int kk, int rows) {
  if (!sw64) return mn ? make_sdesc_sw128_mn(base + kk * 2048) : make_sdesc_sw128(base + kk * 32);
  if (mn) return make_sdesc_sw64_mn(base + kk * 1024);
  return make_sdesc_sw64(base + (kk >> 1) * rows * 64 + (kk & 1) * 32);
}

constexpr int WS_EPI_WARPS = 4;  // one epilogue warp per TMEM lane quarter (8 measured no faster)
constexpr int WS_GEMM_THREADS = 160 + 32 * WS_EPI_WARPS;  // 4 producer warps + MMA warp + epilogue

template <int BN, bool A_MN, bool B_MN, int STAGES, typename TC, bool TMA>
__global__ void __launch_bounds__(WS_GEMM_THREADS, 1) bgemm_ws_kernel(MatArg A, MatArg B, MatArg C, uint32_t M, uint32_t N,
                                                          uint32_t K, float alpha, float beta, int c_mode, int splits,
                                                          float* __restrict__ ws, int batch,
                                                          const __grid_constant__ CUtensorMap tmA,
                                                          const __grid_constant__ CUtensorMap tmB, TmaOp opA,
                                                          TmaOp opB) {
  pdl_wait();
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_sh;
  constexpr uint32_t A_BYTES = GEMM_BM * GEMM_BK * 2;
  constexpr uint32_t B_BYTES = BN * GEMM_BK * 2;
  constexpr int PITCH = BN * (int)sizeof(TC) + 16;
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sA = sbase, sB = sbase + STAGES * A_BYTES;
  uint8_t* stile = smem + STAGES * (A_BYTES + B_BYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const uint32_t mt = (M + GEMM_BM - 1) / GEMM_BM, nt = (N + BN - 1) / BN;
  const uint32_t total = mt * nt * (uint32_t)batch * (uint32_t)splits;
  const int KT_all = (K + GEMM_BK - 1) / GEMM_BK;
  const int KT_per = (KT_all + splits - 1) / splits;
  // tile id -> (batch, split, m-tile, n-tile); n fastest so consecutive CTAs share the A rows
  auto decode = [&](uint32_t t, uint32_t& b, int& sp, uint32_t& m0, uint32_t& n0, int& kt0, int& ktn) {
    const uint32_t n_i = t % nt;
    t /= nt;
    const uint32_t m_i = t % mt;
    t /= mt;
    sp = (int)(t % splits);
    b = t / splits;
    m0 = m_i * GEMM_BM;
    n0 = n_i * BN;
    kt0 = sp * KT_per;
    ktn = KT_all - kt0 < KT_per ? KT_all - kt0 : KT_per;
  };

  if (warp == 0) tmem_alloc(&tmem_sh, 2 * BN);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], TMA ? 1 : 128);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 32 * WS_EPI_WARPS);
    }
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;

  if (TMA && warp < 4) {
    // ---------------- TMA producer (one thread)
    if (threadIdx.x == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
        uint32_t b, m0, n0;
        int sp, kt0, ktn;
        decode(t, b, sp, m0, n0, kt0, ktn);
        for (int kt = 0; kt < ktn; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], A_BYTES + B_BYTES);
          const int k0 = (kt0 + kt) * GEMM_BK;
          // one box per operand and stage when the map has a contiguous-hi dim (the box then
          // spans the atoms: [atom][64 k][mn run] MN-major, [k run][rows][32 k] K-major);
          // otherwise MN-major tiles take one [64 k][64 mn] box per 64 rows
          if (!A_MN || opA.chi) {
            tma_issue(opA, sA + stage * A_BYTES, &tmA, A_MN ? (int)m0 : k0, A_MN ? k0 : (int)m0, (int)b, &full[stage]);
          } else {
#pragma unroll
            for (int j = 0; j < GEMM_BM / 64; ++j)
              tma_issue(opA, sA + stage * A_BYTES + j * 8192, &tmA, (int)m0 + 64 * j, k0, (int)b, &full[stage]);
          }
          if (!B_MN || opB.chi) {
            tma_issue(opB, sB + stage * B_BYTES, &tmB, B_MN ? (int)n0 : k0, B_MN ? k0 : (int)n0, (int)b, &full[stage]);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_issue(opB, sB + stage * B_BYTES + j * 8192, &tmB, (int)n0 + 64 * j, k0, (int)b, &full[stage]);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp < 4) {
    // ---------------- producers (warps 0..3)
    const int tid = threadIdx.x;
    int stage = 0;
    uint32_t phase = 0;
    TileLoader<GEMM_BM, A_MN> la;
    TileLoader<BN, B_MN> lb;
    for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
      uint32_t b, m0, n0;
      int sp, kt0, ktn;
      decode(t, b, sp, m0, n0, kt0, ktn);
      const char* Abase = A.ptr + (int64_t)b * A.bs * 2;
      const char* Bbase = B.ptr + (int64_t)b * B.bs * 2;
      la.setup(A, m0, M, tid);
      lb.setup(B, n0, N, tid);
      for (int kt = 0; kt < ktn; ++kt) {
        mbar_wait(&empty[stage], phase ^ 1);
        la.load(sA + stage * A_BYTES, A, Abase, (kt0 + kt) * GEMM_BK, K, tid);
        lb.load(sB + stage * B_BYTES, B, Bbase, (kt0 + kt) * GEMM_BK, K, tid);
        cp_async_mbar_arrive_noinc(&full[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    cp_async_wait<0>();
  } else if (warp == 4) {
    // ---------------- MMA issuer
    constexpr uint32_t IDESC = make_idesc_bf16(GEMM_BM, BN, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (uint32_t t = blockIdx.x; t < total; t += gridDim.x, ++it) {
      uint32_t b, m0, n0;
      int sp, kt0, ktn;
      decode(t, b, sp, m0, n0, kt0, ktn);
      const int buf = it & 1;
      mbar_wait(&tempty[buf], ((it >> 1) & 1) ^ 1);  // epilogue drained this accumulator
      tc_fence_after();
      for (int kt = 0; kt < ktn; ++kt) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
#pragma unroll
          for (int kk = 0; kk < GEMM_BK / 16; ++kk) {
            uint64_t ad, bd;
            if constexpr (TMA) {
              ad = tma_desc(A_MN, opA.c2, sA + stage * A_BYTES, kk, GEMM_BM);
              bd = tma_desc(B_MN, opB.c2, sB + stage * B_BYTES, kk, BN);
            } else {
              ad = make_sdesc(sA + stage * A_BYTES + kk * 2 * (GEMM_BM / 8) * 128, (GEMM_BM / 8) * 128, 128);
              bd = make_sdesc(sB + stage * B_BYTES + kk * 2 * (BN / 8) * 128, (BN / 8) * 128, 128);
            }
            mma_bf16(tmem + buf * BN, ad, bd, IDESC, (kt | kk) != 0);
          }
          mma_commit(&empty[stage]);
          if (kt == ktn - 1) mma_commit(&tfull[buf]);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue (warps 5..12 -> TMEM lane quarters 1,2,3,0,1,2,3,0; the two
    // warps of a quarter split the tile's columns)
    constexpr int NE = 32 * WS_EPI_WARPS;
    constexpr int CH = BN / (WS_EPI_WARPS / 4);  // columns per epilogue warp
    const int q = warp & 3;            // lane quarter of this warp
    const int c_lo = ((warp - 5) / 4) * CH;
    const int et = threadIdx.x - 160;  // 0..NE-1 epilogue thread id
    int it = 0;
    for (uint32_t t = blockIdx.x; t < total; t += gridDim.x, ++it) {
      uint32_t b, m0, n0;
      int sp, kt0, ktn;
      decode(t, b, sp, m0, n0, kt0, ktn);
      const int buf = it & 1;
      mbar_wait(&tfull[buf], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t row = m0 + q * 32 + lane;
      const bool row_ok = row < M;
      char* Cbase = const_cast<char*>(C.ptr) + (int64_t)b * C.bs * (int64_t)sizeof(TC);
      const uint32_t tbase = tmem + buf * BN + ((uint32_t)(q * 32) << 16);
      if (c_mode == 1 && ws == nullptr) {
#pragma unroll 1
        for (int c0 = c_lo; c0 < c_lo + CH; c0 += 32) {
          float v[32];
          tmem_ld32(tbase + c0, v);
          tmem_ld_wait();
          uint8_t* dst = stile + (q * 32 + lane) * PITCH + c0 * (int)sizeof(TC);
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            if constexpr (sizeof(TC) == 2) {
              *reinterpret_cast<uint4*>(dst + j * 2) = make_uint4(
                  pack_bf16x2(alpha * v[j], alpha * v[j + 1]), pack_bf16x2(alpha * v[j + 2], alpha * v[j + 3]),
                  pack_bf16x2(alpha * v[j + 4], alpha * v[j + 5]), pack_bf16x2(alpha * v[j + 6], alpha * v[j + 7]));
            } else {
              *reinterpret_cast<float4*>(dst + j * 4) =
                  make_float4(alpha * v[j], alpha * v[j + 1], alpha * v[j + 2], alpha * v[j + 3]);
              *reinterpret_cast<float4*>(dst + j * 4 + 16) =
                  make_float4(alpha * v[j + 4], alpha * v[j + 5], alpha * v[j + 6], alpha * v[j + 7]);
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[buf]);  // accumulator free for tile t + 2*gridDim.x
        named_sync(1, NE);
        constexpr int CPR = BN * (int)sizeof(TC) / 16;
        constexpr int EPC = 16 / (int)sizeof(TC);
        constexpr int RSTEP = NE / CPR;
        const int cc = et % CPR;
        const uint32_t gcol = n0 + cc * EPC;
        const bool col_ok = gcol < N;
        TC* cbase = reinterpret_cast<TC*>(Cbase) + (col_ok ? off_dim1(C, gcol) : 0);
        for (int r = et / CPR; r < GEMM_BM; r += RSTEP) {
          const uint32_t grow = m0 + r;
          if (grow >= M || !col_ok) continue;
          TC* p = cbase + off_dim0(C, grow);
          uint4 val = *reinterpret_cast<const uint4*>(stile + r * PITCH + cc * 16);
          if (beta != 0.f) {
            const TC* sv = reinterpret_cast<const TC*>(&val);
            uint4 outv;
            TC* ov = reinterpret_cast<TC*>(&outv);
#pragma unroll
            for (int e = 0; e < EPC; ++e) stf<TC>(ov + e, ldf<TC>(sv + e) + beta * ldf<TC>(p + e));
            val = outv;
          }
          *reinterpret_cast<uint4*>(p) = val;
        }
        named_sync(1, NE);  // staging tile reusable
      } else {
        int64_t roff = 0;
        if (row_ok) {
          uint32_t qq = fdiv(row, C.mul0, C.sh0), r = row - qq * C.split0;
          roff = (int64_t)qq * C.hi0 + (int64_t)r * C.lo0;
        }
#pragma unroll 1
        for (int c0 = c_lo; c0 < c_lo + CH; c0 += 32) {
          float v[32];
          tmem_ld32(tbase + c0, v);
          tmem_ld_wait();
          if (!row_ok) continue;
          if (ws != nullptr) {
            float* wrow = ws + (((int64_t)sp * batch + b) * M + row) * N;
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const uint32_t col = n0 + c0 + j;
              if (col + 4 <= N)
                *reinterpret_cast<float4*>(wrow + col) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
              else
                for (int e = 0; e < 4; ++e)
                  if (col + e < N) wrow[col + e] = v[j + e];
            }
            continue;
          }
          TC* crow = reinterpret_cast<TC*>(Cbase) + roff;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            uint32_t col = n0 + c0 + j;
            if (col >= N) break;
            uint32_t qq = fdiv(col, C.mul1, C.sh1), r = col - qq * C.split1;
            TC* p = crow + (int64_t)qq * C.hi1 + (int64_t)r * C.lo1;
            float o = alpha * v[j];
            if (beta != 0.f) o += beta * ldf<TC>(p);
            stf<TC>(p, o);
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[buf]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 2 * BN);
}

static MatArg to_arg(const EvoMat* m, int64_t ext0, int64_t ext1) {
  MatArg a;
  a.ptr = static_cast<const char*>(m->ptr);
  a.bs = m->batch_stride;
  auto sp = [](int64_t s, int64_t ext) -> uint32_t {
    int64_t v = (s <= 0 || s > ext) ? ext : s;
    if (v < 1) v = 1;
    return (uint32_t)v;
  };
  a.split0 = sp(m->split[0], ext0);
  a.split1 = sp(m->split[1], ext1);
  auto magic = [](uint32_t d, uint32_t& mul, uint32_t& sh) {
    if (d == 1) {
      mul = sh = 0;
      return;
    }
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;  // ceil(log2 d)
    const uint64_t p = 31 + l;
    mul = (uint32_t)(((1ull << p) + d - 1) / d);
    sh = (uint32_t)(p - 32);
  };
  magic(a.split0, a.mul0, a.sh0);
  magic(a.split1, a.mul1, a.sh1);
  a.hi0 = m->stride_hi[0];
  a.lo0 = m->stride_lo[0];
  a.hi1 = m->stride_hi[1];
  a.lo1 = m->stride_lo[1];
  return a;
}

// contiguous along dim d in runs of 8 elements?
static bool runs8(const MatArg& a, int d) {
  uint32_t split = d == 0 ? a.split0 : a.split1;
  int64_t lo = d == 0 ? a.lo0 : a.lo1;
  return lo == 1 && (split % 8) == 0;
}

template <int BN, bool AM, bool BMN, typename TC, int STAGES>
static int launch_bgemm_s(MatArg A, MatArg B, MatArg C, int64_t batch, int64_t M, int64_t N, int64_t K, float alpha,
                          float beta, int c_mode, int splits, float* ws, cudaStream_t st) {
  const size_t pipe = STAGES * (GEMM_BM * GEMM_BK * 2 + BN * GEMM_BK * 2);
  const size_t stage_tile = (size_t)GEMM_BM * (BN * sizeof(TC) + 16);  // epilogue staging (reuses the ring)
  const size_t smem = pipe > stage_tile ? pipe : stage_tile;
  auto kern = bgemm_kernel<BN, AM, BMN, STAGES, TC>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "bgemm attr");
    attr_set = true;
  }
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + GEMM_BM - 1) / GEMM_BM), (unsigned)(batch * splits));
  ::evo::pdl_launch(kern, grid, 128, smem, st, A, B, C, (uint32_t)M, (uint32_t)N, (uint32_t)K, alpha, beta, c_mode, splits,
                                splits > 1 ? ws : nullptr);
  EVO_LAUNCH_CHECK("bgemm launch");
  if (splits > 1) {
    const bool rows_contig = C.lo0 == 1 && C.split0 % 8 == 0 && M % 8 == 0;
    EVO_CHECK_ARG(rows_contig || N % 8 == 0, EVO_ERR_ALIGN, "bgemm split-K: M or N must be a multiple of 8");
    int64_t n8 = batch * M * N / 8;
    int64_t g = (n8 + 255) / 256, cap = (int64_t)sm_count() * 16;
    ::evo::pdl_launch(bgemm_splitk_reduce<TC>, (unsigned)(g < cap ? g : cap), 256, 0, st, ws, C, (uint32_t)M, (uint32_t)N, batch,
                                                                           splits, alpha, beta, rows_contig ? 1 : 0);
    EVO_LAUNCH_CHECK("bgemm split-K reduce");
  }
  return EVO_OK;
}

// cuTensorMapEncodeTiled from the driver, fetched once through the runtime (no -lcuda)
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// Tensor map of one operand (rows = M or N extent).  K-major: box [box_rows][64 k];
// MN-major: box [64 k][64 rows] (128-byte swizzle).  The contiguous dim may be plain (one run)
// or two-level with runs of exactly 32 elements (64 B: 64-byte swizzle, one box per run); the
// other dim may be plain or two-level with a split dividing the box extent.  Returns false (-> cp.async
// producer) for anything else.
static bool tma_map(CUtensorMap* map, TmaOp* op, const MatArg& a, bool mn_major, int64_t rows, int64_t K,
                    int64_t batch, int box_rows) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc || ((uintptr_t)a.ptr & 15)) return false;
  // contiguous (c) and other (o) dims of the MatArg
  const int64_t ext_c = mn_major ? rows : K, ext_o = mn_major ? K : rows;
  const uint32_t split_c = mn_major ? a.split0 : a.split1, split_o = mn_major ? a.split1 : a.split0;
  const int64_t lo_c = mn_major ? a.lo0 : a.lo1, hi_c = mn_major ? a.hi0 : a.hi1;
  const int64_t lo_o = mn_major ? a.lo1 : a.lo0, hi_o = mn_major ? a.hi1 : a.hi0;
  const int box_o = mn_major ? GEMM_BK : box_rows;     // other-dim extent of one stage tile
  const int tile_c = mn_major ? box_rows : GEMM_BK;    // contiguous-dim extent of one stage tile
  if (lo_c != 1) return false;
  auto stride_ok = [](int64_t el) { return el > 0 && (el * 2) % 16 == 0 && el * 2 < (1LL << 40); };
  TmaOp o{};
  cuuint64_t cdim_lo, cdim_hi = 0, cstride_hi = 0;
  cuuint32_t cbox_lo, cbox_hi = 1;
  if ((int64_t)split_c >= ext_c) {                 // one run
    if (mn_major && ext_c % 64 == 0) {             // split into 64-wide atoms, one box per tile
      o.chi = 1; o.cw = 64;
      cdim_lo = 64; cbox_lo = 64; cdim_hi = ext_c / 64; cstride_hi = 64; cbox_hi = tile_c / 64;
    } else {
      cdim_lo = ext_c; cbox_lo = 64; o.cw = 1 << 30;
    }
  } else if (split_c == 32 && ext_c % 32 == 0 && stride_ok(hi_c)) {  // 64-byte runs: SWIZZLE_64B
    o.c2 = 1; o.chi = 1; o.cw = 32;
    cdim_lo = 32; cbox_lo = 32; cdim_hi = ext_c / 32; cstride_hi = hi_c; cbox_hi = tile_c / 32;
  } else {
    return false;
  }
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
  int nd = 0;
  dims[nd] = cdim_lo; box[nd] = cbox_lo; ++nd;
  if ((int64_t)split_o >= ext_o) {
    if (!stride_ok(lo_o)) return false;
    dims[nd] = (cuuint64_t)ext_o; strides[nd - 1] = (cuuint64_t)lo_o * 2; box[nd] = (cuuint32_t)box_o; ++nd;
    o.split_o = 1 << 30;
  } else if (box_o % split_o == 0 && ext_o % split_o == 0 && stride_ok(lo_o) && stride_ok(hi_o)) {
    dims[nd] = split_o; strides[nd - 1] = (cuuint64_t)lo_o * 2; box[nd] = split_o; ++nd;
    dims[nd] = (cuuint64_t)(ext_o / split_o); strides[nd - 1] = (cuuint64_t)hi_o * 2;
    box[nd] = (cuuint32_t)(box_o / split_o); ++nd;
    o.o2 = 1;
    o.split_o = (int)split_o;
  } else {
    return false;
  }
  if (o.chi) {
    if (!stride_ok((int64_t)cstride_hi)) return false;
    dims[nd] = cdim_hi; strides[nd - 1] = cstride_hi * 2; box[nd] = cbox_hi; ++nd;
  }
  // batch dim always present (unit extent when batch == 1) so every map is 3-, 4- or 5-D
  if (batch > 1 && !stride_ok(a.bs)) return false;
  dims[nd] = (cuuint64_t)batch;
  strides[nd - 1] = batch > 1 ? (cuuint64_t)a.bs * 2 : strides[nd - 2] * (cuuint64_t)dims[nd - 1];
  box[nd] = 1;
  ++nd;
  if (nd < 3 || nd > 5) return false;
  *op = o;
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, (cuuint32_t)nd, const_cast<char*>(a.ptr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, o.c2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, bool AM, bool BMN, typename TC>
static int launch_bgemm_ws(MatArg A, MatArg B, MatArg C, int64_t batch, int64_t M, int64_t N, int64_t K, float alpha,
                           float beta, int c_mode, int splits, float* ws, cudaStream_t st, bool reduce = true) {
  // 256-wide N tiles (long-K, large problems) halve the A-tile re-reads per FLOP; 3 stages
  // keep the ring + staging tile within shared memory
  // split-K partials leave from registers (no staging tile): 256-wide N tiles keep 4 stages
  constexpr int STAGES = (BN >= 256 && sizeof(TC) == 2) ? 3 : 4;
  const size_t pipe = STAGES * (GEMM_BM * GEMM_BK * 2 + BN * GEMM_BK * 2);
  const size_t smem = pipe + (splits > 1 ? 0 : (size_t)GEMM_BM * (BN * sizeof(TC) + 16));
  if (smem > 227 * 1024) return set_error("bgemm_ws: tile config exceeds shared memory"), EVO_ERR_SHAPE;
  // operands whose addressing maps onto a tensor map take the TMA producer (128-byte swizzle)
  CUtensorMap ta, tb;
  memset(&ta, 0, sizeof(ta));
  memset(&tb, 0, sizeof(tb));
  static const bool tma_off = [] { const char* e = getenv("EVO_BGEMM_NO_TMA"); return e && e[0] == '1'; }();
  TmaOp oa{}, ob{};
  const bool tma = !tma_off && tma_map(&ta, &oa, A, AM, M, K, batch, GEMM_BM) && tma_map(&tb, &ob, B, BMN, N, K, batch, BN);
  const int64_t tiles = ((M + GEMM_BM - 1) / GEMM_BM) * ((N + BN - 1) / BN) * batch * splits;
  const int64_t grid = tiles < sm_count() ? tiles : sm_count();
  auto run = [&](auto kern, size_t& attr_set) -> int {
    if (attr_set < smem) {  // the split-K form needs no staging tile: the attribute tracks the largest launch
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return cuda_status(e, "bgemm_ws attr");
      attr_set = smem;
    }
    ::evo::pdl_launch(kern, (unsigned)grid, WS_GEMM_THREADS, smem, st, A, B, C, (uint32_t)M, (uint32_t)N, (uint32_t)K, alpha, beta,
                                                        c_mode, splits, splits > 1 ? ws : nullptr, (int)batch, ta, tb,
                                                        oa, ob);
    return EVO_OK;
  };
  static size_t attr_plain = 0, attr_tma = 0;
  int rc;
  if (tma) rc = run(bgemm_ws_kernel<BN, AM, BMN, STAGES, TC, true>, attr_tma);
  else rc = run(bgemm_ws_kernel<BN, AM, BMN, STAGES, TC, false>, attr_plain);
  if (rc) return rc;
  EVO_LAUNCH_CHECK("bgemm_ws launch");
  if (splits > 1 && reduce) {
    const bool rows_contig = C.lo0 == 1 && C.split0 % 8 == 0 && M % 8 == 0;
    EVO_CHECK_ARG(rows_contig || N % 8 == 0, EVO_ERR_ALIGN, "bgemm split-K: M or N must be a multiple of 8");
    int64_t n8 = batch * M * N / 8;
    int64_t g = (n8 + 255) / 256, cap = (int64_t)sm_count() * 16;
    ::evo::pdl_launch(bgemm_splitk_reduce<TC>, (unsigned)(g < cap ? g : cap), 256, 0, st, ws, C, (uint32_t)M, (uint32_t)N, batch,
                                                                           splits, alpha, beta, rows_contig ? 1 : 0);
    EVO_LAUNCH_CHECK("bgemm split-K reduce");
  }
  return EVO_OK;
}

static bool use_v1() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EVO_BGEMM_V1");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// short K (<= 2 k-tiles, e.g. the OPM contraction over N_s = 128): 2 stages -> 64 KB smem,
// 3 CTAs per SM so one CTA's epilogue overlaps another's main loop
template <int BN, bool AM, bool BMN, typename TC>
static int launch_bgemm(MatArg A, MatArg B, MatArg C, int64_t batch, int64_t M, int64_t N, int64_t K, float alpha,
                        float beta, int c_mode, int splits, float* ws, cudaStream_t st) {
  if (!use_v1()) return launch_bgemm_ws<BN, AM, BMN, TC>(A, B, C, batch, M, N, K, alpha, beta, c_mode, splits, ws, st);
  const int64_t kt = (K + GEMM_BK - 1) / GEMM_BK / splits;
  if (kt <= 2) return launch_bgemm_s<BN, AM, BMN, TC, 2>(A, B, C, batch, M, N, K, alpha, beta, c_mode, splits, ws, st);
  return launch_bgemm_s<BN, AM, BMN, TC, 3>(A, B, C, batch, M, N, K, alpha, beta, c_mode, splits, ws, st);
}

template <int BN, typename TC>
static int dispatch_major(bool am, bool bm, MatArg A, MatArg B, MatArg C, int64_t batch, int64_t M, int64_t N,
                          int64_t K, float alpha, float beta, int c_mode, int splits, float* ws, cudaStream_t st) {
  if (!am && !bm)
    return launch_bgemm<BN, false, false, TC>(A, B, C, batch, M, N, K, alpha, beta, c_mode, splits, ws, st);
  if (!am && bm)
    return launch_bgemm<BN, false, true, TC>(A, B, C, batch, M, N, K, alpha, beta, c_mode, splits, ws, st);
  if (am && !bm)
    return launch_bgemm<BN, true, false, TC>(A, B, C, batch, M, N, K, alpha, beta, c_mode, splits, ws, st);
  return launch_bgemm<BN, true, true, TC>(A, B, C, batch, M, N, K, alpha, beta, c_mode, splits, ws, st);
}

// split-K factor: only when the output tiles cannot fill the machine and K is long
// N tile width.  A long-K product with 64 < N <= 128 (OPM backward: M = 8192, N = 128,
// K = 8192) takes one 128-wide N tile so the (HBM-sized) A operand is streamed once rather
// than once per 64-wide N tile; split-K restores the parallelism.
// Otherwise the persistent grid (one CTA per SM) should hold every tile in one wave: 64-wide
// tiles when even those fit, else 128-wide ones when those fit (triangle einsums: 128 tiles of
// 128 x 128 over 32 channels, 7.5 -> 6.2 us; measured).
static int pick_bn(int64_t batch, int64_t M, int64_t N, int64_t K, bool small, bool wide) {
  static const int forced = [] { const char* e = getenv("EVO_BGEMM_BN"); return e ? atoi(e) : 0; }();
  if (forced == 64 || forced == 128) return forced;
  if (N > 64 && N <= 128 && K >= 2048) return 128;
  if (N <= 64) return 64;
  const int64_t mt = (M + 127) / 128;
  if (small) return mt * ((N + 63) / 64) * batch <= (int64_t)sm_count() ? 64 : 128;
  return wide ? 256 : 128;
}

// split-K for long-K products with fewer output tiles than SMs: the persistent grid is one
// CTA per SM, so the split count keeps every (tile, split) unit in ONE wave (tiles * splits <=
// SMs).  Measured on the OPM backward (64 tiles, K = 8192): 2 splits 56 us, 3 -> 71, 5 -> 77,
// 9 -> 85, 16 -> 115 (more waves and more fp32 partial traffic).
static int pick_splits(int64_t batch, int64_t M, int64_t N, int64_t K, int bn) {
  static const int forced = [] { const char* e = getenv("EVO_BGEMM_SPLITS"); return e ? atoi(e) : 0; }();
  if (forced > 0 && K >= 2048) return forced;
  const int64_t tiles = ((M + 127) / 128) * ((N + bn - 1) / bn) * batch;
  const int64_t kt = (K + GEMM_BK - 1) / GEMM_BK;
  const int64_t slots = (int64_t)sm_count();
  if (tiles * 2 > slots || kt < 16) return 1;
  int64_t s = slots / tiles;
  if (s > kt / 8) s = kt / 8;  // >= 8 k-tiles per split
  if (s > 16) s = 16;
  if (s < 1) s = 1;
  const int64_t per = (kt + s - 1) / s;
  return (int)((kt + per - 1) / per);  // every split owns >= 1 k-tile
}


static int bgemm_entry(const EvoMat* A, const EvoMat* B, const EvoMat* C, int64_t batch, int64_t M, int64_t N,
                       int64_t K, float alpha, float beta, void* workspace, int64_t ws_bytes, void* stream) {
  EVO_CHECK_ARG(A && B && C && A->ptr && B->ptr && C->ptr, EVO_ERR_ARG, "bgemm: null operand");
  EVO_CHECK_ARG(batch >= 1 && M >= 1 && N >= 1 && K >= 1, EVO_ERR_SHAPE, "bgemm: bad extents b=%lld M=%lld N=%lld K=%lld",
                (long long)batch, (long long)M, (long long)N, (long long)K);
  EVO_CHECK_ARG(M < (1LL << 31) && N < (1LL << 31) && K < (1LL << 31) && batch < 65536, EVO_ERR_SHAPE,
                "bgemm: extents too large");
  EVO_CHECK_ARG(A->dtype == EVO_BF16 && B->dtype == EVO_BF16, EVO_ERR_DTYPE, "bgemm: A/B must be bf16");
  EVO_CHECK_ARG(C->dtype == EVO_BF16 || C->dtype == EVO_F32, EVO_ERR_DTYPE, "bgemm: C must be bf16/f32");
  MatArg a = to_arg(A, M, K), b = to_arg(B, N, K), c = to_arg(C, M, N);
  bool a_k = runs8(a, 1), a_mn = runs8(a, 0), b_k = runs8(b, 1), b_mn = runs8(b, 0);
  EVO_CHECK_ARG(a_k || a_mn, EVO_ERR_ALIGN, "bgemm: A must be contiguous in runs of 8 along M or K");
  EVO_CHECK_ARG(b_k || b_mn, EVO_ERR_ALIGN, "bgemm: B must be contiguous in runs of 8 along N or K");
  bool am = !a_k, bm = !b_k;
  EVO_CHECK_ARG(K % 8 == 0 && (!am || M % 8 == 0) && (!bm || N % 8 == 0), EVO_ERR_ALIGN,
                "bgemm: K (and M/N for MN-major operands) must be multiples of 8");
  uintptr_t align_or = (uintptr_t)A->ptr | (uintptr_t)B->ptr;
  EVO_CHECK_ARG((align_or & 15) == 0, EVO_ERR_ALIGN, "bgemm: A/B pointers must be 16-byte aligned");
  int c_mode = 0;
  if (runs8(c, 1) && N % 8 == 0 && ((uintptr_t)C->ptr & 15) == 0 && (c.hi1 % 8) == 0 && (c.hi0 % 8) == 0 &&
      (c.lo0 % 8) == 0 && (c.bs % 8) == 0)
    c_mode = 1;
  cudaStream_t st = (cudaStream_t)stream;
  // wide N tiles amortise the A-tile loads; N=64 keeps small problems parallel
  bool small = ((M + 127) / 128) * ((N + 127) / 128) * batch < 148;
  const bool wide = !small && C->dtype == EVO_BF16 && N >= 256 && K >= 512 && !use_v1() &&
                    ((M + 127) / 128) * ((N + 255) / 256) * batch >= 2 * 148;
  const int bn = pick_bn(batch, M, N, K, small, wide);
  int splits = pick_splits(batch, M, N, K, bn);
  if (splits > 1 && (!workspace || ws_bytes < splits * batch * M * N * 4)) splits = 1;
  float* ws = (float*)workspace;
  if (C->dtype == EVO_BF16) {
    if (bn == 64) return dispatch_major<64, bf16>(am, bm, a, b, c, batch, M, N, K, alpha, beta, c_mode, splits, ws, st);
    if (bn == 256) return dispatch_major<256, bf16>(am, bm, a, b, c, batch, M, N, K, alpha, beta, c_mode, splits, ws, st);
    return dispatch_major<128, bf16>(am, bm, a, b, c, batch, M, N, K, alpha, beta, c_mode, splits, ws, st);
  }
  if (bn == 64) return dispatch_major<64, float>(am, bm, a, b, c, batch, M, N, K, alpha, beta, c_mode, splits, ws, st);
  return dispatch_major<128, float>(am, bm, a, b, c, batch, M, N, K, alpha, beta, c_mode, splits, ws, st);
}

// Weight gradient dW[M][N] (fp32) += X^T dY with X [rows][M], dY [rows][N] bf16 row-major (K = rows,
// tens of thousands): both operands MN-major through TMA, 256-wide N tiles (the 128-row A tile is
// re-read once per 256 output columns instead of once per 64), and split-K sized so the
// (tile, split) units form ONE wave over the SMs - every SM streams its K slice of
// X and dY at HBM rate (the fp32 partials, units x BN x 512 B, are reduced by all SMs); the deterministic
// reduction adds the partials into dW in split order (beta = 1: gradients accumulate).
static int wgrad_splits(int64_t M, int64_t N, int64_t rows, int bn) {
  const int64_t tiles = ((M + 127) / 128) * ((N + bn - 1) / bn);
  const int64_t kt = (rows + GEMM_BK - 1) / GEMM_BK;
  int64_t s = sm_count() / tiles;
  if (s > kt / 4) s = kt / 4;  // >= 4 k-tiles per split
  if (s < 1) s = 1;
  const int64_t per = (kt + s - 1) / s;
  return (int)((kt + per - 1) / per);
}
static int wgrad_bn(int64_t N) { return N >= 192 ? 256 : (N > 64 ? 128 : 64); }

// dw[m][n] (row stride ldw) += sum_s ws[s][m][n]: a CTA owns 32 four-element column groups and its 8
// warps split the partials (warp w takes s = w, w + 8, ...; 4 loads in flight per thread); the 8
// per-warp sums meet in shared memory and are added in warp order (deterministic).
__global__ void __launch_bounds__(256) wgrad_reduce(const float* __restrict__ ws, float* __restrict__ dw, int64_t ldw,
                                                    int M, int N, int splits) {
  pdl_wait();
  __shared__ float4 part[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t MN = (int64_t)M * N;
  const int64_t e = ((int64_t)blockIdx.x * 32 + lane) * 4;  // first of 4 elements (N % 4 == 0)
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (e < MN) {
    int s = w;
    for (; s + 24 < splits; s += 32) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(reinterpret_cast<const float4*>(ws + (int64_t)(s + 8 * u) * MN + e));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
      }
    }
    for (; s < splits; s += 8) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(ws + (int64_t)s * MN + e));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  part[w][lane] = acc;
  __syncthreads();
  if (w == 0 && e < MN) {
    float4 t = part[0][lane];
#pragma unroll
    for (int i = 1; i < 8; ++i) {
      t.x += part[i][lane].x; t.y += part[i][lane].y; t.z += part[i][lane].z; t.w += part[i][lane].w;
    }
    const int64_t m = e / N, n = e % N;
    float4* d = reinterpret_cast<float4*>(dw + m * ldw + n);
    float4 o = *d;
    o.x += t.x; o.y += t.y; o.z += t.z; o.w += t.w;
    *d = o;
  }
}

}  // namespace evo

extern "C" int64_t evo_wgrad_workspace(int64_t rows, int64_t M, int64_t N) {
  const int bn = evo::wgrad_bn(N);
  const int s = evo::wgrad_splits(M, N, rows, bn);
  return s > 1 ? (int64_t)s * M * N * 4 : 0;
}

extern "C" int evo_wgrad(const void* x, int64_t ldx, const void* dy, int64_t ldy, float* dw, int64_t ldw, int64_t rows,
                         int64_t M, int64_t N, void* workspace, int64_t ws_bytes, void* stream) {
  using namespace evo;
  EVO_CHECK_ARG(x && dy && dw, EVO_ERR_ARG, "wgrad: null operand");
  EVO_CHECK_ARG(rows >= 1 && M >= 8 && N >= 8 && M % 8 == 0 && N % 8 == 0 && ldx % 8 == 0 && ldy % 8 == 0 &&
                    rows < (1LL << 31),
                EVO_ERR_SHAPE, "wgrad: M, N, ldx, ldy must be multiples of 8");
  EVO_CHECK_ARG((((uintptr_t)x | (uintptr_t)dy) & 15) == 0 && ((uintptr_t)dw & 15) == 0, EVO_ERR_ALIGN,
                "wgrad: operands must be 16-byte aligned");
  int bn = wgrad_bn(N);
  int splits = wgrad_splits(M, N, rows, bn);
  if (splits > 1 && (!workspace || ws_bytes < (int64_t)splits * M * N * 4)) splits = 1;
  if (splits == 1 && bn == 256) bn = 128;  // the unsplit form stages its tile in shared memory
  EvoMat A{const_cast<void*>(x), EVO_BF16, 0, {0, 0}, {0, 0}, {1, ldx}};   // A[m][k] = x[k][m]
  EvoMat B{const_cast<void*>(dy), EVO_BF16, 0, {0, 0}, {0, 0}, {1, ldy}};  // B[n][k] = dy[k][n]
  EvoMat C{dw, EVO_F32, 0, {0, 0}, {0, 0}, {ldw, 1}};
  MatArg a = to_arg(&A, M, rows), b = to_arg(&B, N, rows), c = to_arg(&C, M, N);
  cudaStream_t st = (cudaStream_t)stream;
  float* ws = (float*)workspace;
  // the main kernel writes the split partials (its own split-K reduction is replaced below)
  const int rc = bn == 256   ? launch_bgemm_ws<256, true, true, float>(a, b, c, 1, M, N, rows, 1.f, 1.f, 0, splits, ws, st, false)
                 : bn == 128 ? launch_bgemm_ws<128, true, true, float>(a, b, c, 1, M, N, rows, 1.f, 1.f, 0, splits, ws, st, false)
                             : launch_bgemm_ws<64, true, true, float>(a, b, c, 1, M, N, rows, 1.f, 1.f, 0, splits, ws, st, false);
  if (rc || splits == 1) return rc;
  EVO_CHECK_ARG(ldw % 4 == 0, EVO_ERR_ALIGN, "wgrad: ldw must be a multiple of 4");
  const int64_t groups = (M * N / 4 + 31) / 32;
  ::evo::pdl_launch(wgrad_reduce, (unsigned)groups, 256, 0, st, ws, dw, ldw, (int)M, (int)N, splits);
  EVO_LAUNCH_CHECK("wgrad reduce");
  return EVO_OK;
}

extern "C" int evo_bgemm(const EvoMat* A, const EvoMat* B, const EvoMat* C, int64_t batch, int64_t M, int64_t N,
                         int64_t K, float alpha, float beta, void* stream) {
  return evo::bgemm_entry(A, B, C, batch, M, N, K, alpha, beta, nullptr, 0, stream);
}

extern "C" int64_t evo_bgemm_workspace(int64_t batch, int64_t M, int64_t N, int64_t K) {
  bool small = ((M + 127) / 128) * ((N + 127) / 128) * batch < 148;
  const int bn = evo::pick_bn(batch, M, N, K, small, false);
  const int splits = evo::pick_splits(batch, M, N, K, bn);
  return splits > 1 ? (int64_t)splits * batch * M * N * 4 : 0;
}

extern "C" int evo_bgemm_ws(const EvoMat* A, const EvoMat* B, const EvoMat* C, int64_t batch, int64_t M, int64_t N,
                            int64_t K, float alpha, float beta, void* workspace, int64_t ws_bytes, void* stream) {
  return evo::bgemm_entry(A, B, C, batch, M, N, K, alpha, beta, workspace, ws_bytes, stream);
}
