// Fused bias + mask softmax (engine.fused_softmax_mask_bias_raw, engine.py:193-203)
//   y = softmax((x + bias) * scale + mask)   over the last axis of x [B, H, Q, K]
// and its backward.  HBM-bound: one warp per row, the row held in registers,
// 16/8-byte vector loads in 32-lane-contiguous chunks (fully coalesced), fp32
// max/sum via warp shuffles, exp2 with log2(e) folded into the scale.  bias and
// mask are broadcast through 4-D strides (stride 0 = broadcast) and read in the
// same vectorised chunks when their key stride is 1.
#include <cstdlib>

#include "common.cuh"

#ifndef SMX_U
#define SMX_U 2  // rows per warp step: 2 measured >= 1 (msa_row 60.4 -> 58.4 us)
#endif

namespace evo {

int sm_count();

struct Bcast {
  const void* p;
  int64_t s0, s1, s2, s3;
  int dtype;
};

template <int VEC>
__device__ __forceinline__ void load_vec(const void* base, int dtype, int64_t off, int64_t s3, bool vec_ok, float* v) {
  if (dtype == EVO_BF16) {
    const bf16* p = static_cast<const bf16*>(base) + off;
    if (vec_ok && VEC == 8) {
      uint4 u = *reinterpret_cast<const uint4*>(p);
      unpack_bf16x2(u.x, v[0], v[1]); unpack_bf16x2(u.y, v[2], v[3]);
      unpack_bf16x2(u.z, v[4], v[5]); unpack_bf16x2(u.w, v[6], v[7]);
    } else if (vec_ok && VEC == 4) {
      uint2 u = *reinterpret_cast<const uint2*>(p);
      unpack_bf16x2(u.x, v[0], v[1]); unpack_bf16x2(u.y, v[2], v[3]);
    } else {
#pragma unroll
      for (int i = 0; i < VEC; ++i) v[i] = bf2f(p[i * s3]);
    }
  } else {
    const float* p = static_cast<const float*>(base) + off;
    if (vec_ok && VEC % 4 == 0) {
#pragma unroll
      for (int i = 0; i < VEC; i += 4) {
        float4 u = *reinterpret_cast<const float4*>(p + i);
        v[i] = u.x; v[i + 1] = u.y; v[i + 2] = u.z; v[i + 3] = u.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < VEC; ++i) v[i] = p[i * s3];
    }
  }
}

template <int VEC>
__device__ __forceinline__ void store_vec(void* base, int dtype, int64_t off, const float* v) {
  if (dtype == EVO_BF16) {
    bf16* p = static_cast<bf16*>(base) + off;
    if (VEC == 8) {
      uint4 u;
      u.x = pack_bf16x2(v[0], v[1]); u.y = pack_bf16x2(v[2], v[3]);
      u.z = pack_bf16x2(v[4], v[5]); u.w = pack_bf16x2(v[6], v[7]);
      *reinterpret_cast<uint4*>(p) = u;
    } else if (VEC == 4) {
      uint2 u;
      u.x = pack_bf16x2(v[0], v[1]); u.y = pack_bf16x2(v[2], v[3]);
      *reinterpret_cast<uint2*>(p) = u;
    } else {
#pragma unroll
      for (int i = 0; i < VEC; ++i) p[i] = f2bf(v[i]);
    }
  } else {
    float* p = static_cast<float*>(base) + off;
    if (VEC % 4 == 0) {
#pragma unroll
      for (int i = 0; i < VEC; i += 4) *reinterpret_cast<float4*>(p + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < VEC; ++i) p[i] = v[i];
    }
  }
}

// lane l handles elements (j*32 + l)*VEC .. +VEC for j < NCH
template <int VEC, int NCH>
__global__ void __launch_bounds__(256) softmax_fwd_kernel(const void* __restrict__ x, int xd, Bcast bias, Bcast mask,
                                                          void* __restrict__ y, int yd, int64_t H, int64_t Q,
                                                          int64_t rows, int K, float scale_log2) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  // 32-bit index math (rows < 2^31, host-checked): 64-bit divisions per row cost more issue
  // slots than the row's arithmetic
  const uint32_t r32 = (uint32_t)row, q = r32 % (uint32_t)Q, bh = r32 / (uint32_t)Q;
  const uint32_t h = bh % (uint32_t)H, b = bh / (uint32_t)H;
  const int64_t boff = bias.p ? b * bias.s0 + h * bias.s1 + q * bias.s2 : 0;
  const int64_t moff = mask.p ? b * mask.s0 + h * mask.s1 + q * mask.s2 : 0;
  const bool bvec = bias.s3 == 1, mvec = mask.s3 == 1;
  float v[NCH][VEC];
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const int k0 = (j * 32 + lane) * VEC;
    if (k0 < K) {
      load_vec<VEC>(x, xd, row * K + k0, 1, true, v[j]);
      if (bias.p) {
        float t[VEC];
        load_vec<VEC>(bias.p, bias.dtype, boff + k0 * bias.s3, bias.s3, bvec, t);
#pragma unroll
        for (int i = 0; i < VEC; ++i) v[j][i] += t[i];
      }
#pragma unroll
      for (int i = 0; i < VEC; ++i) v[j][i] *= scale_log2;
      if (mask.p) {
        float t[VEC];
        load_vec<VEC>(mask.p, mask.dtype, moff + k0 * mask.s3, mask.s3, mvec, t);
#pragma unroll
        for (int i = 0; i < VEC; ++i) v[j][i] += t[i] * 1.4426950408889634f;
      }
#pragma unroll
      for (int i = 0; i < VEC; ++i) mx = fmaxf(mx, v[j][i]);
    }
  }
  mx = warp_max(mx);
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const int k0 = (j * 32 + lane) * VEC;
    if (k0 < K) {
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        v[j][i] = ex2f(v[j][i] - mx);
        s += v[j][i];
      }
    }
  }
  const float inv = rcpf(warp_sum(s));
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const int k0 = (j * 32 + lane) * VEC;
    if (k0 < K) {
#pragma unroll
      for (int i = 0; i < VEC; ++i) v[j][i] *= inv;
      store_vec<VEC>(y, yd, row * K + k0, v[j]);
    }
  }
}

// Persistent, software-pipelined forward for the common case (bf16 x / y, K a multiple of 256 up to
// 512, bias / mask absent or bf16 with unit key stride): each warp walks rows with the raw 16-byte loads
// of its next row (x, bias, mask) issued before this row's reductions and stores, so every warp keeps a
// row in flight instead of one DRAM round trip per launched row; (b, h, q) splits are shifts when H and
// Q are powers of two.
template <int NCH, int U>
__global__ void __launch_bounds__(256) softmax_fwd_pipe(const bf16* __restrict__ x, const bf16* __restrict__ bias,
                                                        int64_t bs0, int64_t bs1, int64_t bs2,
                                                        const bf16* __restrict__ mask, int64_t ms0, int64_t ms1,
                                                        int64_t ms2, bf16* __restrict__ y, uint32_t H, uint32_t Q,
                                                        int sh_h, int sh_q, int64_t rows, int K, float sl2) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  // a warp owns U consecutive rows per step; the step's successor is U * nw rows further
  int64_t row0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * U;
  const int64_t stride = nw * U;
  uint4 nx[U][NCH], nb[U][NCH], nm[U][NCH];
  auto load = [&](int64_t r0) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u;
      if (r >= rows) continue;
      const uint32_t r32 = (uint32_t)r;
      const uint32_t bh = sh_q >= 0 ? r32 >> sh_q : r32 / Q, q = r32 - bh * Q;
      const uint32_t b = sh_h >= 0 ? bh >> sh_h : bh / H, h = bh - b * H;
      const bf16* xb = x + r * K;
      const bf16* bb = bias ? bias + b * bs0 + h * bs1 + q * bs2 : nullptr;
      const bf16* mb = mask ? mask + b * ms0 + h * ms1 + q * ms2 : nullptr;
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const int k0 = (j * 32 + lane) * 8;
        nx[u][j] = __ldcs(reinterpret_cast<const uint4*>(xb + k0));
        nb[u][j] = bb ? *reinterpret_cast<const uint4*>(bb + k0) : make_uint4(0, 0, 0, 0);
        nm[u][j] = mb ? *reinterpret_cast<const uint4*>(mb + k0) : make_uint4(0, 0, 0, 0);
      }
    }
  };
  if (row0 < rows) load(row0);
  for (; row0 < rows; row0 += stride) {
    uint4 cx[U][NCH], cb[U][NCH], cm[U][NCH];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < NCH; ++j) { cx[u][j] = nx[u][j]; cb[u][j] = nb[u][j]; cm[u][j] = nm[u][j]; }
    if (row0 + stride < rows) load(row0 + stride);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = row0 + u;
      if (row >= rows) break;
      float v[NCH][8];
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        float xv[8], bv[8], mv[8];
        unpack_bf16x2(cx[u][j].x, xv[0], xv[1]); unpack_bf16x2(cx[u][j].y, xv[2], xv[3]);
        unpack_bf16x2(cx[u][j].z, xv[4], xv[5]); unpack_bf16x2(cx[u][j].w, xv[6], xv[7]);
        unpack_bf16x2(cb[u][j].x, bv[0], bv[1]); unpack_bf16x2(cb[u][j].y, bv[2], bv[3]);
        unpack_bf16x2(cb[u][j].z, bv[4], bv[5]); unpack_bf16x2(cb[u][j].w, bv[6], bv[7]);
        unpack_bf16x2(cm[u][j].x, mv[0], mv[1]); unpack_bf16x2(cm[u][j].y, mv[2], mv[3]);
        unpack_bf16x2(cm[u][j].z, mv[4], mv[5]); unpack_bf16x2(cm[u][j].w, mv[6], mv[7]);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v[j][i] = (xv[i] + bv[i]) * sl2 + mv[i] * 1.4426950408889634f;
          mx = fmaxf(mx, v[j][i]);
        }
      }
      mx = warp_max(mx);
      float sum = 0.f;
#pragma unroll
      for (int j = 0; j < NCH; ++j)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v[j][i] = ex2f(v[j][i] - mx);
          sum += v[j][i];
        }
      const float inv = rcpf(warp_sum(sum));
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        uint4 w;
        w.x = pack_bf16x2(v[j][0] * inv, v[j][1] * inv); w.y = pack_bf16x2(v[j][2] * inv, v[j][3] * inv);
        w.z = pack_bf16x2(v[j][4] * inv, v[j][5] * inv); w.w = pack_bf16x2(v[j][6] * inv, v[j][7] * inv);
        *reinterpret_cast<uint4*>(y + row * K + (j * 32 + lane) * 8) = w;
      }
    }
  }
}

template <int VEC, int NCH>
__global__ void __launch_bounds__(256) softmax_bwd_kernel(const void* __restrict__ y, int yd, const void* __restrict__ dy,
                                                          int dyd, void* __restrict__ dx, int dxd, int64_t rows, int K,
                                                          float scale) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  float yv[NCH][VEC], gv[NCH][VEC];
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const int k0 = (j * 32 + lane) * VEC;
    if (k0 < K) {
      load_vec<VEC>(y, yd, row * K + k0, 1, true, yv[j]);
      load_vec<VEC>(dy, dyd, row * K + k0, 1, true, gv[j]);
#pragma unroll
      for (int i = 0; i < VEC; ++i) s += yv[j][i] * gv[j][i];
    }
  }
  s = warp_sum(s);
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const int k0 = (j * 32 + lane) * VEC;
    if (k0 < K) {
      float o[VEC];
#pragma unroll
      for (int i = 0; i < VEC; ++i) o[i] = scale * yv[j][i] * (gv[j][i] - s);
      store_vec<VEC>(dx, dxd, row * K + k0, o);
    }
  }
}

}  // namespace evo

using namespace evo;

#define SM_DISPATCH(KERN, ...)                                                       \
  do {                                                                               \
    int vec = (K % 8 == 0) ? 8 : (K % 4 == 0 ? 4 : 1);                               \
    int nch = (int)((K + 32 * vec - 1) / (32 * vec));                                \
    if (vec == 8) {                                                                  \
      switch (nch) {                                                                 \
        case 1: ::evo::pdl_launch(KERN<8, 1>, grid, 256, 0, st, __VA_ARGS__); break;                \
        case 2: ::evo::pdl_launch(KERN<8, 2>, grid, 256, 0, st, __VA_ARGS__); break;                \
        case 3: ::evo::pdl_launch(KERN<8, 3>, grid, 256, 0, st, __VA_ARGS__); break;                \
        case 4: ::evo::pdl_launch(KERN<8, 4>, grid, 256, 0, st, __VA_ARGS__); break;                \
        case 5: case 6: ::evo::pdl_launch(KERN<8, 6>, grid, 256, 0, st, __VA_ARGS__); break;        \
        case 7: case 8: ::evo::pdl_launch(KERN<8, 8>, grid, 256, 0, st, __VA_ARGS__); break;        \
        default: set_error("softmax: K=%lld too large (max 2048)", (long long)K);   \
                 return EVO_ERR_SHAPE;                                               \
      }                                                                              \
    } else if (vec == 4) {                                                           \
      switch (nch) {                                                                 \
        case 1: ::evo::pdl_launch(KERN<4, 1>, grid, 256, 0, st, __VA_ARGS__); break;                \
        case 2: ::evo::pdl_launch(KERN<4, 2>, grid, 256, 0, st, __VA_ARGS__); break;                \
        case 3: case 4: ::evo::pdl_launch(KERN<4, 4>, grid, 256, 0, st, __VA_ARGS__); break;        \
        default: set_error("softmax: K=%lld unsupported", (long long)K);             \
                 return EVO_ERR_SHAPE;                                               \
      }                                                                              \
    } else {                                                                         \
      switch (nch) {                                                                 \
        case 1: ::evo::pdl_launch(KERN<1, 1>, grid, 256, 0, st, __VA_ARGS__); break;                \
        case 2: ::evo::pdl_launch(KERN<1, 2>, grid, 256, 0, st, __VA_ARGS__); break;                \
        case 3: case 4: ::evo::pdl_launch(KERN<1, 4>, grid, 256, 0, st, __VA_ARGS__); break;        \
        case 5: case 6: case 7: case 8: ::evo::pdl_launch(KERN<1, 8>, grid, 256, 0, st, __VA_ARGS__); break; \
        default: set_error("softmax: K=%lld unsupported", (long long)K);             \
                 return EVO_ERR_SHAPE;                                               \
      }                                                                              \
    }                                                                                \
  } while (0)

extern "C" int evo_softmax_fwd(const void* x, int x_dtype, const void* bias, int bias_dtype,
                               const int64_t* bias_strides, const void* mask, int mask_dtype,
                               const int64_t* mask_strides, void* y, int y_dtype, int64_t B, int64_t H, int64_t Q,
                               int64_t K, float scale, void* stream) {
  EVO_CHECK_ARG(x && y, EVO_ERR_ARG, "softmax: null x/y");
  EVO_CHECK_ARG(B >= 0 && H >= 1 && Q >= 1 && K >= 1, EVO_ERR_SHAPE, "softmax: bad extents");
  EVO_CHECK_ARG(!bias || bias_strides, EVO_ERR_ARG, "softmax: bias strides missing");
  EVO_CHECK_ARG(!mask || mask_strides, EVO_ERR_ARG, "softmax: mask strides missing");
  const int64_t rows = B * H * Q;
  if (rows == 0) return EVO_OK;
  Bcast bb{bias, 0, 0, 0, 0, bias_dtype}, mm{mask, 0, 0, 0, 0, mask_dtype};
  if (bias) { bb.s0 = bias_strides[0]; bb.s1 = bias_strides[1]; bb.s2 = bias_strides[2]; bb.s3 = bias_strides[3]; }
  if (mask) { mm.s0 = mask_strides[0]; mm.s1 = mask_strides[1]; mm.s2 = mask_strides[2]; mm.s3 = mask_strides[3]; }
  int vec = (K % 8 == 0) ? 8 : (K % 4 == 0 ? 4 : 1);
  uintptr_t al = (uintptr_t)x | (uintptr_t)y;
  EVO_CHECK_ARG((al & 15) == 0 || vec == 1, EVO_ERR_ALIGN, "softmax: x/y must be 16B aligned");
  // vectorised bias/mask loads need aligned base + row offsets
  auto vec_ok = [&](const Bcast& c) {
    if (!c.p || c.s3 != 1) return true;
    int es = c.dtype == EVO_BF16 ? 2 : 4;
    return (((uintptr_t)c.p) % (vec * es) == 0) && c.s0 % vec == 0 && c.s1 % vec == 0 && c.s2 % vec == 0;
  };
  EVO_CHECK_ARG(vec_ok(bb) && vec_ok(mm), EVO_ERR_ALIGN, "softmax: bias/mask rows must be vector aligned");
  cudaStream_t st = (cudaStream_t)stream;
  EVO_CHECK_ARG(rows < (1LL << 31), EVO_ERR_SHAPE, "softmax: more than 2^31 rows");
  const float sl2 = scale * 1.4426950408889634f;
  const bool pipe_ok = x_dtype == EVO_BF16 && y_dtype == EVO_BF16 && (K == 256 || K == 512) &&
                       (!bias || (bias_dtype == EVO_BF16 && bb.s3 == 1)) && (!mask || (mask_dtype == EVO_BF16 && mm.s3 == 1));
  static const bool no_pipe = getenv("EVO_SOFTMAX_NO_PIPE") != nullptr;  // A/B switch
  if (pipe_ok && !no_pipe) {
    auto lg2 = [](int64_t v) { int k = 0; while ((int64_t(1) << k) < v) ++k; return (int64_t(1) << k) == v ? k : -1; };
    const int64_t need = (rows + 8 * SMX_U - 1) / (8 * SMX_U), cap = (int64_t)sm_count() * 8;
    dim3 gp((unsigned)(need < cap ? need : cap));
    if (K == 256)
      ::evo::pdl_launch(softmax_fwd_pipe<1, SMX_U>, gp, 256, 0, st, (const bf16*)x, (const bf16*)bias, bb.s0, bb.s1, bb.s2,
                        (const bf16*)mask, mm.s0, mm.s1, mm.s2, (bf16*)y, (uint32_t)H, (uint32_t)Q, lg2(H), lg2(Q), rows,
                        (int)K, sl2);
    else
      ::evo::pdl_launch(softmax_fwd_pipe<2, SMX_U>, gp, 256, 0, st, (const bf16*)x, (const bf16*)bias, bb.s0, bb.s1, bb.s2,
                        (const bf16*)mask, mm.s0, mm.s1, mm.s2, (bf16*)y, (uint32_t)H, (uint32_t)Q, lg2(H), lg2(Q), rows,
                        (int)K, sl2);
    EVO_LAUNCH_CHECK("softmax fwd");
    return EVO_OK;
  }
  dim3 grid((unsigned)((rows + 7) / 8));
  SM_DISPATCH(softmax_fwd_kernel, x, x_dtype, bb, mm, y, y_dtype, H, Q, rows, (int)K, sl2);
  EVO_LAUNCH_CHECK("softmax fwd");
  return EVO_OK;
}

extern "C" int evo_softmax_bwd(const void* y, int y_dtype, const void* dy, int dy_dtype, void* dx, int dx_dtype,
                               int64_t rows, int64_t K, float scale, void* stream) {
  EVO_CHECK_ARG(y && dy && dx, EVO_ERR_ARG, "softmax bwd: null pointer");
  if (rows == 0) return EVO_OK;
  uintptr_t al = (uintptr_t)y | (uintptr_t)dy | (uintptr_t)dx;
  EVO_CHECK_ARG((al & 15) == 0 || K % 4 != 0, EVO_ERR_ALIGN, "softmax bwd: pointers must be 16B aligned");
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid((unsigned)((rows + 7) / 8));
  SM_DISPATCH(softmax_bwd_kernel, y, y_dtype, dy, dy_dtype, dx, dx_dtype, rows, (int)K, scale);
  EVO_LAUNCH_CHECK("softmax bwd");
  return EVO_OK;
}
