/*
 * evo.h - C ABI of libevo.so, the sm_100a (B200) kernels of the Evoformer hot path.
 *
 * The reference (evoplan, /root/reference/pkg/src/evoplan) is pure Python/numpy:
 * it has no FFI.  Each entry point below replaces the numpy arithmetic of one
 * reference function (cited per function); the Python package
 * paper_2203_00854_b200 keeps the reference's module API and binds these through
 * ctypes.
 *
 * Conventions
 *   - plain pointers + element counts/strides (int64, in ELEMENTS, not bytes);
 *   - every pointer is device memory owned by the caller; kernels never allocate,
 *     free or synchronize; all work is enqueued on `stream` (a cudaStream_t, may be 0);
 *   - activations are bf16 (EVO_BF16) or fp32 (EVO_F32); parameters fp32;
 *     accumulation and statistics always fp32;
 *   - return 0 (EVO_OK) or an EVO_ERR_* code; evo_last_error_string() explains.
 *     The Python layer maps EVO_ERR_SHAPE -> DimensionError, EVO_ERR_DOMAIN ->
 *     DomainError (errors.py:8-13), everything else -> KernelError.
 */
#ifndef EVO_H_
#define EVO_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  EVO_OK = 0,
  EVO_ERR_SHAPE = 1,   /* DimensionError */
  EVO_ERR_DTYPE = 2,
  EVO_ERR_ALIGN = 3,   /* pointer/stride alignment required by 16-byte vector paths */
  EVO_ERR_CUDA = 4,    /* launch/runtime error */
  EVO_ERR_ARG = 5,
  EVO_ERR_DOMAIN = 6   /* DomainError (non-finite input), only from evo_count_nonfinite users */
};

enum { EVO_BF16 = 0, EVO_F32 = 1 };

/* ------------------------------------------------------------------ library */
const char* evo_version(void);
const char* evo_last_error_string(void);
/* number of SMs and compute capability of the current device */
int evo_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* ------------------------------------------------------------------ LayerNorm
 * Replaces engine.layernorm_raw (engine.py:206-217): population variance, eps
 * inside the square root.  Element (r, c) of x is at x[r*x_rs + c*x_cs] (so a
 * channel-major input, e.g. the triangle product t[h][i][j] of
 * evoformer.py:269, is normalised without a transpose); y is row-major [rows, cols].
 * mean/rstd (fp32 [rows]) are saved for the backward; may be NULL.
 */
int evo_layernorm_fwd(const void* x, int x_dtype, int64_t x_rs, int64_t x_cs,
                      const float* gamma, const float* beta,
                      void* y, int y_dtype, float* mean, float* rstd,
                      int64_t rows, int64_t cols, float eps, void* stream);
/* dx = res + dLN/dx (res may be NULL, or alias dx to accumulate in place - the residual
 * stream's gradient); dgamma/dbeta are ACCUMULATED (caller zeroes them); dx and res are
 * addressed like x. */
int evo_layernorm_bwd(const void* dy, int dy_dtype, const void* x, int x_dtype, int64_t x_rs, int64_t x_cs,
                      const float* gamma, const float* mean, const float* rstd,
                      void* dx, int dx_dtype, const void* res,
                      float* dgamma, float* dbeta, int64_t rows, int64_t cols, void* stream);

/* same, plus dx_colsum[c] += sum_r dx[r, c] (fp32, ACCUMULATED): the bias gradient of the
 * module that consumes this residual-stream gradient, fused into the pass that writes dx
 * (contiguous rows of 32/64/128/256 columns; EVO_ERR_SHAPE otherwise). */
int evo_layernorm_bwd_colsum(const void* dy, int dy_dtype, const void* x, int x_dtype, int64_t x_rs, int64_t x_cs,
                             const float* gamma, const float* mean, const float* rstd,
                             void* dx, int dx_dtype, const void* res,
                             float* dgamma, float* dbeta, float* dx_colsum, int64_t rows, int64_t cols, void* stream);

/* LN followed by k = 8 dot products per row (msa_row_bias, evoformer.py:201-207; fewer
 * heads are zero-padded to 8):  out[h*out_hs + r] = sum_c LN(x)[r, c] * w[c*8 + h].
 * ln_out (row-major, may be NULL) receives LN(x); mean/rstd are saved. bf16. */
int evo_layernorm_rowdot_fwd(const void* x, int x_dtype, const float* gamma, const float* beta,
                             const float* w, int k, void* out, int out_dtype, int64_t out_hs,
                             void* ln_out, float* mean, float* rstd,
                             int64_t rows, int64_t cols, float eps, void* stream);
/* its backward in one pass: dy = w . dout[:, r], dw += LN(x)^T dout (fp32 [cols][8]),
 * dgamma/dbeta accumulated, dx = res + dLN (res may alias dx). dout fp32 [8][rows]. */
int evo_layernorm_rowdot_bwd(const void* x, int x_dtype, const float* gamma, const float* beta,
                             const float* w, int k, const float* dout, int64_t out_hs,
                             const float* mean, const float* rstd, const void* res, void* dx,
                             float* dgamma, float* dbeta, float* dw, int64_t rows, int64_t cols, void* stream);

/* Residual epilogue fused with the NEXT module's LayerNorm (bf16 only, cols 32/64/128/256):
 *   out = res + [sigmoid(gp) *] (y + bias)      (evoformer.py:316-324 residual adds; gp may be NULL)
 *   ln  = LayerNorm(out) with gamma/beta, mean/rstd saved (engine.py:206-217; stats of the
 *         bf16-rounded out, exactly what a separate evo_layernorm_fwd of out would see)   */
int evo_residual_layernorm_fwd(const void* res, const void* y, int64_t y_rs, const float* bias,
                               const void* gp, int64_t gp_rs, void* out, const float* gamma,
                               const float* beta, void* ln, float* mean, float* rstd, int64_t rows,
                               int64_t cols, float eps, void* stream);

/* ------------------------------------------------------------------ fused softmax
 * Replaces engine.fused_softmax_mask_bias_raw (engine.py:193-203) and the block's
 * softmax (evoformer.py:186-190):  y = softmax((x + bias) * scale + mask) over the
 * last axis.  x, y contiguous [B, H, Q, K]; bias/mask are read at
 *   ptr[b*s[0] + h*s[1] + q*s[2] + k*s[3]]   (stride 0 = broadcast), may be NULL.
 * scale = 1 reproduces engine.py; mask = NULL, scale = c^-1/2 the block.
 * Rows are processed in registers (K <= 8192).                                   */
int evo_softmax_fwd(const void* x, int x_dtype, const void* bias, int bias_dtype, const int64_t* bias_strides,
                    const void* mask, int mask_dtype, const int64_t* mask_strides,
                    void* y, int y_dtype, int64_t B, int64_t H, int64_t Q, int64_t K,
                    float scale, void* stream);
/* dx = scale * y * (dy - sum_k dy*y)   (gradient w.r.t. x and, unreduced, bias) */
int evo_softmax_bwd(const void* y, int y_dtype, const void* dy, int dy_dtype, void* dx, int dx_dtype,
                    int64_t rows, int64_t K, float scale, void* stream);

/* ------------------------------------------------------------------ gated attention
 * Replaces _attention_core's per-head loop (evoformer.py:182-192) for all four
 * variants (msa_row with pair bias, msa_col, pair_row / pair_col with per-key
 * bias, evoformer.py:201-311).  Per (batch b, head h):
 *   s   = (q k^T + bias) * scale              (bias BEFORE scale, G1)
 *   a   = softmax_k(s)
 *   o   = a v                                 -> o_raw (ungated, kept for backward)
 *   out = sigmoid(g) * o                      -> o_gated (feeds the output projection)
 * Element (b, l, h, d) of q is at q[b*q_sb + l*q_sl + h*c + d] (same for k, v, g,
 * o_gated, o_raw with their own strides), so the transposed variants (msa_col,
 * pair_col) run without a transpose copy.  bias (bf16) element (b, h, i, j) is at
 * bias[b*bias_s[0] + h*bias_s[1] + i*bias_s[2] + j*bias_s[3]].
 * lse: fp32 [B, H, L] natural-log log-sum-exp of s (for the backward).
 * QK^T and PV run on tcgen05 (bf16 -> fp32 TMEM accumulators); c <= 64.        */
typedef struct EvoAttnDesc {
  const void* q; const void* k; const void* v; const void* g;
  int64_t q_sb, q_sl, k_sb, k_sl, v_sb, v_sl, g_sb, g_sl;
  const void* bias; int64_t bias_s[4];
  void* o_gated; int64_t o_sb, o_sl;
  void* o_raw; int64_t r_sb, r_sl;
  float* lse;
  int64_t B, L;
  int H, c;
  float scale;
  int flags;   /* EVO_ATTN_* kernel-selection hints (0 = automatic); per call, no global state */
} EvoAttnDesc;
/* Kernel selection is automatic: sequences with L >= 4096 and a per-key (or no) bias take
 * the warp-specialised forward (attention_ws.cu: 1 CTA/SM, loader warp, per-warpgroup MMA
 * warps, two softmax warpgroups), everything else the persistent flash kernel; a full
 * bias is staged through shared memory when its rows are 16-byte aligned.  Every
 * variant computes the same function; the flags force one for tests and A/B timing. */
enum {
  EVO_ATTN_FORCE_WS = 1,        /* warp-specialised forward at any L (any bias) */
  EVO_ATTN_FORCE_FLASH = 2,     /* persistent flash forward at any L */
  EVO_ATTN_NO_BIAS_SMEM = 4     /* full bias read from global memory, not staged in smem */
};
int evo_gated_attention_fwd(const EvoAttnDesc* d, void* stream);

/* Backward of the same op (flash-style: P is recomputed from q, k, bias and lse).
 * Inputs: the forward descriptor (q,k,v,g,bias,o_raw,lse) plus dout (gradient of
 * o_gated, strides like o_gated).  Outputs (bf16, strides like q/k/v/g): dq, dk, dv,
 * dg (gradient of the gate PRE-activation).  dbias is fp32 and ACCUMULATED at
 * dbias[b*s[0] + h*s[1] + i*s[2] + j*s[3]]; a zero stride reduces over that axis
 * (msa_row sums over sequences: s[0] = 0; per-key pair bias: s[2] = 0).
 * workspace: device scratch of evo_gated_attention_bwd_workspace(B, L, H, c, batch_reduced)
 * bytes, batch_reduced = (bias given and dbias_s[0] == 0 and dbias_s[2] != 0). */
typedef struct EvoAttnBwdDesc {
  EvoAttnDesc f;
  const void* dout; int64_t do_sb, do_sl;
  void* dq; void* dk; void* dv; void* dg;
  int64_t dq_sb, dq_sl, dk_sb, dk_sl, dv_sb, dv_sl, dg_sb, dg_sl;
  float* dbias; int64_t dbias_s[4];
  void* workspace; int64_t workspace_bytes;
} EvoAttnBwdDesc;
int64_t evo_gated_attention_bwd_workspace(int64_t B, int64_t L, int H, int c, int bias_batch_reduced);
int evo_gated_attention_bwd(const EvoAttnBwdDesc* d, void* stream);

/* ------------------------------------------------------------------ batched GEMM (tcgen05)
 * C[b] = alpha * A[b] . B[b]^T + beta * C[b]   with A:[M,K], B:[N,K], C:[M,N].
 * The dense contractions of the block run through this: the triangle einsums
 * (evoformer.py:276, 283) and the outer-product contraction (evoformer.py:253),
 * forward and backward.  Matrix element (b, i0, i1) lives at
 *   ptr[b*batch_stride + sum_d ((i_d / split[d]) * stride_hi[d] + (i_d % split[d]) * stride_lo[d])]
 * which expresses rank-major gathered layouts (DAP all-gather outputs) and the
 * [i][j][p][q] OPM layout without packing.  A and B must each be contiguous along
 * M/N (MN-major) or K (K-major) in runs of 8 (bf16).  C is bf16 or fp32.         */
typedef struct EvoMat {
  void* ptr;
  int dtype;
  int64_t batch_stride;
  int64_t split[2];
  int64_t stride_hi[2];
  int64_t stride_lo[2];
} EvoMat;
int evo_bgemm(const EvoMat* A, const EvoMat* B, const EvoMat* C,
              int64_t batch, int64_t M, int64_t N, int64_t K,
              float alpha, float beta, void* stream);
/* Same with a workspace enabling split-K when the output tiles cannot fill the
 * GPU and K is long (the OPM backward contractions, K = N_r * p): fp32 partials in
 * workspace, then a reduction applying alpha/beta and C's addressing.
 * evo_bgemm_workspace() returns the bytes needed (0 = no split chosen). */
int64_t evo_bgemm_workspace(int64_t batch, int64_t M, int64_t N, int64_t K);
int evo_bgemm_ws(const EvoMat* A, const EvoMat* B, const EvoMat* C,
                 int64_t batch, int64_t M, int64_t N, int64_t K,
                 float alpha, float beta, void* workspace, int64_t workspace_bytes, void* stream);

/* Weight gradient of a projection: dW[M][N] (fp32, row stride ldw) += X^T dY, X bf16 [rows][M]
 * (row stride ldx), dY bf16 [rows][N] (ldy); K = rows.  tcgen05, MN-major TMA operands, split-K
 * with fp32 partials in workspace (evo_wgrad_workspace() bytes; 0 = no split) reduced in a fixed
 * order (deterministic).  Replaces the weight-gradient products of every projection of the block
 * (the reference has no backward; these are the transposes of evoformer.py:183-195, 239-240,
 * 246-247, 255, 260-264, 270). */
int64_t evo_wgrad_workspace(int64_t rows, int64_t M, int64_t N);
int evo_wgrad(const void* x, int64_t ldx, const void* dy, int64_t ldy, float* dw, int64_t ldw, int64_t rows,
              int64_t M, int64_t N, void* workspace, int64_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------ fused OuterProductMean
 * outer_product_mean (evoformer.py:243-255) after its projections: with
 *   o[i,j,p,q] = alpha * sum_s a[s,i,p] b[s,j,q]     (alpha = 1/N_s, evoformer.py:253)
 * writes y[(i*J + j)*y_ld + c] = sum_{p,q} o[i,j,p,q] W_o[p*P+q, c] (bf16, before the output bias
 * and the residual add of evoformer.py:255/318) as two back-to-back tcgen05 GEMMs per tile: o
 * stays on chip.  o_save (may be NULL): also store o, bf16 [I][J][P][P] (the backward's operand).
 * a_t: a as bf16 [I][P][N_s] (sequence-contiguous, evo_opm_transpose), b_t: b as [J][P][N_s]
 * (a DAP all-gather of per-rank [J/N][P][N_s] blocks is already in this layout).
 * W_o bf16 [P*P][Hz] row-major.  Supported extents: evo_opm_fused_supported() != 0 (P = 32,
 * N_s <= 128 and a multiple of 8, I % 32 == 0, J % 8 == 0, Hz in {32, 64, 128}); the caller
 * composes evo_bgemm + a projection GEMM otherwise.
 * Replaces: the einsum + reshape + matmul of outer_product_mean, evoformer.py:251-255. */
int evo_opm_fused_supported(int64_t I, int64_t J, int64_t S, int64_t P, int64_t Hz);
int evo_opm_fused_fwd(const void* a_t, const void* b_t, const void* w_o, void* y, int64_t y_ld, void* o_save,
                      int64_t I, int64_t J, int64_t S, int64_t P, int64_t Hz, float alpha, void* stream);
/* Backward of the fused OPM for one factor, without materialising do = dy W_o^T:
 *   role 0:  da[s,i,p] = alpha sum_{j,q} b[s,j,q] do[i,j,p,q]    (x = i, y = j, other_t = b_t [J][P][N_s])
 *   role 1:  db[s,j,q] = alpha sum_{i,p} a[s,i,p] do[i,j,p,q]    (x = j, y = i, other_t = a_t [I][P][N_s])
 * with do[i,j,p,q] = sum_c dy[(i*J + j)*ldy + c] W_o[p*P+q, c] (X = extent of x, Y = of y).  Output
 * element (s, x, p) at out + s*o_ss + (x / x_split)*o_sr + (x % x_split)*o_sx + p, bf16 (out_f32 = 0)
 * or fp32 (the rank-major partial a DAP reduce-scatter takes).  Two tcgen05 GEMMs per 128-pair step
 * (dy W^T into TMEM, converted to bf16 in shared memory, times the other factor) accumulating in
 * TMEM; fp32 partials over y splits in workspace (evo_opm_bwd_workspace(X) bytes) summed in order.
 * Supported extents: evo_opm_bwd_supported(I, J, N_s, P, Hz) (P = 32, N_s <= 128, I, J % 32 == 0,
 * Hz in {64, 128}).  Replaces the backward of the einsum + matmul of evoformer.py:251-255. */
int evo_opm_bwd_supported(int64_t I, int64_t J, int64_t S, int64_t P, int64_t Hz);
int64_t evo_opm_bwd_workspace(int64_t X);
int evo_opm_bwd_factor(int role, const void* dy, int64_t ldy, const void* w_o, const void* other_t,
                       int64_t X, int64_t Y, int64_t S, int64_t P, int64_t Hz, float alpha, void* out, int out_f32,
                       int64_t o_ss, int64_t o_sr, int64_t o_sx, int64_t x_split, void* workspace,
                       int64_t workspace_bytes, void* stream);
/* The OPM projections [N_s*R][ld] (rows (s, r); channels col0 .. col0+P, and col0+P .. col0+2P
 * when out_b != NULL) to the sequence-contiguous layout out[r][p][s] the fused kernel reads (bf16). */
int evo_opm_transpose(const void* x, int64_t ld, int64_t col0, int64_t S, int64_t R, int64_t P, void* out_a,
                      void* out_b, void* stream);

/* ------------------------------------------------------------------ triangle gating
 * _triangle_projections epilogue (evoformer.py:260-264) for the merged projection
 * Y = LN(z) @ [W_g | W_a_sig | W_a_lin | W_b_sig | W_b_lin] + bias, Y bf16
 * row-major [rows = n0*n1, hz + 4p]:
 *   a[h][r] = sigmoid(Y[r, hz+h]) * Y[r, hz+p+h],  b[h][r] = sigmoid(Y[r, hz+2p+h]) * Y[r, hz+3p+h]
 * written CHANNEL-MAJOR (a_cm[h*rows + r]) so that the einsum is a plain batched
 * GEMM over h.  The g gate stays in Y (sigmoid applied by evo_gated_residual_fwd). */
int evo_tri_gate_fwd(const void* y, int64_t rows, int hz, int p, void* a_cm, void* b_cm, void* stream);
/* dY[:, hz:] from da_cm, db_cm (channel-major fp32 or bf16); writes bf16 dY row-major;
 * dsum (fp32 [4p], may be NULL): += column sums of dY[:, hz:] in fp32 (the bias gradient of
 * the a/b projections, before the bf16 rounding of dY) */
int evo_tri_gate_bwd(const void* y, const void* da_cm, const void* db_cm, int d_dtype,
                     int64_t rows, int hz, int p, void* dy, float* dsum, void* stream);

/* ------------------------------------------------------------------ residual epilogues
 * out = res + gate(gp) * (y + bias), gate(gp) = sigmoid(gp) or 1 when gp == NULL.
 * Covers every residual add of evoformer_block (evoformer.py:316-324) with the
 * output bias and, for the triangle updates, the g gate (evoformer.py:270).
 * y/gp/out rows have their own row strides (elements); cols contiguous.           */
int evo_gated_residual_fwd(const void* res, const void* y, int64_t y_rs, const float* bias,
                           const void* gp, int64_t gp_rs, void* out, int dtype,
                           int64_t rows, int64_t cols, void* stream);
/* dy = dout * gate, dgp = dout * (y+bias) * gate*(1-gate) (if gp), dbias += sum_r dy (fp32),
 * dgp_sum += sum_r dgp (fp32, may be NULL: the gate projection's bias gradient). */
int evo_gated_residual_bwd(const void* dout, const void* y, int64_t y_rs, const float* bias,
                           const void* gp, int64_t gp_rs, void* dy, void* dgp, int64_t dgp_rs,
                           float* dbias, float* dgp_sum, int dtype, int64_t rows, int64_t cols, void* stream);

/* out[r*out_rs + c] = act(gate[r*gate_rs + c]) * (y[r*y_rs + c] + bias[c]); act 0 = identity,
 * 1 = sigmoid, 2 = ReLU; gate NULL -> 1, y NULL -> (y + bias) = 1, bias may be NULL.
 * The reference-API helpers _triangle_projections / _triangle_finish (evoformer.py:258-270)
 * and engine.sigmoid_raw / relu_raw (engine.py:220-225); any cols, any row strides.   */
int evo_gate_mul_fwd(const void* gate, int64_t gate_rs, int gate_act, const void* y, int64_t y_rs,
                     const float* bias, void* out, int64_t out_rs, int dtype, int64_t rows, int64_t cols,
                     void* stream);

/* out[c] += sum_r x[r*ld + c]  (fp32 out; bias gradients of the projection GEMMs) */
int evo_colsum(const void* x, int dtype, int64_t ld, int64_t rows, int64_t cols, float* out, void* stream);

/* h = act(y + bias) in place (act 0 = identity, 1 = ReLU: transition, evoformer.py:239) */
int evo_bias_act_fwd(void* y, const float* bias, int64_t rows, int64_t cols, int act, int dtype, void* stream);
/* dy = dh * (h > 0) (act 1) and dbias += sum_r dy; h is the activated output */
int evo_bias_act_bwd(const void* dh, const void* h, void* dy, float* dbias, int64_t rows, int64_t cols,
                     int act, int dtype, void* stream);

/* number of non-finite elements of x (fp32 counter, accumulated) - the GPU twin of
 * softmax_raw's DomainError check (engine.py:186-187) */
int evo_count_nonfinite(const void* x, int dtype, int64_t n, unsigned int* counter, void* stream);
/* Per-key (pair) bias gradient into the bias columns of the fused qkv gradient (the per-key
 * bias is the 4 extra projection columns of _pair_bias_fn, evoformer.py:287-292):
 * dst[b*dst_sb + l*dst_sl + h] = bf16(dbias[(b*nh + h)*L + l]) for h < nh, 0 for nh <= h < cols. */
int evo_key_bias_grad_cols(const float* dbias, int64_t B, int nh, int64_t L, void* dst, int64_t dst_sb,
                           int64_t dst_sl, int cols, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* EVO_H_ */
