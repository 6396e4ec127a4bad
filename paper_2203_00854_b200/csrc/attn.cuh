// Shared parameter block of the attention forward / backward kernels.
#pragma once
#include "common.cuh"

namespace evo {

struct AttnParams {
  const bf16 *q, *k, *v, *g, *bias;
  int64_t q_sb, q_sl, k_sb, k_sl, v_sb, v_sl, g_sb, g_sl;
  int64_t bs0, bs1, bs2, bs3;
  bf16 *og, *orw;
  int64_t o_sb, o_sl, r_sb, r_sl;
  float* lse;
  int L, H, c;
  float scale_log2;
  int bias_vec;  // full-bias rows are contiguous and 16-byte aligned
};

// validate an EvoAttnDesc (include/evo.h) and convert it
int attn_params_from_desc(const EvoAttnDesc* d, AttnParams& p);

}  // namespace evo
