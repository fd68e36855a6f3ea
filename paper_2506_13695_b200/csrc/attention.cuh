// Segmented multi-head attention: for each batch item b, query rows
// [q.start(b), +q.len(b)) attend (non-causal, softmax(QK^T/sqrt(dh))V) to key
// rows [k.start(b), +k.len(b)) and write rows [o.start(b), +q.len(b)).
// Covers every non-causal mha_core use of the hot path (tape.cpp:822-905):
// encoder self-attention (policy.cpp:261), lifelong QFormer cross-attention
// with ragged key counts (nn.cpp:97-100) and decoder cross-attention of beam
// rows to the per-user encoder K/V cache (policy.cpp:284).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace orx {

struct Seg {
  const int32_t* start = nullptr;  // device [B] or null -> b * stride
  const int32_t* len = nullptr;    // device [B] or null -> fixed_len
  int stride = 0;
  int fixed_len = 0;
};

// tcgen05 flash attention (bf16, dh 64 / 128; attention_tc.cu). K is row
// major (keys x heads*dh at column k_col0); V is given transposed per
// (segment user, head): Vt rows ((vt_user[b] or b) * heads + h) * dh + c,
// columns = key position within the segment (vt_ld >= segment length, the
// padding columns finite). Q / K are buffer bases with head 0 at q_col0 / k_col0.
struct FmhaArgs {
  int B = 0, max_q = 0, heads = 0, dh = 0;
  const void* Q = nullptr;
  long long q_rows = 0;
  int ldq = 0, q_col0 = 0;
  const void* K = nullptr;
  long long k_rows = 0;
  int ldk = 0, k_col0 = 0;
  const void* Vt = nullptr;
  long long vt_rows = 0, vt_cols = 0;
  int vt_ld = 0;
  const int32_t* vt_user = nullptr;
  void* O = nullptr;
  int ldo = 0;
  Seg q, k, o;
  double flops = 0.0;
  int prof_cat = 2;    // PROF_ATTN; the decoder's cross attention reports as PROF_XATTN
  double bytes = 0.0;  // algorithmic HBM bytes (cached K / V^T + Q + O) for the HBM-bound uses
};
bool fmha_supported(int dh);
void launch_fmha_tc(const FmhaArgs& a, cudaStream_t s);

template <class T>
void launch_attention(int B, int max_q, int heads, int dh, const T* Q, int ldq, const T* K, int ldk, const T* V,
                      int ldv, T* O, int ldo, Seg q, Seg k, Seg o, cudaStream_t s, double flops = 0.0);

}  // namespace orx
