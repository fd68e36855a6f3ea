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

template <class T>
void launch_attention(int B, int max_q, int heads, int dh, const T* Q, int ldq, const T* K, int ldk, const T* V,
                      int ldv, T* O, int ldo, Seg q, Seg k, Seg o, cudaStream_t s, double flops = 0.0);

}  // namespace orx
