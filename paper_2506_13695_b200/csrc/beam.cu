#include <cfloat>
#include <stdexcept>

#include "beam.cuh"
#include "common.cuh"
#include "gemm.cuh"

namespace orx {

namespace {

__device__ __forceinline__ uint32_t ord_f32(float f) {
  uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unord_f32(uint32_t o) {
  uint32_t b = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
  return __uint_as_float(b);
}

// Block-wide radix select: returns tau such that exactly k of the n (unique)
// keys satisfy key >= tau. MSB-first 8-bit digits, early exit once the
// boundary bucket is taken whole.
template <int NT, class Get>
__device__ uint64_t block_kth_largest(int n, int k, Get get, uint32_t* hist, uint32_t* bc) {
  if (n <= k) return 0;
  uint64_t prefix = 0, mask = 0;
  int krem = k;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += NT) hist[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += NT) {
      uint64_t key = get(i);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      // lane handles bins [248 - 8*lane, 255 - 8*lane], i.e. lane 0 = top bins
      uint32_t c[8], tot = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = hist[255 - 8 * lane - j];
        tot += c[j];
      }
      uint32_t incl = tot;  // inclusive prefix over lanes (from the top)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      uint32_t above = incl - tot;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (above < static_cast<uint32_t>(krem) && above + c[j] >= static_cast<uint32_t>(krem)) {
          bc[0] = 255 - 8 * lane - j;
          bc[1] = above;
          bc[2] = c[j];
        }
        above += c[j];
      }
    }
    __syncthreads();
    const uint32_t dgt = bc[0], above = bc[1], cnt = bc[2];
    __syncthreads();
    prefix |= static_cast<uint64_t>(dgt) << shift;
    mask |= static_cast<uint64_t>(255u) << shift;
    krem -= static_cast<int>(above);
    if (static_cast<int>(cnt) == krem) break;
  }
  return prefix;
}

// Bitonic sort (descending) of n <= NP keys in shared memory, padded with 0.
template <int NP, int NT>
__device__ void block_sort_desc(uint64_t* a, int n) {
  for (int i = n + threadIdx.x; i < NP; i += NT) a[i] = 0;
  __syncthreads();
  for (int size = 2; size <= NP; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < NP / 2; i += NT) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool desc = ((lo & size) == 0);
        uint64_t x = a[lo], y = a[hi];
        if ((x < y) == desc) {
          a[lo] = y;
          a[hi] = x;
        }
      }
      __syncthreads();
    }
  }
}

constexpr int kRowThreads = 256;

__global__ void __launch_bounds__(kRowThreads) row_topk_kernel(int V, int k_sel, const float* __restrict__ logits,
                                                               const float* __restrict__ pscore,
                                                               const int32_t* __restrict__ plex,
                                                               float* __restrict__ lse_out,
                                                               uint64_t* __restrict__ cand) {
  extern __shared__ uint64_t keys[];  // [V]
  __shared__ uint32_t hist[256];
  __shared__ uint32_t bc[4];
  __shared__ float red[kRowThreads / 32];
  __shared__ uint32_t counter;
  const int row = blockIdx.x;
  const float* lg = logits + (size_t)row * V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // log-softmax normaliser (max-subtracted, generation.cpp:10-20)
  float mx = -FLT_MAX;
  for (int i = threadIdx.x; i < V; i += kRowThreads) mx = fmaxf(mx, lg[i]);
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < kRowThreads / 32; ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float sum = 0.f;
  for (int i = threadIdx.x; i < V; i += kRowThreads) sum += __expf(lg[i] - mx);
  sum = warp_sum(sum);
  if (lane == 0) red[warp] = sum;
  __syncthreads();
  sum = 0.f;
  for (int w = 0; w < kRowThreads / 32; ++w) sum += red[w];
  const float lse = mx + logf(sum);
  const float ps = pscore[row];
  const uint32_t lbase = static_cast<uint32_t>(plex[row]) * static_cast<uint32_t>(V);
  for (int i = threadIdx.x; i < V; i += kRowThreads) {
    float sc = ps + (lg[i] - lse);
    keys[i] = (static_cast<uint64_t>(ord_f32(sc)) << 32) | (0xFFFFFFFFu - (lbase + static_cast<uint32_t>(i)));
  }
  if (threadIdx.x == 0) {
    lse_out[row] = lse;
    counter = 0;
  }
  __syncthreads();
  uint64_t tau = block_kth_largest<kRowThreads>(V, k_sel, [&](int i) { return keys[i]; }, hist, bc);
  __syncthreads();
  uint64_t* out = cand + (size_t)row * k_sel;
  for (int i = threadIdx.x; i < V; i += kRowThreads) {
    uint64_t key = keys[i];
    if (key >= tau) {
      uint32_t pos = atomicAdd(&counter, 1u);
      if (pos < static_cast<uint32_t>(k_sel)) out[pos] = key;
    }
  }
}

// Fast path (V <= 8192, k_sel < V, k_sel <= 1024): the row stays in registers
// (32 per thread). Bisection on the fp32 score finds a threshold whose
// candidate count lies in [k_sel, cap]; the candidates are sorted in shared
// memory (bitonic) and the first k_sel keys written. Exact: the key order
// is the same as row_topk_kernel's, so ties at the threshold are all kept
// and resolved by the lexicographic part of the key. Rows where bisection
// cannot isolate such a threshold (massive exact ties) take the radix path.
constexpr int kTopkPer = 32;
constexpr int kTopkCap = 2048;

__device__ __forceinline__ float block_reduce_sum256(float v, float* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int w = 0; w < kRowThreads / 32; ++w) t += red[w];
  return t;
}
__device__ __forceinline__ float block_reduce_max256(float v, float* red) {
  v = warp_max(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float t = -FLT_MAX;
#pragma unroll
  for (int w = 0; w < kRowThreads / 32; ++w) t = fmaxf(t, red[w]);
  return t;
}

__global__ void __launch_bounds__(kRowThreads) row_topk_fast_kernel(int V, int k_sel, const float* __restrict__ logits,
                                                                    const float* __restrict__ pscore,
                                                                    const int32_t* __restrict__ plex,
                                                                    float* __restrict__ lse_out,
                                                                    uint64_t* __restrict__ cand) {
  __shared__ uint64_t buf[kTopkCap];
  __shared__ float red[kRowThreads / 32];
  __shared__ uint32_t hist[256];
  __shared__ uint32_t bc[4];
  __shared__ uint32_t counter;
  const int row = blockIdx.x, tid = threadIdx.x;
  const float* lg = logits + (size_t)row * V;
  float v[kTopkPer];
  float mx = -FLT_MAX;
#pragma unroll
  for (int j = 0; j < kTopkPer; ++j) {
    const int i = tid + kRowThreads * j;
    v[j] = i < V ? __ldg(lg + i) : -FLT_MAX;
    mx = fmaxf(mx, v[j]);
  }
  mx = block_reduce_max256(mx, red);
  float se = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int j = 0; j < kTopkPer; ++j)
    if (tid + kRowThreads * j < V) {
      se += __expf(v[j] - mx);
      s1 += v[j] - mx;
      s2 += (v[j] - mx) * (v[j] - mx);
    }
  se = block_reduce_sum256(se, red);
  s1 = block_reduce_sum256(s1, red);
  s2 = block_reduce_sum256(s2, red);
  const float lse = mx + logf(se);  // log-softmax normaliser (generation.cpp:10-20)
  const float ps = pscore[row];
  // scores (the ranking quantity of the candidate key)
  float smin = FLT_MAX;
#pragma unroll
  for (int j = 0; j < kTopkPer; ++j) {
    v[j] = tid + kRowThreads * j < V ? ps + (v[j] - lse) : -FLT_MAX;
    if (tid + kRowThreads * j < V) smin = fminf(smin, v[j]);
  }
  smin = -block_reduce_max256(-smin, red);
  const float smax = ps + (mx - lse);
  // bisection: count(score >= tau) in [k_sel, cap]
  const int cap = min(kTopkCap, max(2 * k_sel, 256));
  float lo = smin, hi = smax;  // count(lo) = V >= k_sel; count(hi) >= 1
  const float mean = s1 / V, sd = sqrtf(fmaxf(s2 / V - mean * mean, 0.f));
  // first probe: normal upper quantile of the top (1.25 k_sel) / V fraction
  // (Abramowitz-Stegun 26.2.23), scores assumed ~normal
  const float pf = fminf(0.5f, 1.25f * k_sel / V);
  const float t = sqrtf(-2.f * logf(pf));
  const float z = t - (2.515517f + 0.802853f * t + 0.010328f * t * t) /
                          (1.f + 1.432788f * t + 0.189269f * t * t + 0.001308f * t * t * t);
  float tau = smax + mean + z * sd;
  tau = fminf(fmaxf(tau, lo), hi);
  int count = -1;
  bool found = false;
  for (int it = 0; it < 48; ++it) {
    int c = 0;
#pragma unroll
    for (int j = 0; j < kTopkPer; ++j) c += v[j] >= tau;
    count = static_cast<int>(block_reduce_sum256(static_cast<float>(c), red));
    if (count >= k_sel && count <= cap) {
      found = true;
      break;
    }
    if (count < k_sel) hi = tau;
    else lo = tau;
    const float nt = 0.5f * (lo + hi);
    if (nt == lo || nt == hi) break;
    tau = nt;
  }
  if (tid == 0) {
    lse_out[row] = lse;
    counter = 0;
  }
  const uint32_t lbase = static_cast<uint32_t>(plex[row]) * static_cast<uint32_t>(V);
  uint64_t* out = cand + (size_t)row * k_sel;
  if (found) {
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kTopkPer; ++j) {
      const int i = tid + kRowThreads * j;
      const bool take = v[j] >= tau;
      const unsigned m = __ballot_sync(0xffffffffu, take);
      uint32_t base = 0;
      if ((tid & 31) == 0 && m) base = atomicAdd(&counter, __popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (take)
        buf[base + __popc(m & ((1u << (tid & 31)) - 1u))] =
            (static_cast<uint64_t>(ord_f32(v[j])) << 32) | (0xFFFFFFFFu - (lbase + static_cast<uint32_t>(i)));
    }
    __syncthreads();
    int np = 256;
    while (np < count) np <<= 1;
    for (int i = count + tid; i < np; i += kRowThreads) buf[i] = 0;
    __syncthreads();
    for (int size = 2; size <= np; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = tid; i < np / 2; i += kRowThreads) {
          const int lo_i = 2 * i - (i & (stride - 1));
          const int hi_i = lo_i + stride;
          const bool desc = (lo_i & size) == 0;
          const uint64_t x = buf[lo_i], y = buf[hi_i];
          if ((x < y) == desc) {
            buf[lo_i] = y;
            buf[hi_i] = x;
          }
        }
        __syncthreads();
      }
    }
    for (int i = tid; i < k_sel; i += kRowThreads) out[i] = buf[i];
    return;
  }
  // fallback: radix select over the keys (rare: massive exact ties)
  __syncthreads();
  auto key_of = [&](int i) -> uint64_t {
    const float sc = ps + (__ldg(lg + i) - lse);
    return (static_cast<uint64_t>(ord_f32(sc)) << 32) | (0xFFFFFFFFu - (lbase + static_cast<uint32_t>(i)));
  };
  uint64_t thr = block_kth_largest<kRowThreads>(V, k_sel, key_of, hist, bc);
  __syncthreads();
  for (int i = tid; i < V; i += kRowThreads) {
    const uint64_t key = key_of(i);
    if (key >= thr) {
      uint32_t pos = atomicAdd(&counter, 1u);
      if (pos < static_cast<uint32_t>(k_sel)) out[pos] = key;
    }
  }
}

constexpr int kMergeThreads = 512;
constexpr int kMaxBeam = 1024;

__global__ void __launch_bounds__(kMergeThreads) beam_merge_kernel(int n_live, int k_sel, int n_new, int V, int L,
                                                                   int step, const uint64_t* __restrict__ cand,
                                                                   const float* __restrict__ logits,
                                                                   const float* __restrict__ lse, BeamState cur,
                                                                   BeamState nxt) {
  __shared__ uint64_t sel[kMaxBeam];
  __shared__ uint64_t lex[kMaxBeam];
  __shared__ uint32_t hist[256];
  __shared__ uint32_t bc[4];
  __shared__ uint32_t counter;
  const int u = blockIdx.x;
  const int n = n_live * k_sel;
  const uint64_t* c = cand + (size_t)u * n;
  if (threadIdx.x == 0) counter = 0;
  __syncthreads();
  uint64_t tau = block_kth_largest<kMergeThreads>(n, n_new, [&](int i) { return c[i]; }, hist, bc);
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += kMergeThreads) {
    uint64_t key = c[i];
    if (key >= tau) {
      uint32_t pos = atomicAdd(&counter, 1u);
      if (pos < static_cast<uint32_t>(n_new)) sel[pos] = key;
    }
  }
  __syncthreads();
  block_sort_desc<kMaxBeam, kMergeThreads>(sel, n_new);
  // beam b (rank order): decode parent lexrank + code, build next state
  for (int b = threadIdx.x; b < n_new; b += kMergeThreads) {
    const uint64_t key = sel[b];
    const uint32_t low = 0xFFFFFFFFu - static_cast<uint32_t>(key & 0xFFFFFFFFu);
    const int plr = static_cast<int>(low / static_cast<uint32_t>(V));
    const int code = static_cast<int>(low % static_cast<uint32_t>(V));
    const int pb = cur.lex2beam[(size_t)u * n_live + plr];
    const int prow = u * n_live + pb;
    const int nrow = u * n_new + b;
    for (int j = 0; j < step; ++j) {
      nxt.codes[(size_t)nrow * L + j] = cur.codes[(size_t)prow * L + j];
      nxt.anc[(size_t)nrow * L + j] = cur.anc[(size_t)prow * L + j];
    }
    nxt.codes[(size_t)nrow * L + step] = code;
    nxt.anc[(size_t)nrow * L + step] = prow;
    nxt.score[nrow] = unord_f32(static_cast<uint32_t>(key >> 32));
    nxt.score64[nrow] = cur.score64[prow] + (static_cast<double>(logits[(size_t)prow * V + code]) -
                                             static_cast<double>(lse[prow]));
    lex[b] = (static_cast<uint64_t>(low) << 32) | static_cast<uint32_t>(b);
  }
  __syncthreads();
  // lexicographic rank of the new prefixes = ascending (plr, code) = ascending low
  for (int i = n_new + threadIdx.x; i < kMaxBeam; i += kMergeThreads) lex[i] = ~0ull;
  __syncthreads();
  // ascending sort: negate by sorting descending of the complement
  for (int i = threadIdx.x; i < kMaxBeam; i += kMergeThreads) lex[i] = ~lex[i];
  __syncthreads();
  block_sort_desc<kMaxBeam, kMergeThreads>(lex, kMaxBeam);
  for (int r = threadIdx.x; r < n_new; r += kMergeThreads) {
    const int b = static_cast<int>(static_cast<uint32_t>(~lex[r]));
    nxt.lexrank[u * n_new + b] = r;
    nxt.lex2beam[(size_t)u * n_new + r] = b;
  }
}

__global__ void beam_init_kernel(int users, BeamState st) {
  int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= users) return;
  st.score[u] = 0.f;
  st.score64[u] = 0.0;
  st.lexrank[u] = 0;
  st.lex2beam[u] = 0;
}

}  // namespace

void launch_row_topk(int rows, int V, int k_sel, const float* logits, const float* parent_score,
                     const int32_t* parent_lexrank, float* lse, uint64_t* cand, cudaStream_t s) {
  if (rows <= 0) return;
  size_t smem = static_cast<size_t>(V) * 8;
  static size_t set = 0;
  if (smem > 48 * 1024 && smem > set) {
    cudaFuncSetAttribute(row_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    set = smem;
  }
  ProfScope ps(PROF_BEAM, s, 0.0, double(rows) * V * 4);
  if (V <= kRowThreads * kTopkPer && k_sel < V && k_sel <= 1024) {
    row_topk_fast_kernel<<<rows, kRowThreads, 0, s>>>(V, k_sel, logits, parent_score, parent_lexrank, lse, cand);
    ++launch_counter();
    return;
  }
  row_topk_kernel<<<rows, kRowThreads, smem, s>>>(V, k_sel, logits, parent_score, parent_lexrank, lse, cand);
  ++launch_counter();
}

void launch_beam_merge(int users, int n_live, int k_sel, int n_new, int V, int L, int step, const uint64_t* cand,
                       const float* logits, const float* lse, const BeamState& cur, BeamState& nxt,
                       cudaStream_t s) {
  if (n_new > kMaxBeam) throw std::invalid_argument("beam width above 1024 is not supported");
  ProfScope ps(PROF_BEAM, s, 0.0, 0.0);
  beam_merge_kernel<<<users, kMergeThreads, 0, s>>>(n_live, k_sel, n_new, V, L, step, cand, logits, lse, cur, nxt);
  ++launch_counter();
}

void launch_beam_init(int users, BeamState& st, cudaStream_t s) {
  beam_init_kernel<<<(users + 127) / 128, 128, 0, s>>>(users, st);
  ++launch_counter();
}

}  // namespace orx
