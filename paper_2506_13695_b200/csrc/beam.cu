#include <algorithm>
#include <cfloat>
#include <climits>
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

// Bitonic sort (descending) of n <= NP keys in shared memory, padded with 0
// up to the next power of two (a[] must hold that many).
template <int NP, int NT>
__device__ void block_sort_desc(uint64_t* a, int n) {
  int np = 2;
  while (np < n) np <<= 1;
  if (np > NP) np = NP;
  for (int i = n + threadIdx.x; i < np; i += NT) a[i] = 0;
  __syncthreads();
  for (int size = 2; size <= np; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < np / 2; i += NT) {
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
                                                               uint64_t* __restrict__ cand,
                                                               const int32_t* __restrict__ row_list) {
  pdl_begin();
  extern __shared__ uint64_t keys[];  // [V]
  __shared__ uint32_t hist[256];
  __shared__ uint32_t bc[4];
  __shared__ float red[kRowThreads / 32];
  __shared__ uint32_t counter;
  // row_list: [0] = n, [1..n] = rows (fallback rows of row_topk_warp_kernel), grid-stride
  const int n_rows = row_list ? row_list[0] : static_cast<int>(gridDim.x);
  for (int li = blockIdx.x; li < n_rows; li += gridDim.x) {
  const int row = row_list ? row_list[1 + li] : li;
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
  __syncthreads();
  }
}

// Fast path: one warp per row, two streaming passes over the logits.
//   pass 1: max, mean and variance of the row's logits
//   pass 2: sum of exp (the log-softmax normaliser, generation.cpp:10-20) and
//           every logit >= tx appended to its lane's 32-slot shared-memory
//           segment, tx = the normal-quantile guess for ~2.5 k_sel survivors
//           (retried with a moved tx if fewer than k_sel survive or a lane
//           segment overflows)
//   select: the survivors (<= 1024, 32 per lane in registers) are scored
//           (parent + logit - lse) and bisected with 8 thresholds per step
//           until exactly k_sel scores are >= tau; their keys are written.
// Selecting by logit then by score is exact because the fp32 score is a
// monotone function of the logit; the one case it cannot decide (a rejected
// logit whose rounded score equals a selected one, or scores tied across the
// k-th position) sends the row to the block radix-select kernel, so the set
// is always identical to row_topk_kernel's. Outputs are unordered.
constexpr int kProbes = 8;
__device__ unsigned long long g_topk_fallback_rows = 0;  // rows sent to the radix path (test hook)

__device__ __forceinline__ float normal_upper_quantile(float p) {  // Abramowitz-Stegun 26.2.23
  p = fminf(0.5f, fmaxf(p, 1e-7f));
  const float t = sqrtf(-2.f * logf(p));
  return t - (2.515517f + 0.802853f * t + 0.010328f * t * t) /
                 (1.f + 1.432788f * t + 0.189269f * t * t + 0.001308f * t * t * t);
}

template <int kLaneSlots, int kWarpRows = 128 / kLaneSlots>  // rows (warps) per block: 33 KB smem
__global__ void __launch_bounds__(32 * kWarpRows) row_topk_warp_kernel(int rows, int V, int k_sel,
                                                                       const float* __restrict__ logits,
                                                                       const float* __restrict__ pscore,
                                                                       const int32_t* __restrict__ plex,
                                                                       float* __restrict__ lse_out,
                                                                       uint64_t* __restrict__ cand,
                                                                       int32_t* __restrict__ fail) {
  pdl_begin();
  __shared__ float bx[kWarpRows][kLaneSlots * 32];
  __shared__ int32_t bi[kWarpRows][kLaneSlots * 32];
  __shared__ int32_t bn[kWarpRows][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int row = blockIdx.x * kWarpRows + w;
  if (row >= rows) return;
  const float* lg = logits + (size_t)row * V;
  const float4* lg4 = reinterpret_cast<const float4*>(lg);
  const int V4 = V >> 2;  // V % 4 == 0 (launch condition)
  // One streaming pass. The survivor threshold tx comes from the first 1024
  // logits (mean / spread estimate); the softmax sum is taken relative to that
  // sample's max (a second pass only if the true max is far above it); loads
  // are issued 8 deep per lane.
  constexpr int U8 = 8;
  float m0 = -FLT_MAX, s1 = 0.f, s2 = 0.f;
  const int nsamp = min(V4, 256);
  for (int i = lane; i < nsamp; i += 32) {
    const float4 x = __ldg(lg4 + i);
    m0 = fmaxf(m0, fmaxf(fmaxf(x.x, x.y), fmaxf(x.z, x.w)));
    s1 += (x.x + x.y) + (x.z + x.w);
    s2 += (x.x * x.x + x.y * x.y) + (x.z * x.z + x.w * x.w);
  }
  m0 = warp_max(m0);
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  const float mean = s1 / (4 * nsamp), sd = sqrtf(fmaxf(s2 / (4 * nsamp) - mean * mean, 0.f));
  // survivors: ~2.5 k_sel, but on average at most half of the slots per lane
  const float target = fminf(2.5f * k_sel, 16.f * kLaneSlots);
  float tx = mean + normal_upper_quantile(target / V) * sd;
  float* sx = bx[w] + lane * kLaneSlots;
  int32_t* si = bi[w] + lane * kLaneSlots;
  float se = 0.f, rej = -FLT_MAX, mx = -FLT_MAX;
  float2 se2 = make_float2(0.f, 0.f);
  const float2 l2e2 = make_float2(1.4426950408889634f, 1.4426950408889634f);
  const float2 nm2 = make_float2(-m0 * 1.4426950408889634f, -m0 * 1.4426950408889634f);
  int n = 0, total = 0;
  bool ok = false;
  for (int attempt = 0; attempt < 4; ++attempt) {
    n = 0;
    rej = -FLT_MAX;
    bool over = false;
    for (int i0 = lane; i0 < V4; i0 += 32 * U8) {
      float4 xb[U8];
#pragma unroll
      for (int u = 0; u < U8; ++u) xb[u] = i0 + 32 * u < V4 ? __ldg(lg4 + i0 + 32 * u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < U8; ++u) {
        const int i = i0 + 32 * u;
        if (i >= V4) continue;
        const float4 x = xb[u];
        if (attempt == 0) {  // packed: one FFMA2 per pair (log2 e and the sample max folded), SFU ex2, FADD2
          mx = fmaxf(mx, fmaxf(fmaxf(x.x, x.y), fmaxf(x.z, x.w)));
          const float2 t01 = ffma2(make_float2(x.x, x.y), l2e2, nm2), t23 = ffma2(make_float2(x.z, x.w), l2e2, nm2);
          se2 = fadd2(se2, make_float2(ex2_fast(t01.x), ex2_fast(t01.y)));
          se2 = fadd2(se2, make_float2(ex2_fast(t23.x), ex2_fast(t23.y)));
        }
        const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {  // branch-free append (predicated stores, no reconvergence per element)
          const bool take = xs[e] >= tx;
          const bool fits = n < kLaneSlots;
          if (take && fits) {
            sx[n] = xs[e];
            si[n] = 4 * i + e;
          }
          over |= take && !fits;
          n += take ? 1 : 0;
          rej = take ? rej : fmaxf(rej, xs[e]);
        }
      }
    }
    if (attempt == 0) mx = warp_max(mx);
    total = __reduce_add_sync(0xffffffffu, n);
    over = __any_sync(0xffffffffu, over);
    if (total >= k_sel && !over) {
      ok = true;
      break;
    }
    // too few survivors: lower tx; a lane overflowed: raise it
    tx = total < k_sel ? tx - 0.75f * sd : tx + 0.25f * sd;
    if (!(sd > 0.f)) break;
  }
  se = warp_sum(se2.x + se2.y);
  if (mx > m0 + 60.f) {  // the sample's max was far below the row's: exact sum in a second pass
    se = 0.f;
    for (int i = lane; i < V4; i += 32) {
      const float4 x = __ldg(lg4 + i);
      se += (__expf(x.x - mx) + __expf(x.y - mx)) + (__expf(x.z - mx) + __expf(x.w - mx));
    }
    se = warp_sum(se);
    m0 = mx;
  }
  const float lse = m0 + logf(se);
  const float ps = pscore[row];
  if (lane == 0) lse_out[row] = lse;
  uint64_t* out = cand + (size_t)row * k_sel;
  const uint32_t lbase = static_cast<uint32_t>(plex[row]) * static_cast<uint32_t>(V);
  if (ok) {
    bn[w][lane] = n;
    __syncwarp();
    // lane owns slots lane, lane + 32, ... of every lane segment j (conflict-free transposed read)
    constexpr int SPL = kLaneSlots / 32;
    float c[kLaneSlots];
#pragma unroll
    for (int j = 0; j < 32; ++j)
#pragma unroll
      for (int s2 = 0; s2 < SPL; ++s2)
        c[j * SPL + s2] =
            lane + 32 * s2 < bn[w][j] ? ps + (bx[w][j * kLaneSlots + 32 * s2 + lane] - lse) : -FLT_MAX;
    float lo = ps + (tx - lse), hi = ps + (mx - lse);  // count(>= lo) = total >= k_sel
    bool hi_open = true, found = total == k_sel;
    float tau = lo;
    for (int it = 0; it < 16 && !found; ++it) {
      float pr[kProbes];
#pragma unroll
      for (int q = 0; q < kProbes; ++q)
        pr[q] = hi_open ? (q == kProbes - 1 ? hi : lo + (hi - lo) * (float)(q + 1) / (float)kProbes)
                        : lo + (hi - lo) * (float)(q + 1) / (float)(kProbes + 1);
      int cq[kProbes];
#pragma unroll
      for (int q = 0; q < kProbes; ++q) {
        int m = 0;
#pragma unroll
        for (int j = 0; j < kLaneSlots; ++j) m += c[j] >= pr[q];
        cq[q] = __reduce_add_sync(0xffffffffu, m);
      }
      float nlo = lo, nhi = hi;
      bool nopen = hi_open, hit = false, got_hi = false;
#pragma unroll
      for (int q = 0; q < kProbes; ++q) {
        if (cq[q] > k_sel) nlo = pr[q];
        if (cq[q] == k_sel && !hit) tau = pr[q], hit = true;
        if (cq[q] < k_sel && !got_hi) nhi = pr[q], nopen = false, got_hi = true;
      }
      if (hit) {
        found = true;
        break;
      }
      if (nlo == lo && nhi == hi && nopen == hi_open) break;  // scores tied across the k-th position
      lo = nlo, hi = nhi, hi_open = nopen;
      if (!(hi > lo)) break;
    }
    // a rejected logit must score strictly below every selected one
    const float rej_score = ps + (warp_max(rej) - lse);
    if (found && rej_score < tau) {
      int pos = 0;
#pragma unroll
      for (int j = 0; j < kLaneSlots; ++j) {
        const bool take = c[j] >= tau;
        const unsigned m = __ballot_sync(0xffffffffu, take);
        if (take) {
          const uint32_t idx = static_cast<uint32_t>(bi[w][(j / SPL) * kLaneSlots + 32 * (j % SPL) + lane]);
          out[pos + __popc(m & ((1u << lane) - 1u))] =
              (static_cast<uint64_t>(ord_f32(c[j])) << 32) | (0xFFFFFFFFu - (lbase + idx));
        }
        pos += __popc(m);
      }
      return;
    }
  }
  if (lane == 0) {
    fail[1 + atomicAdd(&fail[0], 1)] = row;
    atomicAdd(&g_topk_fallback_rows, 1ull);
  }
}

constexpr int kMergeThreads = 512;
constexpr int kMaxBeam = 1024;

// Next BeamState from the n_new selected candidate keys of user u, sorted
// descending in sel[] (shared): codes, ancestors, scores, trie nodes and the
// lexicographic ranks of the new prefixes. lex[] is kMaxBeam shared scratch.
template <int NT, class LseOf>
__device__ void build_next_state(int u, int n_live, int n_new, int V, int L, int step, const uint64_t* sel, uint64_t* lex,
                                 const float* __restrict__ logits, LseOf lse_of, const BeamState& cur,
                                 const BeamState& nxt, const TrieDev& trie, int use_trie) {
  // beam b (rank order): decode parent lexrank + code, build next state
  for (int b = threadIdx.x; b < n_new; b += NT) {
    const uint64_t key = sel[b];
    const int nrow = u * n_new + b;
    if (key == 0) {  // empty slot: decodes harmlessly (code 0, ancestors = its user's first row)
      const int prow = u * n_live;
      for (int j = 0; j < step; ++j) {
        nxt.codes[(size_t)nrow * L + j] = 0;
        nxt.anc[(size_t)nrow * L + j] = cur.anc[(size_t)prow * L + j];
      }
      nxt.codes[(size_t)nrow * L + step] = 0;
      nxt.anc[(size_t)nrow * L + step] = prow;
      nxt.score[nrow] = -FLT_MAX;
      nxt.score64[nrow] = -INFINITY;
      if (use_trie) nxt.node[nrow] = -1;
      lex[b] = (static_cast<uint64_t>(0xFFFFFFFFu) << 32) | static_cast<uint32_t>(b);
      continue;
    }
    const uint32_t low = 0xFFFFFFFFu - static_cast<uint32_t>(key & 0xFFFFFFFFu);
    const int plr = static_cast<int>(low / static_cast<uint32_t>(V));
    const int code = static_cast<int>(low % static_cast<uint32_t>(V));
    const int pb = cur.lex2beam[(size_t)u * n_live + plr];
    const int prow = u * n_live + pb;
    if (use_trie) {  // child of the parent's node with this code (codes ascending)
      const int p = cur.node[prow];
      int lo = trie.child_off[p], hi = trie.child_off[p + 1] - 1, found = -1;
      while (lo <= hi) {
        const int mid = (lo + hi) >> 1, cc = trie.child_code[mid];
        if (cc == code) {
          found = trie.child_node[mid];
          break;
        }
        if (cc < code) lo = mid + 1;
        else hi = mid - 1;
      }
      nxt.node[nrow] = found;
    }
    for (int j = 0; j < step; ++j) {
      nxt.codes[(size_t)nrow * L + j] = cur.codes[(size_t)prow * L + j];
      nxt.anc[(size_t)nrow * L + j] = cur.anc[(size_t)prow * L + j];
    }
    nxt.codes[(size_t)nrow * L + step] = code;
    nxt.anc[(size_t)nrow * L + step] = prow;
    nxt.score[nrow] = unord_f32(static_cast<uint32_t>(key >> 32));
    nxt.score64[nrow] = cur.score64[prow] + (static_cast<double>(logits[(size_t)prow * V + code]) -
                                             static_cast<double>(lse_of(prow)));
    lex[b] = (static_cast<uint64_t>(low) << 32) | static_cast<uint32_t>(b);
  }
  __syncthreads();
  // lexicographic rank of the new prefixes = ascending (plr, code) = ascending
  // low: sort the complements descending (padding 0 sorts last)
  for (int i = threadIdx.x; i < n_new; i += NT) lex[i] = ~lex[i];
  __syncthreads();
  block_sort_desc<kMaxBeam, NT>(lex, n_new);
  for (int r = threadIdx.x; r < n_new; r += NT) {
    const int b = static_cast<int>(static_cast<uint32_t>(~lex[r]));
    nxt.lexrank[u * n_new + b] = r;
    nxt.lex2beam[(size_t)u * n_new + r] = b;
  }
}

__global__ void __launch_bounds__(kMergeThreads) beam_merge_kernel(int n_live, int k_sel, int n_new, int V, int L,
                                                                   int step, const uint64_t* __restrict__ cand,
                                                                   const float* __restrict__ logits,
                                                                   const float* __restrict__ lse, BeamState cur,
                                                                   BeamState nxt, TrieDev trie, int use_trie) {
  pdl_begin();
  __shared__ uint64_t sel[kMaxBeam];
  __shared__ uint64_t lex[kMaxBeam];
  __shared__ uint32_t hist[256];
  __shared__ uint32_t bc[4];
  __shared__ uint32_t counter;
  const int u = blockIdx.x;
  const int n = n_live * k_sel;
  const uint64_t* c = cand + (size_t)u * n;
  if (cur.nonfinite)
    for (int r = threadIdx.x; r < n_live; r += kMergeThreads)
      if (!isfinite(lse[(size_t)u * n_live + r])) *cur.nonfinite = 1;
  if (threadIdx.x == 0) counter = 0;
  __syncthreads();
  uint64_t tau = block_kth_largest<kMergeThreads>(n, n_new, [&](int i) { return c[i]; }, hist, bc);
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += kMergeThreads) {
    uint64_t key = c[i];
    if (key >= tau && key != 0) {  // key 0 = no candidate (constrained search)
      uint32_t pos = atomicAdd(&counter, 1u);
      if (pos < static_cast<uint32_t>(n_new)) sel[pos] = key;
    }
  }
  __syncthreads();
  for (int i = static_cast<int>(min(counter, static_cast<uint32_t>(n_new))) + threadIdx.x; i < n_new; i += kMergeThreads)
    sel[i] = 0;  // fewer candidates than slots: empty slots sort last
  __syncthreads();
  block_sort_desc<kMaxBeam, kMergeThreads>(sel, n_new);
  build_next_state<kMergeThreads>(u, n_live, n_new, V, L, step, sel, lex, logits,
                                  [&](int prow) { return lse[prow]; }, cur, nxt, trie, use_trie);
}

// ---------------------------------------------------------------------------
// Fused log-softmax + beam selection (unconstrained steps whose head GEMM
// wrote chunk statistics, EPI_STATS). One block per user; the logits are
// read only where they can hold a winner.
//
// Per parent row b: lse_b from the row's (max, sum exp) pairs of its 32-column
// chunks (generation.cpp:10-20). Chunk key = ord(ps_b + (cmax - lse_b)), the
// exact fp32 score of the chunk's best element. tau = a chunk key with at
// least n_new chunk keys >= tau (block_threshold32, at or just below the
// n_new-th largest): at least n_new elements score >= tau, so the n_new-th best
// candidate does too, and since fp32 rounding is monotone every element
// scoring >= tau lies in a chunk whose key is >= tau. Only those chunks are
// read (typically ~n_new of n_live * V / 32): their elements with score >=
// tau become the candidates (64-bit keys as in row_topk), the exact top n_new
// of which form the next beams -- the same set the full per-row top-k +
// merge selects. Degenerate inputs that overflow the candidate buffers
// (massive ties) take an exact radix select over all n_live * V keys.
// ---------------------------------------------------------------------------
constexpr int kSelThreads = 512;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kSelChunkKeys = 32768;  // chunk keys cached in shared memory (128 KB)
constexpr int kSelCand = 16384;       // candidate capacity (aliases the chunk-key cache)
constexpr int kSelIds = 4096;         // selected-chunk capacity
struct SelSmem {
  uint64_t sel[kMaxBeam];
  uint64_t lex[kMaxBeam];
  uint32_t hist[kSelWarps * 256];
  uint32_t ids[kSelIds];
  float lse[kMaxBeam];
  float ps[kMaxBeam];
  uint32_t lbase[kMaxBeam];
  uint32_t tot[256];
  uint32_t bc[4];
  uint32_t counter, nids;
};
constexpr size_t kSelSmemBytes = sizeof(uint32_t) * kSelChunkKeys + sizeof(SelSmem);
static_assert(sizeof(uint32_t) * kSelChunkKeys >= sizeof(uint64_t) * kSelCand, "candidate alias");

// A threshold tau over n 32-bit ordered-float keys with count(key >= tau) >= k,
// close to the k-th largest: one 2048-bucket histogram over the float range
// (bucket index is monotone in the key), the bucket where the count from the
// top reaches k, tau = the smallest key in that bucket. Three passes over the
// keys, no multi-pass radix contention.
template <class Get>
__device__ uint32_t block_threshold32(int n, int k, Get get, SelSmem& S) {
  if (n <= k) return 0;
  constexpr int NB = 2048;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t lo = 0xFFFFFFFFu, hi = 0;
  for (int i = threadIdx.x; i < n; i += kSelThreads) {
    const uint32_t x = get(i);
    lo = min(lo, x);
    hi = max(hi, x);
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if (lane == 0) {
    S.tot[warp] = lo;
    S.tot[kSelWarps + warp] = hi;
  }
  for (int b = threadIdx.x; b < NB; b += kSelThreads) S.hist[b] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t L = 0xFFFFFFFFu, H = 0;
    for (int w = 0; w < kSelWarps; ++w) L = min(L, S.tot[w]), H = max(H, S.tot[kSelWarps + w]);
    S.bc[0] = L;
    S.bc[1] = H;
    S.bc[3] = 0xFFFFFFFFu;
  }
  __syncthreads();
  const uint32_t L = S.bc[0], H = S.bc[1];
  if (L == H) return L;
  const float flo = unord_f32(L), fhi = unord_f32(H);
  float scale = static_cast<float>(NB) / (fhi - flo);
  if (!(scale > 0.f) || !isfinite(scale)) scale = 0.f;  // degenerate range: one bucket, tau = min
  auto bucket = [&](uint32_t x) {
    const float f = (unord_f32(x) - flo) * scale;
    return f >= static_cast<float>(NB - 1) ? NB - 1 : (f > 0.f ? static_cast<int>(f) : 0);
  };
  for (int i = threadIdx.x; i < n; i += kSelThreads) atomicAdd(&S.hist[bucket(get(i))], 1u);
  __syncthreads();
  // suffix counts: thread t owns buckets [4t, 4t + 4); scan over threads from the top
  const int t = threadIdx.x;
  uint32_t c4[4], own = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    c4[j] = S.hist[4 * t + j];
    own += c4[j];
  }
  // inclusive suffix over lanes (higher lanes = higher buckets)
  uint32_t suf = own;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_down_sync(0xffffffffu, suf, o);
    if (lane + o < 32) suf += v;
  }
  if (lane == 0) S.tot[64 + warp] = suf;  // warp total
  __syncthreads();
  uint32_t above_warps = 0;
  for (int w = warp + 1; w < kSelWarps; ++w) above_warps += S.tot[64 + w];
  uint32_t above = above_warps + suf - own;  // keys in buckets above this thread's
#pragma unroll
  for (int j = 3; j >= 0; --j) {
    if (above < static_cast<uint32_t>(k) && above + c4[j] >= static_cast<uint32_t>(k)) S.bc[2] = 4 * t + j;
    above += c4[j];
  }
  __syncthreads();
  const int bstar = static_cast<int>(S.bc[2]);
  uint32_t mn = 0xFFFFFFFFu;
  for (int i = threadIdx.x; i < n; i += kSelThreads) {
    const uint32_t x = get(i);
    if (bucket(x) == bstar) mn = min(mn, x);
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  if (lane == 0) atomicMin(&S.bc[3], mn);
  __syncthreads();
  const uint32_t tau = S.bc[3];
  __syncthreads();
  return tau;
}

__global__ void __launch_bounds__(kSelThreads, 1)
    beam_select_kernel(int n_live, int n_new, int V, int L, int step, const float* __restrict__ logits,
                       const float2* __restrict__ stats, long long stats_ld, float* __restrict__ lse_out,
                       uint32_t* __restrict__ gkeys, BeamState cur, BeamState nxt) {
  pdl_begin();
  extern __shared__ __align__(16) uint8_t sel_smem[];
  uint32_t* ckeys = reinterpret_cast<uint32_t*>(sel_smem);
  uint64_t* cand = reinterpret_cast<uint64_t*>(sel_smem);  // after the chunk selection
  SelSmem& S = *reinterpret_cast<SelSmem*>(sel_smem + sizeof(uint32_t) * kSelChunkKeys);
  const int u = blockIdx.x, r0 = u * n_live;
  const int NC = V >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // 1. log-softmax normaliser per parent row from its chunk statistics: P
  //    threads per row over interleaved chunks (consecutive threads read
  //    consecutive rows), 8 independent loads in flight per thread, online
  //    (max, sum) combine; the chunk maxima are kept (keys[], as floats) for
  //    step 2, the per-thread partials combined through S.hist
  const int nck = n_live * NC;
  const bool in_smem = nck <= kSelChunkKeys;
  uint32_t* keys = in_smem ? ckeys : gkeys + (size_t)u * nck;
  float* cmax = reinterpret_cast<float*>(keys);  // [c * n_live + b] before step 2
  {
    const int P = n_live >= kSelThreads ? 1 : kSelThreads / n_live;
    float2* part = reinterpret_cast<float2*>(S.hist);  // [P][n_live] (P * n_live <= 2048)
    const int Pn = P * n_live <= 2048 ? P : 2048 / n_live;
    for (int t = threadIdx.x; t < Pn * n_live; t += kSelThreads) {
      const int b = t % n_live, p = t / n_live;
      float M = -INFINITY, Ssum = 0.f;
      for (int c0 = p; c0 < NC; c0 += 8 * Pn) {
        float2 st[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = c0 + j * Pn;
          st[j] = c < NC ? __ldg(stats + (long long)c * stats_ld + r0 + b) : make_float2(-INFINITY, 0.f);
        }
        float mb = M;
#pragma unroll
        for (int j = 0; j < 8; ++j) mb = fmaxf(mb, st[j].x);
        float acc = M == -INFINITY ? 0.f : Ssum * __expf(M - mb);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = c0 + j * Pn;
          if (c < NC) {
            acc += st[j].y * __expf(st[j].x - mb);
            cmax[(size_t)c * n_live + b] = st[j].x;
          }
        }
        M = mb;
        Ssum = acc;
      }
      part[p * n_live + b] = make_float2(M, Ssum);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < n_live; b += kSelThreads) {
      float m = -INFINITY;
      for (int p = 0; p < Pn; ++p) m = fmaxf(m, part[p * n_live + b].x);
      float sum = 0.f;
      for (int p = 0; p < Pn; ++p) {
        const float2 q = part[p * n_live + b];
        sum += q.y * __expf(q.x - m);
      }
      const float lse = m + logf(sum);
      if (!isfinite(lse) && cur.nonfinite) *cur.nonfinite = 1;
      S.lse[b] = lse;
      S.ps[b] = cur.score[r0 + b];
      S.lbase[b] = static_cast<uint32_t>(cur.lexrank[r0 + b]) * static_cast<uint32_t>(V);
      lse_out[r0 + b] = lse;
    }
    if (threadIdx.x == 0) {
      S.counter = 0;
      S.nids = 0;
    }
    __syncthreads();
  }

  // 2. chunk keys in place: ord(ps + (cmax - lse)), index i = c * n_live + b
  for (int i = threadIdx.x; i < nck; i += kSelThreads) {
    const int c = i / n_live, b = i - c * n_live;
    keys[i] = ord_f32(S.ps[b] + (cmax[i] - S.lse[b]));
  }
  __syncthreads();
  const uint32_t tau = block_threshold32(nck, n_new, [&](int i) { return keys[i]; }, S);

  // 3. the chunks that can hold a winner
  for (int i0 = warp * 32; i0 < nck; i0 += kSelThreads) {
    const int i = i0 + lane;
    const bool take = i < nck && keys[i] >= tau;
    const uint32_t m = __ballot_sync(0xffffffffu, take);
    uint32_t base = 0;
    if (lane == 0 && m) base = atomicAdd(&S.nids, static_cast<uint32_t>(__popc(m)));
    base = __shfl_sync(0xffffffffu, base, 0);
    const uint32_t pos = base + __popc(m & ((1u << lane) - 1u));
    if (take && pos < static_cast<uint32_t>(kSelIds)) S.ids[pos] = static_cast<uint32_t>(i);
  }
  __syncthreads();
  const int nids = static_cast<int>(S.nids);

  // 4. candidates: elements of the selected chunks scoring >= tau (warp per chunk)
  if (nids <= kSelIds) {
    constexpr int kU = 4;  // chunks in flight per warp
    for (int j0 = warp; j0 < nids; j0 += kSelWarps * kU) {
      float x[kU];
      int bb[kU], cc[kU];
#pragma unroll
      for (int q = 0; q < kU; ++q) {
        const int j = j0 + q * kSelWarps;
        const int i = j < nids ? static_cast<int>(S.ids[j]) : 0;
        cc[q] = i / n_live;
        bb[q] = i - cc[q] * n_live;
        x[q] = j < nids ? __ldg(logits + (size_t)(r0 + bb[q]) * V + cc[q] * 32 + lane) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < kU; ++q) {
      if (j0 + q * kSelWarps >= nids) break;
      const int b = bb[q];
      const int code = cc[q] * 32 + lane;
      const float sc = S.ps[b] + (x[q] - S.lse[b]);
      const uint32_t k32 = ord_f32(sc);
      const bool take = k32 >= tau;
      const uint32_t m = __ballot_sync(0xffffffffu, take);
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(&S.counter, static_cast<uint32_t>(__popc(m)));
      base = __shfl_sync(0xffffffffu, base, 0);
      const uint32_t pos = base + __popc(m & ((1u << lane) - 1u));
      if (take && pos < static_cast<uint32_t>(kSelCand))
        cand[pos] = (static_cast<uint64_t>(k32) << 32) | (0xFFFFFFFFu - (S.lbase[b] + static_cast<uint32_t>(code)));
      }
    }
  }
  __syncthreads();
  const int ncand = static_cast<int>(S.counter);
  const bool fallback = nids > kSelIds || ncand > kSelCand;
  __syncthreads();
  if (threadIdx.x == 0) S.counter = 0;
  if (!fallback) {
    const uint64_t t64 =
        block_kth_largest<kSelThreads>(ncand, n_new, [&](int i) { return cand[i]; }, S.hist, S.bc);
    __syncthreads();
    for (int i = threadIdx.x; i < ncand; i += kSelThreads) {
      const uint64_t key = cand[i];
      if (key >= t64) {
        const uint32_t pos = atomicAdd(&S.counter, 1u);
        if (pos < static_cast<uint32_t>(n_new)) S.sel[pos] = key;
      }
    }
  } else {  // exact select over every (row, code) of the user
    auto key_of = [&](int i) {
      const int b = i / V, code = i - b * V;
      const float sc = S.ps[b] + (logits[(size_t)(r0 + b) * V + code] - S.lse[b]);
      return (static_cast<uint64_t>(ord_f32(sc)) << 32) | (0xFFFFFFFFu - (S.lbase[b] + static_cast<uint32_t>(code)));
    };
    const int n = n_live * V;
    const uint64_t t64 = block_kth_largest<kSelThreads>(n, n_new, key_of, S.hist, S.bc);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += kSelThreads) {
      const uint64_t key = key_of(i);
      if (key >= t64) {
        const uint32_t pos = atomicAdd(&S.counter, 1u);
        if (pos < static_cast<uint32_t>(n_new)) S.sel[pos] = key;
      }
    }
    if (threadIdx.x == 0) atomicAdd(&g_topk_fallback_rows, 1ull);
  }
  __syncthreads();
  block_sort_desc<kMaxBeam, kSelThreads>(S.sel, n_new);
  build_next_state<kSelThreads>(u, n_live, n_new, V, L, step, S.sel, S.lex, logits,
                                [&](int prow) { return S.lse[prow - r0]; }, cur, nxt, TrieDev{}, 0);
}

__global__ void beam_init_kernel(int users, BeamState st) {
  pdl_begin();
  int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= users) return;
  st.score[u] = 0.f;
  st.score64[u] = 0.0;
  st.lexrank[u] = 0;
  st.lex2beam[u] = 0;
  if (st.node) st.node[u] = 0;  // trie root
  if (st.nonfinite && u == 0) *st.nonfinite = 0;
}

// Constrained candidates (generation.cpp:58-64): block per row; the log-softmax
// normaliser runs over the whole row, candidates are the node's trie children.
__global__ void __launch_bounds__(kRowThreads) row_topk_trie_kernel(int V, int k_sel, const float* __restrict__ logits,
                                                                    const float* __restrict__ pscore,
                                                                    const int32_t* __restrict__ plex,
                                                                    const int32_t* __restrict__ node, TrieDev trie,
                                                                    float* __restrict__ lse_out,
                                                                    uint64_t* __restrict__ cand) {
  pdl_begin();
  __shared__ uint32_t hist[256];
  __shared__ uint32_t bc[4];
  __shared__ float red[kRowThreads / 32];
  __shared__ uint32_t counter;
  const int row = blockIdx.x;
  const float* lg = logits + (size_t)row * V;
  uint64_t* out = cand + (size_t)row * k_sel;
  const int nd = node[row];
  if (nd < 0) {  // empty slot: no candidates
    for (int i = threadIdx.x; i < k_sel; i += kRowThreads) out[i] = 0;
    if (threadIdx.x == 0) lse_out[row] = 0.f;
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
  const int o0 = trie.child_off[nd], nc = trie.child_off[nd + 1] - o0;
  auto key_of = [&](int i) -> uint64_t {
    const int code = trie.child_code[o0 + i];
    const float sc = ps + (lg[code] - lse);
    return (static_cast<uint64_t>(ord_f32(sc)) << 32) | (0xFFFFFFFFu - (lbase + static_cast<uint32_t>(code)));
  };
  if (threadIdx.x == 0) {
    lse_out[row] = lse;
    counter = 0;
  }
  if (nc <= k_sel) {
    for (int i = threadIdx.x; i < k_sel; i += kRowThreads) out[i] = i < nc ? key_of(i) : 0;
    return;
  }
  __syncthreads();
  const uint64_t tau = block_kth_largest<kRowThreads>(nc, k_sel, key_of, hist, bc);
  __syncthreads();
  for (int i = threadIdx.x; i < nc; i += kRowThreads) {
    const uint64_t key = key_of(i);
    if (key >= tau) {
      const uint32_t pos = atomicAdd(&counter, 1u);
      if (pos < static_cast<uint32_t>(k_sel)) out[pos] = key;
    }
  }
}

// Warp per row: acc[r] += logits[r][code] - lse(logits[r]) in f64.
__global__ void pick_logprob_kernel(int rows, int V, const float* __restrict__ logits, const int32_t* __restrict__ codes,
                                    int code_stride, int step, double* __restrict__ acc) {
  pdl_begin();
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* lg = logits + (size_t)r * V;
  float mx = -FLT_MAX;
  for (int i = lane; i < V; i += 32) mx = fmaxf(mx, lg[i]);
  mx = warp_max(mx);
  float sum = 0.f;
  for (int i = lane; i < V; i += 32) sum += __expf(lg[i] - mx);
  sum = warp_sum(sum);
  if (lane == 0) {
    const int code = codes[(size_t)r * code_stride + step];
    acc[r] += static_cast<double>(lg[code]) - (static_cast<double>(mx) + log(static_cast<double>(sum)));
  }
}

// Top-k / top-p sampling step (sample_topk_topp, generation.cpp:90-148), one
// block per sample row: tempered probabilities sorted by (p desc, index asc)
// (bitonic, stable like std::stable_sort), cut to top_k, then to the smallest
// prefix reaching top_p of the kept mass, then the first sorted entry whose
// running sum reaches u * total; log_prob accumulates the untempered
// log-softmax of the pick (f64).
constexpr int kSampleThreads = 512;
__global__ void __launch_bounds__(kSampleThreads) sample_kernel(int V, int vpad, int L, int step, float inv_temp,
                                                                int top_k, double top_p,
                                                                const float* __restrict__ logits,
                                                                const double* __restrict__ uniforms,
                                                                int32_t* __restrict__ codes,
                                                                double* __restrict__ logp) {
  pdl_begin();
  extern __shared__ uint64_t skeys[];  // [vpad]
  __shared__ double dscan[kSampleThreads];
  __shared__ float red[kSampleThreads / 32];
  __shared__ int sidx[2];
  __shared__ double stotal;
  const int row = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* lg = logits + (size_t)row * V;
  auto bmax = [&](float v) {
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float t = -FLT_MAX;
    for (int w = 0; w < kSampleThreads / 32; ++w) t = fmaxf(t, red[w]);
    return t;
  };
  auto bsum = [&](float v) {
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float t = 0.f;
    for (int w = 0; w < kSampleThreads / 32; ++w) t += red[w];
    return t;
  };
  float mx = -FLT_MAX;
  for (int i = tid; i < V; i += kSampleThreads) mx = fmaxf(mx, lg[i]);
  mx = bmax(mx);
  float se = 0.f, st = 0.f;
  for (int i = tid; i < V; i += kSampleThreads) se += __expf(lg[i] - mx);
  se = bsum(se);
  const float lse = mx + logf(se);  // model log-softmax (untempered)
  for (int i = tid; i < V; i += kSampleThreads) st += __expf((lg[i] - mx) * inv_temp);
  st = bsum(st);
  const float lse_t = mx * inv_temp + logf(st);
  for (int i = tid; i < vpad; i += kSampleThreads) {
    const float pr = i < V ? __expf(lg[i] * inv_temp - lse_t) : 0.f;
    skeys[i] = i < V ? (static_cast<uint64_t>(ord_f32(pr)) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(i)) : 0;
  }
  __syncthreads();
  for (int size = 2; size <= vpad; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < vpad / 2; i += kSampleThreads) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool desc = (lo & size) == 0;
        const uint64_t x = skeys[lo], y = skeys[hi];
        if ((x < y) == desc) skeys[lo] = y, skeys[hi] = x;
      }
      __syncthreads();
    }
  const int keep = top_k > 0 ? min(top_k, V) : V;
  // inclusive prefix sums (f64) of the sorted probabilities, thread-contiguous segments
  const int per = (keep + kSampleThreads - 1) / kSampleThreads;
  const int b0 = tid * per, b1 = min(keep, b0 + per);
  double loc = 0.0;
  for (int i = b0; i < b1; ++i) loc += static_cast<double>(unord_f32(static_cast<uint32_t>(skeys[i] >> 32)));
  dscan[tid] = loc;
  __syncthreads();
  if (tid == 0) {  // exclusive scan of 512 partials (tiny)
    double run = 0.0;
    for (int t = 0; t < kSampleThreads; ++t) {
      const double v = dscan[t];
      dscan[t] = run;
      run += v;
    }
    stotal = run;  // mass of the kept set
    sidx[0] = keep;
    sidx[1] = INT_MAX;
  }
  __syncthreads();
  const double target = top_p * stotal;
  double acc = dscan[tid];
  for (int i = b0; i < b1; ++i) {
    acc += static_cast<double>(unord_f32(static_cast<uint32_t>(skeys[i] >> 32)));
    if (acc >= target - 1e-15) {
      atomicMin(&sidx[0], i + 1);
      break;
    }
  }
  __syncthreads();
  const int cut = sidx[0];
  // total = prefix(cut - 1)
  if (cut - 1 >= b0 && cut - 1 < b1) {
    double a2 = dscan[tid];
    for (int i = b0; i < cut; ++i) a2 += static_cast<double>(unord_f32(static_cast<uint32_t>(skeys[i] >> 32)));
    stotal = a2;
  }
  __syncthreads();
  const double u = uniforms[(size_t)row * L + step] * stotal;
  acc = dscan[tid];
  for (int i = b0; i < min(b1, cut); ++i) {
    acc += static_cast<double>(unord_f32(static_cast<uint32_t>(skeys[i] >> 32)));
    if (acc >= u) {
      atomicMin(&sidx[1], i);
      break;
    }
  }
  __syncthreads();
  if (tid == 0) {
    const int pos = sidx[1] == INT_MAX ? cut - 1 : sidx[1];
    const int code = static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(skeys[pos] & 0xFFFFFFFFu));
    codes[(size_t)row * L + step] = code;
    logp[row] += static_cast<double>(lg[code]) - static_cast<double>(lse);
  }
}

}  // namespace

void launch_row_topk(int rows, int V, int k_sel, const float* logits, const float* parent_score,
                     const int32_t* parent_lexrank, float* lse, uint64_t* cand, int32_t* fail, cudaStream_t s) {
  if (rows <= 0) return;
  size_t smem = static_cast<size_t>(V) * 8;
  static size_t set = 0;
  if (smem > 48 * 1024 && smem > set) {
    cudaFuncSetAttribute(row_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    set = smem;
  }
  ProfScope ps(PROF_BEAM, s, 0.0, double(rows) * V * 4);
  if (fail && V % 4 == 0 && k_sel < V && k_sel <= 1024) {
    cudaMemsetAsync(fail, 0, sizeof(int32_t), s);
    if (k_sel <= 192)
      launch_pdl(row_topk_warp_kernel<32>, (rows + 3) / 4, 128, 0, s, rows, V, k_sel, logits, parent_score, parent_lexrank,
                                                              lse, cand, fail);
    else
      launch_pdl(row_topk_warp_kernel<64>, (rows + 1) / 2, 64, 0, s, rows, V, k_sel, logits, parent_score, parent_lexrank,
                                                             lse, cand, fail);
    // rows the warp kernel could not decide (usually none): exact radix select
    launch_pdl(row_topk_kernel, std::min(rows, 32), kRowThreads, smem, s, V, k_sel, logits, parent_score,
                                                                            parent_lexrank, lse, cand, fail);
    launch_counter() += 2;
    return;
  }
  launch_pdl(row_topk_kernel, rows, kRowThreads, smem, s, V, k_sel, logits, parent_score, parent_lexrank, lse, cand, nullptr);
  ++launch_counter();
}

void launch_row_topk_trie(int rows, int V, int k_sel, const float* logits, const float* parent_score,
                          const int32_t* parent_lexrank, const int32_t* node, TrieDev trie, float* lse,
                          uint64_t* cand, cudaStream_t s) {
  if (rows <= 0) return;
  ProfScope ps(PROF_BEAM, s, 0.0, double(rows) * V * 4);
  launch_pdl(row_topk_trie_kernel, rows, kRowThreads, 0, s, V, k_sel, logits, parent_score, parent_lexrank, node, trie, lse,
                                                    cand);
  ++launch_counter();
}

void launch_pick_logprob(int rows, int V, const float* logits, const int32_t* codes, int code_stride, int step,
                         double* acc, cudaStream_t s) {
  if (rows <= 0) return;
  ProfScope ps(PROF_BEAM, s, 0.0, double(rows) * V * 4);
  launch_pdl(pick_logprob_kernel, (rows + 7) / 8, 256, 0, s, rows, V, logits, codes, code_stride, step, acc);
  ++launch_counter();
}

void launch_sample(int rows, int V, int L, int step, float temperature, int top_k, double top_p, const float* logits,
                   const double* uniforms, int32_t* codes, double* logp, cudaStream_t s) {
  if (rows <= 0) return;
  int vpad = 1;
  while (vpad < V) vpad <<= 1;
  const size_t smem = static_cast<size_t>(vpad) * 8;
  if (smem > 200 * 1024) throw std::invalid_argument("sampling supports codebooks up to 25600 codes");
  static size_t set = 0;
  if (smem > 48 * 1024 && smem > set) {
    cudaFuncSetAttribute(sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    set = smem;
  }
  ProfScope ps(PROF_BEAM, s, 0.0, double(rows) * V * 4);
  launch_pdl(sample_kernel, rows, kSampleThreads, smem, s, V, vpad, L, step, 1.f / temperature, top_k, top_p, logits,
                                                   uniforms, codes, logp);
  ++launch_counter();
}

unsigned long long topk_fallback_rows(bool reset) {
  unsigned long long v = 0;
  cudaMemcpyFromSymbol(&v, g_topk_fallback_rows, sizeof(v));
  if (reset) {
    unsigned long long z = 0;
    cudaMemcpyToSymbol(g_topk_fallback_rows, &z, sizeof(z));
  }
  return v;
}

void launch_beam_merge(int users, int n_live, int k_sel, int n_new, int V, int L, int step, const uint64_t* cand,
                       const float* logits, const float* lse, const BeamState& cur, BeamState& nxt, cudaStream_t s,
                       const TrieDev* trie) {
  if (n_new > kMaxBeam) throw std::invalid_argument("beam width above 1024 is not supported");
  ProfScope ps(PROF_BEAM, s, 0.0, 0.0);
  launch_pdl(beam_merge_kernel, users, kMergeThreads, 0, s, n_live, k_sel, n_new, V, L, step, cand, logits, lse, cur, nxt,
                                                    trie ? *trie : TrieDev{}, trie ? 1 : 0);
  ++launch_counter();
}

void launch_beam_select(int users, int n_live, int n_new, int V, int L, int step, const float* logits,
                        const float2* stats, long long stats_ld, float* lse, uint32_t* scratch, const BeamState& cur,
                        BeamState& nxt, cudaStream_t s) {
  if (n_new > kMaxBeam) throw std::invalid_argument("beam width above 1024 is not supported");
  if (V % 32 != 0) throw std::invalid_argument("beam_select: codebook size must be a multiple of 32");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(beam_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSelSmemBytes));
    attr = true;
  }
  // algorithmic bytes: the chunk statistics plus ~2 logit chunks per new beam
  ProfScope ps(PROF_BEAM, s, 0.0, double(users) * (double(n_live) * (V / 32) * 8 + 2.0 * n_new * 128));
  launch_pdl(beam_select_kernel, users, kSelThreads, kSelSmemBytes, s, n_live, n_new, V, L, step, logits, stats,
             stats_ld, lse, scratch, cur, nxt);
  ++launch_counter();
}

size_t beam_select_scratch_words(int n_live, int V) {
  const size_t nck = size_t(n_live) * (V / 32);
  return nck <= size_t(kSelChunkKeys) ? 0 : nck;
}

void launch_beam_init(int users, BeamState& st, cudaStream_t s) {
  launch_pdl(beam_init_kernel, (users + 127) / 128, 128, 0, s, users, st);
  ++launch_counter();
}

}  // namespace orx
