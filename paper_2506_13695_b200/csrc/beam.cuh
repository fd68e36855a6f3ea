// Beam pruning over 3-level semantic IDs (beam_search, generation.cpp:41-88).
//
// Candidate key (64 bit, larger = better) reproduces the reference sort
// (log_prob desc, codes lexicographic asc, generation.cpp:74-77):
//   hi 32 bits: order-preserving bits of the fp32 score parent + (logit - lse)
//   lo 32 bits: 0xFFFFFFFF - (parent_lexrank * V + code)
// where parent_lexrank is the rank of the parent's code prefix among the live
// beams of its user, so lexicographic order of the extended prefixes is the
// order of (parent_lexrank, code).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace orx {

struct BeamState {  // live beams of one step, row r = user * n_live + beam
  int32_t* codes = nullptr;     // [rows][L]
  float* score = nullptr;       // [rows] fp32 ranking score
  double* score64 = nullptr;    // [rows] f64 accumulated log-prob (output)
  int32_t* lexrank = nullptr;   // [rows]
  int32_t* lex2beam = nullptr;  // [users][n_live]
  int32_t* anc = nullptr;       // [rows][L] ancestor row per position
  int32_t* node = nullptr;      // [rows] semantic-trie node of the prefix (constrained search), -1 = empty slot
  // [1] (shared by both states of a search): set when a scored row's
  // log-softmax normaliser is non-finite, i.e. a NaN/Inf reached the logits
  // (the reference throws "non-finite value produced on tape", tape.cpp:29)
  int32_t* nonfinite = nullptr;
};

// Semantic-ID trie on the device (SemanticTrie, trie.hpp:27-62) as CSR over
// prefix nodes: node 0 = root; children of n are [child_off[n], child_off[n+1])
// of child_code (ascending) / child_node.
struct TrieDev {
  const int32_t* child_off = nullptr;
  const int32_t* child_code = nullptr;
  const int32_t* child_node = nullptr;
};

// Constrained variant of launch_row_topk (generation.cpp:58-64): lse over the
// whole row, candidates only the trie children of the row's node; rows with
// fewer than k_sel children (or no node) pad with key 0 (= no candidate).
void launch_row_topk_trie(int rows, int V, int k_sel, const float* logits, const float* parent_score,
                          const int32_t* parent_lexrank, const int32_t* node, TrieDev trie, float* lse,
                          uint64_t* cand, cudaStream_t s);

// One step of top-k / top-p sampling for `rows` sample rows: writes
// codes[r * L + step] and adds the pick's model log-softmax to logp[r] (f64);
// uniforms[r * L + step] are the reference Rng's draws for that row / step.
void launch_sample(int rows, int V, int L, int step, float temperature, int top_k, double top_p, const float* logits,
                   const double* uniforms, int32_t* codes, double* logp, cudaStream_t s);

// acc[r] += logits[r][code[r * code_stride + step]] - logsumexp(logits[r]) (f64):
// one position of PolicyModel::sequence_log_prob (policy.cpp:297-310).
void launch_pick_logprob(int rows, int V, const float* logits, const int32_t* codes, int code_stride, int step,
                         double* acc, cudaStream_t s);

// Per row: lse = logsumexp(logits), then the top k_sel candidate keys.
// fail: device workspace of rows + 1 ints (fast path's undecided rows); NULL
// selects the block radix-select kernel for every row.
void launch_row_topk(int rows, int V, int k_sel, const float* logits, const float* parent_score,
                     const int32_t* parent_lexrank, float* lse, uint64_t* cand, int32_t* fail, cudaStream_t s);

// Rows of the fast top-k kernel that fell back to the radix select since the last reset.
unsigned long long topk_fallback_rows(bool reset);

// Per user: top n_new of n_live * k_sel candidates, sorted; builds the next
// BeamState (codes, scores, lexranks, ancestors).
// With a trie (constrained search) key 0 marks "no candidate": users may end a
// step with fewer than n_new live beams (the rest are empty slots, node -1).
void launch_beam_merge(int users, int n_live, int k_sel, int n_new, int V, int L, int step, const uint64_t* cand,
                       const float* logits, const float* lse, const BeamState& cur, BeamState& nxt, cudaStream_t s,
                       const TrieDev* trie = nullptr);

// Fused log-softmax + exact beam selection from the head GEMM's chunk
// statistics (Epi::stats, stats[c * stats_ld + row] = (max, sum exp) of the
// row's 32-column chunk c): replaces launch_row_topk + launch_beam_merge for
// unconstrained steps and reads only the logit chunks that can hold a winner.
// Writes lse[rows] and the next BeamState. scratch: per user
// beam_select_scratch_words(n_live, V) words (0 when the chunk keys fit on chip).
void launch_beam_select(int users, int n_live, int n_new, int V, int L, int step, const float* logits,
                        const float2* stats, long long stats_ld, float* lse, uint32_t* scratch, const BeamState& cur,
                        BeamState& nxt, cudaStream_t s);
size_t beam_select_scratch_words(int n_live, int V);

}  // namespace orx
