// One-GPU inference engine for the OneRec hot path (encode + beam search).
#pragma once

#include <memory>
#include <vector>

#include "../../include/orx.h"
#include "model.hpp"

namespace orx {

// Expert parallelism over NVLink peer memory: rank `rank`
// of `world` computes the experts the placement gives it (ep_plan.hpp): by
// default experts [rank * E / world, (rank + 1) * E / world) of every MoE
// layer; `owner` ([moe_layers][E], rank or -1 = replicated) overrides it and
// must be the same on every rank.
struct EpConfig {
  int rank = 0, world = 1;
  uint8_t unique_id[128] = {};  // ncclUniqueId (bootstraps the region exchange)
  std::vector<int32_t> owner;
};

class Engine {
 public:
  virtual ~Engine() = default;
  static std::unique_ptr<Engine> create(const HostWeights& w, int device, int precision, int max_users,
                                        int max_width, const EpConfig* ep = nullptr);
  virtual void stage_batch(const orx_user_batch& b) = 0;
  virtual void encode(float* z_out) = 0;
  virtual void beam_search(int width, orx_beam_out* out) = 0;
  // Trie-constrained beam search (generation.cpp:58-64; needs set_trie).
  virtual void beam_search_constrained(int width, orx_beam_out* out) = 0;
  // Pipelined serving: stage + launch a request without waiting (at most two
  // in flight, one per staging slot); collect() returns the oldest one's beams.
  virtual void submit_beam(const orx_user_batch& b, int width) = 0;
  virtual void collect(orx_beam_out* out) = 0;
  // CSR trie (see TrieDev in beam.cuh), uploaded to the device.
  virtual void set_trie(int n_nodes, const int32_t* child_off, int64_t n_edges, const int32_t* child_code,
                        const int32_t* child_node) = 0;
  // PolicyModel::sequence_log_prob (policy.cpp:297-310) for n (user, full code) queries.
  virtual void sequence_log_prob(int n, const int32_t* user, const int32_t* codes, double* out) = 0;
  // sample_topk_topp (generation.cpp:90-148): width samples per user, user u
  // drawing from Rng(seed).split(streams[u]) (streams NULL: u).
  virtual void sample(int width, double temperature, int top_k, double top_p, uint64_t seed, const uint64_t* streams,
                      orx_beam_out* out) = 0;
  virtual void next_logits(const float* z, int n_z, int n, const int32_t* z_index, const int32_t* prefixes,
                           const int32_t* prefix_len, float* logits) = 0;
  virtual void score_prefixes(int n, const int32_t* user, const int32_t* prefixes, const int32_t* prefix_len,
                              float* logits) = 0;
  // Expert parallelism: rows routed to each expert of each MoE layer, summed
  // over every rank and every MoE call since creation (or the last reset):
  // out [moe_layers][E]; identical on every rank. Zeros without expert parallelism.
  virtual void expert_load(int64_t* out, bool reset) = 0;
  virtual void* stream() = 0;
  // Synchronous entry points refuse to run while a submitted search is in
  // flight (they would reuse its staging slot / drain its result).
  virtual void require_idle() const = 0;
  int64_t h2d_bytes = 0, d2h_bytes = 0;
};

void validate_batch(const orx_config& cfg, const orx_user_batch& b);
void nccl_unique_id(uint8_t out[128]);
long long launch_counter_value();

}  // namespace orx
