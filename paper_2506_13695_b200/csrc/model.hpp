// Host-side model description: config helpers, the parameter inventory in the
// reference's insertion order, a bit-exact re-implementation of the
// reference Rng (xoshiro256** + Box-Muller, rng.cpp:11-77), seeded weight
// init (PolicyModel ctor, policy.cpp:59-137) and GRCP checkpoint I/O
// (policy.cpp:344-443, io.cpp:22-95).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/orx.h"

namespace orx {

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct RuntimeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void require(bool cond, const std::string& msg) {
  if (!cond) throw InvalidArgument(msg);
}

// ---- config -----------------------------------------------------------------
orx_config config_default();
orx_config config_preset(const std::string& name);
inline int enc_layers(const orx_config& c) { return c.n_layers / 2; }
inline int dec_layers(const orx_config& c) { return c.n_layers - c.n_layers / 2; }
inline int enc_seq_len(const orx_config& c) { return 1 + c.short_len + c.positive_len + c.n_queries; }
inline int aid_dim(const orx_config& c) { return c.d_model / 2 > 1 ? c.d_model / 2 : 1; }
inline int minor_dim(const orx_config& c) { return c.d_model / 8 > 1 ? c.d_model / 8 : 1; }
inline int static_dim(const orx_config& c) { return c.d_model / 16 > 1 ? c.d_model / 16 : 1; }
int expert_hidden_size(int d_model, int multiple);  // nn.cpp:192-196
inline int expert_hidden(const orx_config& c) { return expert_hidden_size(c.d_model, c.expert_round_multiple); }
inline int feat_dim(const orx_config& c) {
  return c.vid_only_features ? c.d_model : c.d_model + aid_dim(c) + 5 * minor_dim(c);
}
inline bool enc_moe(const orx_config& c) { return c.moe_enabled && c.moe_location == 1; }
// MoE layers in engine order: encoder layers (when they are MoE), then decoder layers
inline int moe_layers(const orx_config& c) {
  return c.moe_enabled ? (enc_moe(c) ? enc_layers(c) : 0) + dec_layers(c) : 0;
}
void validate_config(const orx_config& c);
std::string config_to_json(const orx_config& c);
orx_config config_from_json(const std::string& s);

// ---- Rng (rng.cpp) ------------------------------------------------------------------
class Rng {
 public:
  explicit Rng(uint64_t seed);
  uint64_t next_u64();
  double uniform();
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double normal();
  int64_t randint(int64_t n);
  Rng split(uint64_t id) const;
  uint64_t s_[4];
  double cached_normal_ = 0.0;
  bool has_cached_normal_ = false;
};

// ---- parameter inventory ----------------------------------------------------------
enum class Init { Normal, Zeros, Ones };
struct ParamSpec {
  std::string name;
  int rows, cols;
  Init init;
  double stddev;
};
std::vector<ParamSpec> param_specs(const orx_config& c);

struct Tensor {
  std::string name;
  int rows = 0, cols = 0;
  std::vector<float> data;
};

class HostWeights {
 public:
  orx_config cfg{};
  std::vector<Tensor> tensors;
  std::unordered_map<std::string, int> index;
  const Tensor& get(const std::string& name) const;
  const float* ptr(const std::string& name) const { return get(name).data.data(); }
  // ep_world > 1: only the experts rank ep_rank computes are materialised
  // (partial = true): contiguous blocks, or per `owner` [moe_layers][E]
  // (rank or -1 = replicated; ep_plan.hpp) when given
  static HostWeights random(const orx_config& cfg, int ep_rank = 0, int ep_world = 1,
                            const int32_t* owner = nullptr);
  bool partial = false;
  static HostWeights load_grcp(const std::string& path);
  void save_grcp(const std::string& path) const;
};

}  // namespace orx
