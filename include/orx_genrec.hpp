// orx_genrec.hpp — header-only C++ drop-in adapter for the reference tree
// (proj/core). Include it after the reference headers and link liborx.so:
// it restores the reference's C++ surface (exceptions, genrec::Array,
// genrec::GeneratedItem, genrec::StepScorer) on top of the C-ABI in orx.h.
//
//   genrec::PolicyModel(cfg)             -> orx_genrec::B200Policy(cfg)        (same seeded weights)
//   genrec::PolicyModel::load(path)      -> orx_genrec::B200Policy::load(path)
//   PolicyModel::encode_eval(ctx)        -> B200Policy::encode_eval(ctx)        policy.cpp:317-321
//   PolicyModel::next_logits_eval(z, p)  -> B200Policy::next_logits_eval(z, p)  policy.cpp:323-329
//   policy_scorer(model, z)              -> B200Policy::scorer(z)               generation.cpp:163-167
//   generate(req{beam}, scorer, ...)     -> B200Policy::generate(ctx, req, trie) generation.cpp:41-88,150-154
//   (new) batched                        -> B200Policy::generate_batch(users, req, trie)
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "genrec/generation.hpp"
#include "genrec/policy.hpp"
#include "orx.h"

namespace orx_genrec {

inline void check(int rc) {
  if (rc == ORX_OK) return;
  if (rc == ORX_EINVAL) throw std::invalid_argument(orx_last_error());
  throw std::runtime_error(orx_last_error());
}

inline orx_config to_orx(const genrec::PolicyConfig& c) {
  orx_config o{};
  o.n_layers = c.n_layers;
  o.d_model = c.d_model;
  o.ffn_hidden = c.ffn_hidden;
  o.n_heads = c.n_heads;
  o.moe_enabled = c.moe_enabled;
  o.n_experts = c.n_experts;
  o.experts_active = c.experts_active;
  o.moe_location = c.moe_location == genrec::MoeLocation::decoder ? 0 : 1;
  o.expert_round_multiple = c.expert_round_multiple;
  o.n_code_layers = c.n_code_layers;
  o.codebook_size = c.codebook_size;
  o.short_len = c.short_len;
  o.positive_len = c.positive_len;
  o.lifelong_len = c.lifelong_len;
  o.n_queries = c.n_queries;
  o.lifelong_blocks = c.lifelong_blocks;
  o.vid_vocab = c.vid_vocab;
  o.aid_vocab = c.aid_vocab;
  o.uid_vocab = c.uid_vocab;
  o.gender_vocab = c.gender_vocab;
  o.age_vocab = c.age_vocab;
  o.n_label_flags = c.n_label_flags;
  o.use_sid_history = c.use_sid_history;
  o.vid_only_features = c.vid_only_features;
  o.compress_threshold = c.compress_threshold;
  o.moe_bias_update = c.moe_bias_update;
  o.seed = c.seed;
  return o;
}

// SoA copy of a set of genrec::UserContext (policy.hpp:15-32) viewable as orx_user_batch.
class PackedUsers {
 public:
  PackedUsers(const std::vector<const genrec::UserContext*>& users, int n_code_layers) {
    for (const auto* u : users) {
      uid_.push_back(u->uid);
      gender_.push_back(u->gender);
      age_.push_back(u->age_bucket);
    }
    const std::vector<genrec::InteractionFeature> genrec::UserContext::*seqs[3] = {
        &genrec::UserContext::short_seq, &genrec::UserContext::positive_seq, &genrec::UserContext::lifelong_seq};
    orx_records* dst[3] = {&view_.short_seq, &view_.positive_seq, &view_.lifelong_seq};
    for (int p = 0; p < 3; ++p) {
      P& s = p_[p];
      s.off.push_back(0);
      bool sid = true;
      for (const auto* u : users) {
        for (const auto& f : u->*seqs[p]) {
          s.vid.push_back(f.vid);
          s.aid.push_back(f.aid);
          s.tag.push_back(f.tag);
          s.ts.push_back(f.ts);
          s.play.push_back(f.playtime);
          s.dur.push_back(f.duration);
          s.labels.push_back(f.labels);
          sid = sid && static_cast<int>(f.sid.size()) == n_code_layers;
          for (int c : f.sid) s.sid.push_back(c);
        }
        s.off.push_back(static_cast<int64_t>(s.vid.size()));
      }
      *dst[p] = orx_records{s.off.data(), s.vid.data(),  s.aid.data(), s.tag.data(), s.ts.data(),
                            s.play.data(), s.dur.data(), s.labels.data(), sid && !s.vid.empty() ? s.sid.data() : nullptr};
    }
    view_.n_users = static_cast<int32_t>(users.size());
    view_.uid = uid_.data();
    view_.gender = gender_.data();
    view_.age_bucket = age_.data();
  }
  const orx_user_batch* get() const { return &view_; }

 private:
  struct P {
    std::vector<int64_t> off, vid;
    std::vector<int32_t> aid, sid;
    std::vector<double> tag, ts, play, dur;
    std::vector<uint32_t> labels;
  };
  std::vector<int32_t> uid_, gender_, age_;
  P p_[3];
  orx_user_batch view_{};
};

class B200Policy {
 public:
  // Same seeded weights as genrec::PolicyModel(cfg) (policy.cpp:59-137).
  explicit B200Policy(const genrec::PolicyConfig& cfg, int device = 0, int precision = ORX_PRECISION_BF16,
                      int max_users = 128, int max_width = 512)
      : cfg_(cfg) {
    orx_config c = to_orx(cfg);
    orx_weights* w = nullptr;
    check(orx_weights_create_random(&c, &w));
    w_.reset(w);
    create(device, precision, max_users, max_width);
  }
  static B200Policy load(const std::string& path, int device = 0, int precision = ORX_PRECISION_BF16,
                         int max_users = 128, int max_width = 512) {
    return B200Policy(path, device, precision, max_users, max_width);
  }

  const genrec::PolicyConfig& config() const { return cfg_; }

  genrec::Array encode_eval(const genrec::UserContext& ctx) {
    PackedUsers b({&ctx}, cfg_.n_code_layers);
    const int T = cfg_.enc_seq_len(), d = cfg_.d_model;
    std::vector<float> z(static_cast<size_t>(T) * d);
    check(orx_encode(e_.get(), b.get(), z.data()));
    return genrec::Array({T, d}, std::vector<double>(z.begin(), z.end()));
  }

  genrec::Array next_logits_eval(const genrec::Array& z_enc, std::span<const int> prefix) {
    std::vector<float> z(z_enc.data(), z_enc.data() + z_enc.size());
    const int L = cfg_.n_code_layers, V = cfg_.codebook_size;
    std::vector<int32_t> pre(static_cast<size_t>(L), -1);
    GENREC_REQUIRE(static_cast<int>(prefix.size()) < L, "no prediction head at this position");
    for (size_t j = 0; j < prefix.size(); ++j) pre[j] = prefix[j];
    int32_t zi = 0, plen = static_cast<int32_t>(prefix.size());
    std::vector<float> logits(static_cast<size_t>(V));
    check(orx_next_logits(e_.get(), z.data(), 1, 1, &zi, pre.data(), &plen, logits.data()));
    return genrec::Array({1, V}, std::vector<double>(logits.begin(), logits.end()));
  }

  // Per-prefix StepScorer (slow path, one decoder call per prefix, kept for drop-in).
  genrec::StepScorer scorer(const genrec::Array& z_enc) {
    return [this, z_enc](std::span<const int> prefix) { return next_logits_eval(z_enc, prefix); };
  }

  std::vector<std::vector<genrec::GeneratedItem>> generate_batch(const std::vector<genrec::UserContext>& users,
                                                                 const genrec::GenerationRequest& req,
                                                                 const genrec::SemanticTrie& trie) {
    genrec::validate_request(req);
    if (req.strategy != genrec::SearchStrategy::beam || req.constrain_to_trie)
      throw std::invalid_argument("B200 path implements unconstrained beam search only");
    std::vector<const genrec::UserContext*> ptrs;
    for (const auto& u : users) ptrs.push_back(&u);
    PackedUsers b(ptrs, cfg_.n_code_layers);
    const int L = cfg_.n_code_layers, W = req.width, U = static_cast<int>(users.size());
    std::vector<int32_t> codes(static_cast<size_t>(U) * W * L), n_items(static_cast<size_t>(U));
    std::vector<double> logp(static_cast<size_t>(U) * W);
    orx_beam_out out{codes.data(), logp.data(), n_items.data()};
    check(orx_beam_search(e_.get(), b.get(), W, &out));
    std::vector<std::vector<genrec::GeneratedItem>> res(static_cast<size_t>(U));
    for (int u = 0; u < U; ++u)
      for (int i = 0; i < n_items[static_cast<size_t>(u)]; ++i) {
        genrec::GeneratedItem item;  // finish(), generation.cpp:22-30
        const int32_t* c = &codes[(static_cast<size_t>(u) * W + i) * L];
        item.codes.codes.assign(c, c + L);
        item.log_prob = logp[static_cast<size_t>(u) * W + i];
        const auto* ids = trie.lookup(item.codes.codes);
        item.legal = ids != nullptr;
        if (ids) item.item_ids = *ids;
        res[static_cast<size_t>(u)].push_back(std::move(item));
      }
    return res;
  }

  std::vector<genrec::GeneratedItem> generate(const genrec::UserContext& ctx, const genrec::GenerationRequest& req,
                                              const genrec::SemanticTrie& trie) {
    return generate_batch({ctx}, req, trie)[0];
  }

 private:
  B200Policy(const std::string& path, int device, int precision, int max_users, int max_width) {
    orx_weights* w = nullptr;
    check(orx_weights_load_grcp(path.c_str(), &w));
    w_.reset(w);
    orx_config c{};
    check(orx_weights_config(w, &c));
    cfg_.n_layers = c.n_layers;
    cfg_.d_model = c.d_model;
    cfg_.ffn_hidden = c.ffn_hidden;
    cfg_.n_heads = c.n_heads;
    cfg_.moe_enabled = c.moe_enabled;
    cfg_.n_experts = c.n_experts;
    cfg_.experts_active = c.experts_active;
    cfg_.moe_location = c.moe_location == 0 ? genrec::MoeLocation::decoder : genrec::MoeLocation::enc_and_dec;
    cfg_.expert_round_multiple = c.expert_round_multiple;
    cfg_.n_code_layers = c.n_code_layers;
    cfg_.codebook_size = c.codebook_size;
    cfg_.short_len = c.short_len;
    cfg_.positive_len = c.positive_len;
    cfg_.lifelong_len = c.lifelong_len;
    cfg_.n_queries = c.n_queries;
    cfg_.lifelong_blocks = c.lifelong_blocks;
    cfg_.vid_vocab = c.vid_vocab;
    cfg_.aid_vocab = c.aid_vocab;
    cfg_.uid_vocab = c.uid_vocab;
    cfg_.gender_vocab = c.gender_vocab;
    cfg_.age_vocab = c.age_vocab;
    cfg_.n_label_flags = c.n_label_flags;
    cfg_.use_sid_history = c.use_sid_history;
    cfg_.vid_only_features = c.vid_only_features;
    cfg_.compress_threshold = c.compress_threshold;
    cfg_.moe_bias_update = c.moe_bias_update;
    cfg_.seed = c.seed;
    create(device, precision, max_users, max_width);
  }
  void create(int device, int precision, int max_users, int max_width) {
    orx_engine* e = nullptr;
    check(orx_engine_create(w_.get(), device, precision, max_users, max_width, &e));
    e_.reset(e);
  }
  struct WDel {
    void operator()(orx_weights* w) const { orx_weights_destroy(w); }
  };
  struct EDel {
    void operator()(orx_engine* e) const { orx_engine_destroy(e); }
  };
  genrec::PolicyConfig cfg_;
  std::unique_ptr<orx_weights, WDel> w_;
  std::unique_ptr<orx_engine, EDel> e_;
};

}  // namespace orx_genrec
