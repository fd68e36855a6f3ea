// ORACLE / TEST INFRASTRUCTURE ONLY.
// Compiles the reference's own types together with include/orx_genrec.hpp to
// show (and test) the drop-in: the same genrec::UserContext goes through the
// reference PolicyModel and through the B200 engine; encodings, logits and the
// generated items are compared. Exit code 0 = parity, 2 = no GPU available.
#include <cmath>
#include <cstdio>
#include <string>

#include "../include/orx_genrec.hpp"
#include "../paper_2506_13695_b200/csrc/synth_users.hpp"

using namespace genrec;

int main(int argc, char** argv) {
  int width = argc > 1 ? std::atoi(argv[1]) : 16;
  PolicyConfig cfg;  // 0.015B (Table 2)
  cfg.n_layers = 4;
  cfg.d_model = 128;
  cfg.ffn_hidden = 256;
  cfg.n_heads = 4;
  cfg.codebook_size = 8192;
  UserContext ctx;
  orx_synth::synth_user<Rng>(
      1, 0, orx_synth::Lengths{},
      [&](int uid, int g, int a) {
        ctx.uid = uid;
        ctx.gender = g;
        ctx.age_bucket = a;
      },
      [&](int p, int64_t vid, int aid, double tag, double ts, double play, double dur, uint32_t lab) {
        InteractionFeature f;
        f.vid = vid;
        f.aid = aid;
        f.tag = tag;
        f.ts = ts;
        f.playtime = play;
        f.duration = dur;
        f.labels = lab;
        (p == 0 ? ctx.short_seq : p == 1 ? ctx.positive_seq : ctx.lifelong_seq).push_back(f);
      });
  PolicyModel ref(cfg);
  std::unique_ptr<orx_genrec::B200Policy> gpu;
  try {
    gpu = std::make_unique<orx_genrec::B200Policy>(cfg, 0, ORX_PRECISION_FP32, 1, width);
  } catch (const std::runtime_error& e) {
    printf("{\"gpu\": false, \"error\": \"%s\"}\n", e.what());
    return 2;
  }
  Array z_ref = ref.encode_eval(ctx);
  Array z_gpu = gpu->encode_eval(ctx);
  double zmax = 0, zerr = 0;
  for (int64_t i = 0; i < z_ref.size(); ++i) {
    zmax = std::max(zmax, std::fabs(z_ref.at(i)));
    zerr = std::max(zerr, std::fabs(z_ref.at(i) - z_gpu.at(i)));
  }
  SemanticTrie trie(cfg.n_code_layers);
  GenerationRequest req;
  req.width = width;
  auto items_ref = beam_search(req, policy_scorer(ref, z_ref), cfg.n_code_layers, cfg.codebook_size, trie);
  auto items_gpu = gpu->generate(ctx, req, trie);
  Array l_ref = ref.next_logits_eval(z_ref, {});
  Array l_gpu = gpu->next_logits_eval(z_ref, {});
  double lmax = 0, lerr = 0;
  for (int64_t i = 0; i < l_ref.size(); ++i) {
    lmax = std::max(lmax, std::fabs(l_ref.at(i)));
    lerr = std::max(lerr, std::fabs(l_ref.at(i) - l_gpu.at(i)));
  }
  int same = 0;
  for (size_t i = 0; i < items_ref.size() && i < items_gpu.size(); ++i) same += items_ref[i].codes == items_gpu[i].codes;
  printf("{\"gpu\": true, \"z_rel\": %.3e, \"logits_rel\": %.3e, \"items\": %zu, \"same_rank\": %d}\n", zerr / zmax,
         lerr / lmax, items_gpu.size(), same);
  bool ok = zerr / zmax < 1e-4 && lerr / lmax < 1e-3 && items_gpu.size() == items_ref.size() &&
            same >= static_cast<int>(items_ref.size()) * 3 / 4;
  return ok ? 0 : 1;
}
