// ORACLE / TEST INFRASTRUCTURE ONLY. Never linked into or called by the product
// path (paper_2506_13695_b200/liborx.so). Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference leg may execute this binary.
//
// Drives the UNMODIFIED reference library (/root/reference/proj/core, compiled
// by oracle/Makefile into oracle/_ref/libgenrec_core.a) through its public API:
//   PolicyModel(cfg)           policy.cpp:59-137   (seeded random init)
//   PolicyModel::save/load     policy.cpp:411-443  (GRCP)
//   PolicyModel::encode_eval   policy.cpp:317-321
//   PolicyModel::next_logits_eval policy.cpp:323-329
//   beam_search + policy_scorer   generation.cpp:41-88,163-167
// on synthetic users from paper_2506_13695_b200/csrc/synth_users.hpp (the same
// generator the engine uses), and writes .npy golden files or timing JSON.
#include <sys/wait.h>
#include <unistd.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "../paper_2506_13695_b200/csrc/synth_users.hpp"
#include "genrec/generation.hpp"
#include "genrec/policy.hpp"

using namespace genrec;

namespace {

// ---- minimal .npy writer ----------------------------------------------------
void write_npy(const std::string& path, const char* descr, const std::vector<size_t>& shape,
               const void* data, size_t bytes) {
  std::ostringstream hdr;
  hdr << "{'descr': '" << descr << "', 'fortran_order': False, 'shape': (";
  for (size_t i = 0; i < shape.size(); ++i) hdr << shape[i] << (shape.size() == 1 ? "," : (i + 1 < shape.size() ? ", " : ""));
  hdr << "), }";
  std::string h = hdr.str();
  size_t total = 10 + h.size() + 1;
  size_t pad = (64 - total % 64) % 64;
  h += std::string(pad, ' ');
  h += '\n';
  std::ofstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot write " + path);
  const char magic[] = "\x93NUMPY";
  f.write(magic, 6);
  char ver[2] = {1, 0};
  f.write(ver, 2);
  uint16_t hl = static_cast<uint16_t>(h.size());
  f.write(reinterpret_cast<const char*>(&hl), 2);
  f.write(h.data(), static_cast<std::streamsize>(h.size()));
  f.write(static_cast<const char*>(data), static_cast<std::streamsize>(bytes));
}

// ---- config presets -------------------
PolicyConfig preset(const std::string& name) {
  PolicyConfig c;
  if (name == "tiny") {  // test_policy.cpp:14-32
    c.n_layers = 4; c.d_model = 16; c.ffn_hidden = 32; c.n_heads = 2; c.n_code_layers = 3;
    c.codebook_size = 8; c.short_len = 4; c.positive_len = 4; c.lifelong_len = 8; c.n_queries = 2;
    c.lifelong_blocks = 1; c.vid_vocab = 64; c.aid_vocab = 16; c.uid_vocab = 32; c.seed = 9;
  } else if (name == "0.015B") {
    c.n_layers = 4; c.d_model = 128; c.ffn_hidden = 256; c.n_heads = 4; c.codebook_size = 8192;
  } else if (name == "0.121B") {
    c.n_layers = 8; c.d_model = 1024; c.ffn_hidden = 2048; c.n_heads = 8; c.codebook_size = 8192;
  } else if (name == "0.935B") {
    c.n_layers = 8; c.d_model = 1024; c.ffn_hidden = 2048; c.n_heads = 8; c.codebook_size = 8192;
    c.moe_enabled = true; c.n_experts = 24; c.experts_active = 2;
  } else if (name == "2.633B") {
    c.n_layers = 24; c.d_model = 1024; c.ffn_hidden = 2048; c.n_heads = 8; c.codebook_size = 8192;
    c.moe_enabled = true; c.n_experts = 24; c.experts_active = 4;
    c.moe_location = MoeLocation::enc_and_dec;
  } else {
    throw std::invalid_argument("unknown preset " + name);
  }
  return c;
}

void apply_override(PolicyConfig& c, const std::string& kv) {
  auto eq = kv.find('=');
  if (eq == std::string::npos) throw std::invalid_argument("bad --set " + kv);
  std::string k = kv.substr(0, eq), v = kv.substr(eq + 1);
  long long x = std::stoll(v == "true" ? "1" : (v == "false" ? "0" : (v == "decoder" || v == "enc_and_dec" ? "0" : v)));
  if (k == "n_layers") c.n_layers = int(x);
  else if (k == "d_model") c.d_model = int(x);
  else if (k == "ffn_hidden") c.ffn_hidden = int(x);
  else if (k == "n_heads") c.n_heads = int(x);
  else if (k == "moe_enabled") c.moe_enabled = x != 0;
  else if (k == "n_experts") c.n_experts = int(x);
  else if (k == "experts_active") c.experts_active = int(x);
  else if (k == "moe_location") c.moe_location = v == "enc_and_dec" ? MoeLocation::enc_and_dec : MoeLocation::decoder;
  else if (k == "expert_round_multiple") c.expert_round_multiple = int(x);
  else if (k == "n_code_layers") c.n_code_layers = int(x);
  else if (k == "codebook_size") c.codebook_size = int(x);
  else if (k == "short_len") c.short_len = int(x);
  else if (k == "positive_len") c.positive_len = int(x);
  else if (k == "lifelong_len") c.lifelong_len = int(x);
  else if (k == "n_queries") c.n_queries = int(x);
  else if (k == "lifelong_blocks") c.lifelong_blocks = int(x);
  else if (k == "vid_vocab") c.vid_vocab = int(x);
  else if (k == "aid_vocab") c.aid_vocab = int(x);
  else if (k == "uid_vocab") c.uid_vocab = int(x);
  else if (k == "gender_vocab") c.gender_vocab = int(x);
  else if (k == "age_vocab") c.age_vocab = int(x);
  else if (k == "use_sid_history") c.use_sid_history = x != 0;
  else if (k == "vid_only_features") c.vid_only_features = x != 0;
  else if (k == "seed") c.seed = static_cast<uint64_t>(x);
  else throw std::invalid_argument("unknown config key " + k);
}

struct Args {
  std::string cmd;
  PolicyConfig cfg;
  std::string grcp;  // load weights from here instead of the seeded init
  std::string out;
  uint64_t user_seed = 1;
  int user_begin = 0, n_users = 1;
  orx_synth::Lengths lens;
  bool lens_set = false;
  int width = 8;
  int n_prefix = 4;
  bool beam = true;
  bool seq = true;         // also dump sequence_log_prob of every beam item
  bool sid_codes = false;  // give every record semantic-id codes sid[l] = (vid >> 8l) % V (use_sid_history)
  int procs = 1;
  int calls = 4;
  int trie_items = 0;      // > 0: constrained beam search over a seeded random trie
  uint64_t trie_seed = 77;
  int trie_fanout = 0;     // > 0: codes drawn from [0, fanout) per level (a dense trie)
  bool sample = false;     // also dump sample_topk_topp with Rng(sample_seed).split(user)
  uint64_t sample_seed = 5;
  double temperature = 1.0, top_p = 1.0;
  int top_k = 0;
  // compress: seeded raw histories + clustered content for compress_lifelong
  int hist_len = 600, content_dim = 32, threshold = 8, max_out = 2000;
};

Args parse(int argc, char** argv) {
  Args a;
  if (argc < 2) throw std::invalid_argument("usage: ref_driver <save-grcp|dump|bench> [options]");
  a.cmd = argv[1];
  a.cfg = preset("0.015B");
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) throw std::invalid_argument("missing value for " + k);
      return argv[++i];
    };
    if (k == "--preset") a.cfg = preset(next());
    else if (k == "--set") apply_override(a.cfg, next());
    else if (k == "--grcp") a.grcp = next();
    else if (k == "--out") a.out = next();
    else if (k == "--user-seed") a.user_seed = std::stoull(next());
    else if (k == "--user-begin") a.user_begin = std::stoi(next());
    else if (k == "--n-users") a.n_users = std::stoi(next());
    else if (k == "--lens") {
      std::string v = next();
      if (sscanf(v.c_str(), "%d,%d,%d", &a.lens.n_short, &a.lens.n_positive, &a.lens.n_lifelong) != 3)
        throw std::invalid_argument("--lens short,positive,lifelong");
      a.lens_set = true;
    } else if (k == "--width") a.width = std::stoi(next());
    else if (k == "--n-prefix") a.n_prefix = std::stoi(next());
    else if (k == "--no-beam") a.beam = false;
    else if (k == "--no-seq") a.seq = false;
    else if (k == "--sid-codes") a.sid_codes = true;
    else if (k == "--procs") a.procs = std::stoi(next());
    else if (k == "--calls") a.calls = std::stoi(next());
    else if (k == "--trie-items") a.trie_items = std::stoi(next());
    else if (k == "--trie-seed") a.trie_seed = std::stoull(next());
    else if (k == "--trie-fanout") a.trie_fanout = std::stoi(next());
    else if (k == "--hist-len") a.hist_len = std::stoi(next());
    else if (k == "--content-dim") a.content_dim = std::stoi(next());
    else if (k == "--threshold") a.threshold = std::stoi(next());
    else if (k == "--max-out") a.max_out = std::stoi(next());
    else if (k == "--sample") a.sample = true;
    else if (k == "--sample-seed") a.sample_seed = std::stoull(next());
    else if (k == "--temperature") a.temperature = std::stod(next());
    else if (k == "--top-k") a.top_k = std::stoi(next());
    else if (k == "--top-p") a.top_p = std::stod(next());
    else throw std::invalid_argument("unknown option " + k);
  }
  if (!a.lens_set) {
    a.lens.n_short = a.cfg.short_len;
    a.lens.n_positive = a.cfg.positive_len;
    a.lens.n_lifelong = a.cfg.lifelong_len;
  }
  return a;
}

UserContext make_user(const Args& a, int index) {
  UserContext ctx;
  orx_synth::synth_user<Rng>(
      a.user_seed, static_cast<uint64_t>(index), a.lens,
      [&](int uid, int gender, int age) {
        ctx.uid = uid;
        ctx.gender = gender;
        ctx.age_bucket = age;
      },
      [&](int pathway, int64_t vid, int aid, double tag, double ts, double playtime, double duration,
          uint32_t labels) {
        InteractionFeature f;
        f.vid = vid;
        f.aid = aid;
        f.tag = tag;
        f.ts = ts;
        f.playtime = playtime;
        f.duration = duration;
        f.labels = labels;
        if (a.sid_codes)
          for (int l = 0; l < a.cfg.n_code_layers; ++l)
            f.sid.push_back(static_cast<int>((vid >> (8 * l)) % a.cfg.codebook_size));
        (pathway == 0 ? ctx.short_seq : pathway == 1 ? ctx.positive_seq : ctx.lifelong_seq).push_back(f);
      });
  return ctx;
}

PolicyModel make_model(const Args& a) {
  if (!a.grcp.empty()) return PolicyModel::load(a.grcp);
  return PolicyModel(a.cfg);
}

std::string upath(const Args& a, const char* what, int u) {
  return a.out + "/" + what + "_u" + std::to_string(u) + ".npy";
}

int cmd_dump(const Args& a) {
  PolicyModel model = make_model(a);
  const PolicyConfig& cfg = model.config();
  int V = cfg.codebook_size, L = cfg.n_code_layers;
  SemanticTrie trie(L);
  if (a.trie_items > 0) {
    // seeded random item catalogue (codes per level in [0, fanout or V)); written for the engine side
    Rng tr(a.trie_seed);
    const int range = a.trie_fanout > 0 ? a.trie_fanout : V;
    std::vector<int32_t> tc;
    for (int it = 0; it < a.trie_items; ++it) {
      std::vector<int> c(static_cast<size_t>(L));
      for (int j = 0; j < L; ++j) c[size_t(j)] = static_cast<int>(tr.randint(range));
      for (int x : c) tc.push_back(x);
      trie.insert(SemanticId{c}, it);
    }
    write_npy(a.out + "/trie_codes.npy", "<i4", {size_t(a.trie_items), size_t(L)}, tc.data(), tc.size() * 4);
  } else {
    trie.insert(SemanticId{std::vector<int>(static_cast<size_t>(L), 0)}, 0);
  }
  for (int i = 0; i < a.n_users; ++i) {
    int u = a.user_begin + i;
    UserContext ctx = make_user(a, u);
    auto t0 = std::chrono::steady_clock::now();
    Array z = model.encode_eval(ctx);
    auto t1 = std::chrono::steady_clock::now();
    write_npy(upath(a, "z", u), "<f8", {size_t(z.rows()), size_t(z.cols())}, z.data(),
              size_t(z.size()) * 8);
    std::vector<std::vector<int>> prefixes{{}};
    if (a.beam) {
      GenerationRequest req;
      req.width = a.width;
      req.constrain_to_trie = a.trie_items > 0;
      auto items = beam_search(req, policy_scorer(model, z), L, V, trie);
      std::vector<int32_t> codes;
      std::vector<double> lp, seq;
      for (auto& it : items) {
        for (int c : it.codes.codes) codes.push_back(c);
        lp.push_back(it.log_prob);
        if (!a.seq) continue;
        // teacher-forced sequence log-prob of the same item (policy.cpp:297-310), eval session
        Tape tape;
        ParamSession ps(tape, model.params(), false);
        Var zv = tape.leaf(z);
        seq.push_back(model.sequence_log_prob(ps, zv, it.codes).value().at(0));
      }
      write_npy(upath(a, "beam_codes", u), "<i4", {items.size(), size_t(L)}, codes.data(), codes.size() * 4);
      write_npy(upath(a, "beam_logp", u), "<f8", {items.size()}, lp.data(), lp.size() * 8);
      if (a.seq) write_npy(upath(a, "seq_logp", u), "<f8", {seq.size()}, seq.data(), seq.size() * 8);
      if (a.sample) {
        GenerationRequest sreq;
        sreq.strategy = SearchStrategy::topk_topp;
        sreq.width = a.width;
        sreq.temperature = a.temperature;
        sreq.top_k = a.top_k;
        sreq.top_p = a.top_p;
        Rng srng = Rng(a.sample_seed).split(static_cast<uint64_t>(u));
        auto smp = generate(sreq, policy_scorer(model, z), L, V, trie, srng);
        std::vector<int32_t> sc;
        std::vector<double> sl;
        for (auto& it : smp) {
          for (int c : it.codes.codes) sc.push_back(c);
          sl.push_back(it.log_prob);
        }
        write_npy(upath(a, "sample_codes", u), "<i4", {smp.size(), size_t(L)}, sc.data(), sc.size() * 4);
        write_npy(upath(a, "sample_logp", u), "<f8", {smp.size()}, sl.data(), sl.size() * 8);
      }
      std::set<std::vector<int>> seen;
      for (int len = 1; len < L; ++len)
        for (int j = 0; j < static_cast<int>(items.size()) && j < a.n_prefix; ++j) {
          std::vector<int> p(items[size_t(j)].codes.codes.begin(), items[size_t(j)].codes.codes.begin() + len);
          if (seen.insert(p).second) prefixes.push_back(p);
        }
    } else {
      // Greedy chain plus seeded random prefixes (teacher forcing only).
      Array l0 = model.next_logits_eval(z, {});
      int best = 0;
      for (int c = 1; c < V; ++c)
        if (l0.at(c) > l0.at(best)) best = c;
      prefixes.push_back({best});
      Rng r(1234 + static_cast<uint64_t>(u));
      for (int j = 1; j < a.n_prefix; ++j) prefixes.push_back({static_cast<int>(r.randint(V))});
      for (int j = 0; j < a.n_prefix; ++j)
        prefixes.push_back({static_cast<int>(r.randint(V)), static_cast<int>(r.randint(V))});
    }
    std::vector<int32_t> pre;
    std::vector<double> logits;
    for (auto& p : prefixes) {
      for (int j = 0; j < L; ++j) pre.push_back(j < static_cast<int>(p.size()) ? p[size_t(j)] : -1);
      Array lg = model.next_logits_eval(z, p);
      for (int c = 0; c < V; ++c) logits.push_back(lg.at(c));
    }
    write_npy(upath(a, "prefixes", u), "<i4", {prefixes.size(), size_t(L)}, pre.data(), pre.size() * 4);
    write_npy(upath(a, "logits", u), "<f8", {prefixes.size(), size_t(V)}, logits.data(), logits.size() * 8);
    auto t2 = std::chrono::steady_clock::now();
    fprintf(stderr, "user %d: encode %.3fs, rest %.3fs\n", u,
            std::chrono::duration<double>(t1 - t0).count(), std::chrono::duration<double>(t2 - t1).count());
  }
  return 0;
}

// compress_lifelong (policy.cpp:447-510) on seeded raw histories: user u has
// hist_len + 37 * u records whose content rows are drawn around 24 latent
// centres; the user's Rng is build_user_context's (policy.cpp:564).
int cmd_compress(const Args& a) {
  const int D = a.content_dim;
  std::vector<int64_t> off{0}, vid, ooff{0}, ovid;
  std::vector<int32_t> aid, oaid;
  std::vector<uint32_t> lab, olab;
  std::vector<double> tag, ts, play, dur, content, otag, ots, oplay, odur;
  std::vector<uint64_t> seeds;
  Rng world(a.user_seed);
  std::vector<double> centres(static_cast<size_t>(24) * D);
  for (auto& c : centres) c = world.normal();
  for (int u = 0; u < a.n_users; ++u) {
    const int n = a.hist_len + 37 * u;
    Rng r = Rng(a.user_seed).split(static_cast<uint64_t>(u));
    std::vector<InteractionFeature> hist;
    Array cont({n, D});
    double t = -static_cast<double>(n) * 0.01;
    for (int i = 0; i < n; ++i) {
      InteractionFeature f;
      f.vid = static_cast<int64_t>(r.randint(1 << 20));
      f.aid = static_cast<int>(r.randint(100000));
      f.tag = r.uniform();
      f.ts = t;
      t += 0.01;
      f.duration = r.uniform(0.05, 1.0);
      f.playtime = f.duration * r.uniform();
      f.labels = static_cast<uint32_t>(r.randint(32));
      hist.push_back(f);
      const int cl = static_cast<int>(r.randint(24));
      for (int j = 0; j < D; ++j) cont.at(i, j) = centres[static_cast<size_t>(cl) * D + j] + 0.3 * r.normal();
    }
    const uint64_t seed = a.cfg.seed ^ (0x9e3779b97f4a7c15ULL * static_cast<uint64_t>(u + 1));
    Rng krng(seed);
    auto out = compress_lifelong(hist, cont, a.threshold, a.max_out, krng);
    seeds.push_back(seed);
    for (int i = 0; i < n; ++i) {
      const auto& f = hist[size_t(i)];
      vid.push_back(f.vid), aid.push_back(f.aid), lab.push_back(f.labels);
      tag.push_back(f.tag), ts.push_back(f.ts), play.push_back(f.playtime), dur.push_back(f.duration);
      for (int j = 0; j < D; ++j) content.push_back(cont.at(i, j));
    }
    off.push_back(off.back() + n);
    for (const auto& f : out) {
      ovid.push_back(f.vid), oaid.push_back(f.aid), olab.push_back(f.labels);
      otag.push_back(f.tag), ots.push_back(f.ts), oplay.push_back(f.playtime), odur.push_back(f.duration);
    }
    ooff.push_back(ooff.back() + static_cast<int64_t>(out.size()));
  }
  auto w8 = [&](const char* n, const std::vector<double>& v) {
    write_npy(a.out + "/" + n + ".npy", "<f8", {v.size()}, v.data(), v.size() * 8);
  };
  auto wi8 = [&](const char* n, const std::vector<int64_t>& v) {
    write_npy(a.out + "/" + n + ".npy", "<i8", {v.size()}, v.data(), v.size() * 8);
  };
  auto wi4 = [&](const char* n, const void* p, size_t cnt) {
    write_npy(a.out + "/" + n + ".npy", "<i4", {cnt}, p, cnt * 4);
  };
  wi8("in_offsets", off), wi8("in_vid", vid), wi4("in_aid", aid.data(), aid.size()), wi4("in_labels", lab.data(), lab.size());
  w8("in_tag", tag), w8("in_ts", ts), w8("in_playtime", play), w8("in_duration", dur);
  write_npy(a.out + "/in_content.npy", "<f8", {content.size() / size_t(D), size_t(D)}, content.data(), content.size() * 8);
  write_npy(a.out + "/seeds.npy", "<u8", {seeds.size()}, seeds.data(), seeds.size() * 8);
  wi8("out_offsets", ooff), wi8("out_vid", ovid), wi4("out_aid", oaid.data(), oaid.size()), wi4("out_labels", olab.data(), olab.size());
  w8("out_tag", otag), w8("out_ts", ots), w8("out_playtime", oplay), w8("out_duration", odur);
  return 0;
}

// Bounded CPU sample of the hot path: per worker process, encode one user and
// time `calls` decoder calls on beam-shaped prefixes; per-user time is
// extrapolated to the full beam (1 + 2W scorer calls, generation.cpp:52-56).
// With calls < 0 the whole beam_search is run and timed (small configs).
int cmd_bench(const Args& a) {
  auto ti = std::chrono::steady_clock::now();
  PolicyModel model = make_model(a);
  double init_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - ti).count();
  const PolicyConfig& cfg = model.config();
  int V = cfg.codebook_size, L = cfg.n_code_layers;
  std::vector<int> pipes;
  std::vector<pid_t> kids;
  auto wall0 = std::chrono::steady_clock::now();
  for (int p = 0; p < a.procs; ++p) {
    int fd[2];
    if (pipe(fd) != 0) throw std::runtime_error("pipe failed");
    pid_t pid = fork();
    if (pid == 0) {
      close(fd[0]);
      SemanticTrie trie(L);
      trie.insert(SemanticId{std::vector<int>(static_cast<size_t>(L), 0)}, 0);
      double enc = 0, call = 0, beam = 0;
      int n_enc = 0, n_call = 0, n_beam = 0;
      for (int i = p; i < a.n_users; i += a.procs) {
        UserContext ctx = make_user(a, a.user_begin + i);
        auto t0 = std::chrono::steady_clock::now();
        Array z = model.encode_eval(ctx);
        auto t1 = std::chrono::steady_clock::now();
        enc += std::chrono::duration<double>(t1 - t0).count();
        ++n_enc;
        if (a.calls < 0) {
          GenerationRequest req;
          req.width = a.width;
          auto items = beam_search(req, policy_scorer(model, z), L, V, trie);
          beam += std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
          ++n_beam;
        } else {
          for (int c = 0; c < a.calls; ++c) {
            std::vector<int> pre;
            for (int j = 0; j < c % L; ++j) pre.push_back((c * 7 + j * 13) % V);
            auto c0 = std::chrono::steady_clock::now();
            Array lg = model.next_logits_eval(z, pre);
            call += std::chrono::duration<double>(std::chrono::steady_clock::now() - c0).count();
            ++n_call;
          }
        }
      }
      char buf[256];
      int n = snprintf(buf, sizeof buf, "%d %d %d %.9f %.9f %.9f\n", n_enc, n_call, n_beam, enc, call, beam);
      if (write(fd[1], buf, size_t(n)) != n) _exit(3);
      _exit(0);
    }
    close(fd[1]);
    pipes.push_back(fd[0]);
    kids.push_back(pid);
  }
  double enc = 0, call = 0, beam = 0;
  long n_enc = 0, n_call = 0, n_beam = 0;
  for (size_t p = 0; p < kids.size(); ++p) {
    char buf[256] = {0};
    ssize_t r = read(pipes[p], buf, sizeof buf - 1);
    int st = 0;
    waitpid(kids[p], &st, 0);
    if (r <= 0 || !WIFEXITED(st) || WEXITSTATUS(st) != 0) throw std::runtime_error("worker failed");
    int e, c, b;
    double te, tc, tb;
    sscanf(buf, "%d %d %d %lf %lf %lf", &e, &c, &b, &te, &tc, &tb);
    n_enc += e; n_call += c; n_beam += b; enc += te; call += tc; beam += tb;
  }
  double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
  double t_enc = n_enc ? enc / double(n_enc) : 0;
  double t_call = n_call ? call / double(n_call) : 0;
  double t_beam = n_beam ? beam / double(n_beam) : (1.0 + 2.0 * a.width) * t_call;
  double t_user = t_enc + t_beam;
  double users_per_s = double(a.procs) / t_user;
  printf("{\"users_per_s\": %.9g, \"procs\": %d, \"t_encode_s\": %.6g, \"t_call_s\": %.6g, "
         "\"t_beam_s\": %.6g, \"beam_measured\": %s, \"n_users\": %d, \"calls\": %d, \"width\": %d, "
         "\"init_s\": %.4g, \"wall_s\": %.4g}\n",
         users_per_s, a.procs, t_enc, t_call, t_beam, n_beam ? "true" : "false", a.n_users, a.calls,
         a.width, init_s, wall);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    Args a = parse(argc, argv);
    if (a.cmd == "save-grcp") {
      if (a.out.empty()) throw std::invalid_argument("--out required");
      PolicyModel(a.cfg).save(a.out);
      return 0;
    }
    if (a.cmd == "dump") return cmd_dump(a);
    if (a.cmd == "compress") {
      if (a.out.empty()) throw std::invalid_argument("--out required");
      return cmd_compress(a);
    }
    if (a.cmd == "bench") return cmd_bench(a);
    throw std::invalid_argument("unknown command " + a.cmd);
  } catch (const std::exception& e) {
    fprintf(stderr, "ref_driver error: %s\n", e.what());
    return 1;
  }
}
