#include "model.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <numbers>
#include <thread>

namespace orx {

// ---- config ---------------------------------------------------------------------

orx_config config_default() {  // PolicyConfig{} defaults, policy.hpp:36-85
  orx_config c{};
  c.n_layers = 4;
  c.d_model = 128;
  c.ffn_hidden = 256;
  c.n_heads = 4;
  c.moe_enabled = 0;
  c.n_experts = 0;
  c.experts_active = 0;
  c.moe_location = 0;
  c.expert_round_multiple = 128;
  c.n_code_layers = 3;
  c.codebook_size = 64;
  c.short_len = 20;
  c.positive_len = 256;
  c.lifelong_len = 2000;
  c.n_queries = 128;
  c.lifelong_blocks = 2;
  c.vid_vocab = 4096;
  c.aid_vocab = 256;
  c.uid_vocab = 1024;
  c.gender_vocab = 3;
  c.age_vocab = 8;
  c.n_label_flags = 5;  // kNumObjectives, world.hpp:15
  c.use_sid_history = 0;
  c.vid_only_features = 0;
  c.compress_threshold = 8;
  c.moe_bias_update = 1e-3;
  c.seed = 123;
  return c;
}

orx_config config_preset(const std::string& name) {
  orx_config c = config_default();
  if (name == "tiny") {  // test_policy.cpp:14-32
    c.n_layers = 4; c.d_model = 16; c.ffn_hidden = 32; c.n_heads = 2; c.n_code_layers = 3;
    c.codebook_size = 8; c.short_len = 4; c.positive_len = 4; c.lifelong_len = 8; c.n_queries = 2;
    c.lifelong_blocks = 1; c.vid_vocab = 64; c.aid_vocab = 16; c.uid_vocab = 32; c.seed = 9;
  } else if (name == "0.015B") {  // PAPER.md:398-413 (Table 2)
    c.n_layers = 4; c.d_model = 128; c.ffn_hidden = 256; c.n_heads = 4; c.codebook_size = 8192;
  } else if (name == "0.121B") {
    c.n_layers = 8; c.d_model = 1024; c.ffn_hidden = 2048; c.n_heads = 8; c.codebook_size = 8192;
  } else if (name == "0.935B") {
    c.n_layers = 8; c.d_model = 1024; c.ffn_hidden = 2048; c.n_heads = 8; c.codebook_size = 8192;
    c.moe_enabled = 1; c.n_experts = 24; c.experts_active = 2;
  } else if (name == "2.633B") {
    c.n_layers = 24; c.d_model = 1024; c.ffn_hidden = 2048; c.n_heads = 8; c.codebook_size = 8192;
    c.moe_enabled = 1; c.n_experts = 24; c.experts_active = 4; c.moe_location = 1;
  } else if (name != "default") {
    throw InvalidArgument("unknown config preset: " + name);
  }
  return c;
}

int expert_hidden_size(int d_model, int multiple) {
  require(multiple >= 1, "expert_hidden_size: multiple must be >= 1");
  int raw = (2 * 4 * d_model + 2) / 3;
  return ((raw + multiple - 1) / multiple) * multiple;
}

void validate_config(const orx_config& c) {
  require(c.n_layers >= 2, "policy needs at least one encoder and one decoder layer");  // policy.cpp:60
  require(c.d_model > 0 && c.n_heads >= 1 && c.d_model % c.n_heads == 0, "heads must divide d_model");
  require(c.n_code_layers >= 1 && c.codebook_size >= 1, "bad code geometry");
  require(c.short_len >= 0 && c.positive_len >= 0 && c.lifelong_len >= 1 && c.n_queries >= 1, "bad lengths");
  if (c.moe_enabled)
    require(c.experts_active >= 1 && c.experts_active <= c.n_experts, "moe: need 1 <= k <= n_experts");
  require(c.n_label_flags >= 1 && c.n_label_flags <= 32, "bad n_label_flags");
}

namespace {

std::string fmt_double(double v) {  // shortest round-trip form
  char buf[40];
  for (int prec = 1; prec <= 17; ++prec) {
    snprintf(buf, sizeof buf, "%.*g", prec, v);
    if (strtod(buf, nullptr) == v) break;
  }
  std::string s(buf);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

// Minimal flat JSON object parser: string keys -> number / bool / string.
std::map<std::string, std::string> parse_flat_json(const std::string& s) {
  std::map<std::string, std::string> out;
  size_t i = 0;
  auto ws = [&] { while (i < s.size() && isspace(static_cast<unsigned char>(s[i]))) ++i; };
  auto str = [&]() {
    if (s[i] != '"') throw RuntimeError("config json: expected string");
    ++i;
    std::string r;
    while (i < s.size() && s[i] != '"') r += s[i++];
    ++i;
    return r;
  };
  ws();
  if (i >= s.size() || s[i] != '{') throw RuntimeError("config json: expected object");
  ++i;
  for (;;) {
    ws();
    if (s[i] == '}') break;
    std::string k = str();
    ws();
    if (s[i] != ':') throw RuntimeError("config json: expected ':'");
    ++i;
    ws();
    std::string v;
    if (s[i] == '"') v = str();
    else
      while (i < s.size() && s[i] != ',' && s[i] != '}' && !isspace(static_cast<unsigned char>(s[i]))) v += s[i++];
    out[k] = v;
    ws();
    if (s[i] == ',') ++i;
  }
  return out;
}

}  // namespace

// Same keys as config_json (policy.cpp:347-375); sorted like nlohmann's dump().
std::string config_to_json(const orx_config& c) {
  std::map<std::string, std::string> kv;
  auto b = [](int v) { return std::string(v ? "true" : "false"); };
  kv["n_layers"] = std::to_string(c.n_layers);
  kv["d_model"] = std::to_string(c.d_model);
  kv["ffn_hidden"] = std::to_string(c.ffn_hidden);
  kv["n_heads"] = std::to_string(c.n_heads);
  kv["moe_enabled"] = b(c.moe_enabled);
  kv["n_experts"] = std::to_string(c.n_experts);
  kv["experts_active"] = std::to_string(c.experts_active);
  kv["moe_location"] = c.moe_location == 0 ? "\"decoder\"" : "\"enc_and_dec\"";
  kv["expert_round_multiple"] = std::to_string(c.expert_round_multiple);
  kv["n_code_layers"] = std::to_string(c.n_code_layers);
  kv["codebook_size"] = std::to_string(c.codebook_size);
  kv["short_len"] = std::to_string(c.short_len);
  kv["positive_len"] = std::to_string(c.positive_len);
  kv["lifelong_len"] = std::to_string(c.lifelong_len);
  kv["n_queries"] = std::to_string(c.n_queries);
  kv["lifelong_blocks"] = std::to_string(c.lifelong_blocks);
  kv["vid_vocab"] = std::to_string(c.vid_vocab);
  kv["aid_vocab"] = std::to_string(c.aid_vocab);
  kv["uid_vocab"] = std::to_string(c.uid_vocab);
  kv["gender_vocab"] = std::to_string(c.gender_vocab);
  kv["age_vocab"] = std::to_string(c.age_vocab);
  kv["n_label_flags"] = std::to_string(c.n_label_flags);
  kv["use_sid_history"] = b(c.use_sid_history);
  kv["vid_only_features"] = b(c.vid_only_features);
  kv["compress_threshold"] = std::to_string(c.compress_threshold);
  kv["moe_bias_update"] = fmt_double(c.moe_bias_update);
  kv["seed"] = std::to_string(c.seed);
  std::string s = "{";
  bool first = true;
  for (auto& [k, v] : kv) {
    if (!first) s += ",";
    first = false;
    s += "\"" + k + "\":" + v;
  }
  return s + "}";
}

orx_config config_from_json(const std::string& js) {  // config_from_json, policy.cpp:377-407
  auto kv = parse_flat_json(js);
  auto get = [&](const char* k) -> const std::string& {
    auto it = kv.find(k);
    if (it == kv.end()) throw RuntimeError(std::string("config json missing key ") + k);
    return it->second;
  };
  auto i = [&](const char* k) { return static_cast<int32_t>(std::stoll(get(k))); };
  auto bl = [&](const char* k) { return get(k) == "true" ? 1 : 0; };
  orx_config c = config_default();
  c.n_layers = i("n_layers");
  c.d_model = i("d_model");
  c.ffn_hidden = i("ffn_hidden");
  c.n_heads = i("n_heads");
  c.moe_enabled = bl("moe_enabled");
  c.n_experts = i("n_experts");
  c.experts_active = i("experts_active");
  c.moe_location = get("moe_location") == "decoder" ? 0 : 1;
  c.expert_round_multiple = i("expert_round_multiple");
  c.n_code_layers = i("n_code_layers");
  c.codebook_size = i("codebook_size");
  c.short_len = i("short_len");
  c.positive_len = i("positive_len");
  c.lifelong_len = i("lifelong_len");
  c.n_queries = i("n_queries");
  c.lifelong_blocks = i("lifelong_blocks");
  c.vid_vocab = i("vid_vocab");
  c.aid_vocab = i("aid_vocab");
  c.uid_vocab = i("uid_vocab");
  c.gender_vocab = i("gender_vocab");
  c.age_vocab = i("age_vocab");
  c.n_label_flags = i("n_label_flags");
  c.use_sid_history = bl("use_sid_history");
  c.vid_only_features = kv.count("vid_only_features") ? bl("vid_only_features") : 0;
  c.compress_threshold = i("compress_threshold");
  c.moe_bias_update = std::stod(get("moe_bias_update"));
  c.seed = std::stoull(get("seed"));
  return c;
}

// ---- Rng: xoshiro256** seeded by splitmix64 (rng.cpp:11-77) -------------------------------

namespace {
uint64_t splitmix64(uint64_t& x) {
  x += 0x9e3779b97f4a7c15ULL;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
}  // namespace

Rng::Rng(uint64_t seed) {
  uint64_t x = seed;
  for (auto& s : s_) s = splitmix64(x);
}

uint64_t Rng::next_u64() {
  uint64_t result = rotl(s_[1] * 5, 7) * 9;
  uint64_t t = s_[1] << 17;
  s_[2] ^= s_[0];
  s_[3] ^= s_[1];
  s_[1] ^= s_[2];
  s_[0] ^= s_[3];
  s_[2] ^= t;
  s_[3] = rotl(s_[3], 45);
  return result;
}

double Rng::uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

double Rng::normal() {
  if (has_cached_normal_) {
    has_cached_normal_ = false;
    return cached_normal_;
  }
  double u1 = uniform();
  while (u1 <= 0.0) u1 = uniform();
  double u2 = uniform();
  double r = std::sqrt(-2.0 * std::log(u1));
  double a = 2.0 * std::numbers::pi * u2;
  cached_normal_ = r * std::sin(a);
  has_cached_normal_ = true;
  return r * std::cos(a);
}

int64_t Rng::randint(int64_t n) {
  if (n <= 0) throw InvalidArgument("randint: n must be positive");
  uint64_t un = static_cast<uint64_t>(n);
  uint64_t limit = UINT64_MAX - UINT64_MAX % un;
  uint64_t v = next_u64();
  while (v >= limit) v = next_u64();
  return static_cast<int64_t>(v % un);
}

Rng Rng::split(uint64_t id) const {
  uint64_t x = s_[0] ^ (s_[3] + 0x632be59bd9b4e019ULL);
  uint64_t mix = x;
  uint64_t h = splitmix64(mix) ^ (id * 0xff51afd7ed558ccdULL + 1);
  return Rng(h);
}

// ---- parameter inventory, constructor order of policy.cpp:59-137 -------------------------

std::vector<ParamSpec> param_specs(const orx_config& c) {
  validate_config(c);
  std::vector<ParamSpec> p;
  const int d = c.d_model;
  auto normal = [&](const std::string& n, int r, int k, double sd) { p.push_back({n, r, k, Init::Normal, sd}); };
  auto table = [&](const std::string& n, int vocab, int dim) { normal(n, vocab, dim, 1.0 / std::sqrt(double(dim))); };
  auto linear = [&](const std::string& n, int in, int out, bool bias) {  // make_linear, nn.cpp:8-16
    normal(n + ".w", in, out, 1.0 / std::sqrt(double(in)));
    if (bias) p.push_back({n + ".b", 1, out, Init::Zeros, 0});
  };
  auto mlp = [&](const std::string& n, int in, int hid, int out) {  // make_mlp, nn.cpp:24-30
    linear(n + ".fc1", in, hid, true);
    linear(n + ".fc2", hid, out, true);
  };
  auto norm = [&](const std::string& n) { p.push_back({n + ".gain", 1, d, Init::Ones, 0}); };
  auto attn = [&](const std::string& n) {  // make_attention, nn.cpp:44-54
    linear(n + ".wq", d, d, false);
    linear(n + ".wk", d, d, false);
    linear(n + ".wv", d, d, false);
    linear(n + ".wo", d, d, false);
  };
  auto ffn = [&](const std::string& n) { mlp(n, d, c.ffn_hidden, d); };  // make_ffn, nn.cpp:64-69
  auto moe = [&](const std::string& n) {                                   // make_moe, nn.cpp:102-115
    linear(n + ".gate", d, c.n_experts, false);
    p.push_back({n + ".routing_bias", 1, c.n_experts, Init::Zeros, 0});
    int h = expert_hidden(c);
    for (int e = 0; e < c.n_experts; ++e) {
      std::string en = n + ".expert" + std::to_string(e);
      linear(en + ".w1", d, h, false);
      linear(en + ".w3", d, h, false);
      linear(en + ".w2", h, d, false);
    }
  };

  table("emb.uid", c.uid_vocab, static_dim(c));
  table("emb.gender", c.gender_vocab, static_dim(c));
  table("emb.age", c.age_vocab, static_dim(c));
  table("emb.vid", c.vid_vocab, d);
  table("emb.aid", c.aid_vocab, aid_dim(c));
  table("emb.label", c.n_label_flags, minor_dim(c));
  normal("emb.tag", 2, minor_dim(c), 0.5);
  normal("emb.ts", 2, minor_dim(c), 0.5);
  normal("emb.playtime", 2, minor_dim(c), 0.5);
  normal("emb.duration", 2, minor_dim(c), 0.5);
  p.push_back({"pad.short", 1, d, Init::Zeros, 0});
  p.push_back({"pad.positive", 1, d, Init::Zeros, 0});
  p.push_back({"pad.lifelong", 1, d, Init::Zeros, 0});
  normal("emb.pos", enc_seq_len(c), d, 1.0 / std::sqrt(double(d)));
  int feat = feat_dim(c);
  mlp("pathway.static", 3 * static_dim(c), d, d);
  mlp("pathway.short", feat, d, d);
  mlp("pathway.positive", feat, d, d);
  mlp("pathway.lifelong", feat, d, d);
  normal("lifelong.queries", c.n_queries, d, 1.0 / std::sqrt(double(d)));
  for (int b = 0; b < c.lifelong_blocks; ++b) {  // make_qformer_block, nn.cpp:88-95
    std::string n = "lifelong.block" + std::to_string(b);
    attn(n + ".attn");
    norm(n + ".norm");
    ffn(n + ".ffn");
  }
  for (int l = 0; l < enc_layers(c); ++l) {
    std::string n = "enc" + std::to_string(l);
    norm(n + ".n1");
    norm(n + ".n2");
    attn(n + ".attn");
    if (enc_moe(c)) moe(n + ".moe");
    else ffn(n + ".ffn");
  }
  normal("dec.bos", 1, d, 1.0 / std::sqrt(double(d)));
  for (int l = 0; l < c.n_code_layers; ++l) table("dec.tokens" + std::to_string(l), c.codebook_size, d);
  for (int l = 0; l < c.n_code_layers; ++l) linear("dec.head" + std::to_string(l), d, c.codebook_size, false);
  for (int l = 0; l < dec_layers(c); ++l) {
    std::string n = "dec" + std::to_string(l);
    norm(n + ".n1");
    norm(n + ".n2");
    norm(n + ".n3");
    attn(n + ".self");
    attn(n + ".cross");
    if (c.moe_enabled) moe(n + ".moe");
    else ffn(n + ".ffn");
  }
  return p;
}

const Tensor& HostWeights::get(const std::string& name) const {
  auto it = index.find(name);
  if (it == index.end()) throw InvalidArgument("unknown parameter: " + name);
  return tensors[static_cast<size_t>(it->second)];
}

// Seeded init, bit-identical to normal_init over one Rng(cfg.seed) stream
// (params.cpp:84-88). Box-Muller pairs consume two u64 draws and yield
// (cos, sin) values in that order, so normal #j is fixed by draws 2*(j/2)
// and 2*(j/2)+1; a sequential pass records the generator state every chunk
// and worker threads fill chunks in parallel.
HostWeights HostWeights::random(const orx_config& cfg, int ep_rank, int ep_world, const int32_t* owner) {
  HostWeights w;
  w.cfg = cfg;
  auto specs = param_specs(cfg);
  // expert parallelism: materialise only this rank's experts (the stream is
  // still laid out over every parameter, so kept values are bit-identical)
  auto kept = [&](const std::string& name) {
    if (ep_world <= 1) return true;
    const size_t at = name.find(".expert");
    if (at == std::string::npos) return true;
    const int e = std::atoi(name.c_str() + at + 7);
    if (!owner) return e / (cfg.n_experts / ep_world) == ep_rank;
    // "enc<l>.moe..." / "dec<l>.moe...": MoE layer index in engine order (moe_layers)
    const int l = std::atoi(name.c_str() + 3);
    const int li = name.compare(0, 3, "enc") == 0 ? l : (enc_moe(cfg) ? enc_layers(cfg) : 0) + l;
    const int32_t o = owner[static_cast<size_t>(li) * cfg.n_experts + e];
    return o < 0 || o == ep_rank;
  };
  if (ep_world > 1) {
    require(cfg.moe_enabled && cfg.n_experts % ep_world == 0, "experts must divide evenly over the ranks");
    require(ep_rank >= 0 && ep_rank < ep_world, "expert-parallel rank outside the world");
    w.partial = true;
  }
  std::vector<std::pair<float*, int64_t>> normal_dst;  // (ptr, count) per Normal tensor, in order
  std::vector<double> normal_sd;
  int64_t n_normal = 0;
  for (auto& s : specs) {
    Tensor t;
    t.name = s.name;
    t.rows = s.rows;
    t.cols = s.cols;
    if (kept(s.name)) t.data.assign(static_cast<size_t>(s.rows) * s.cols, s.init == Init::Ones ? 1.f : 0.f);
    w.index[s.name] = static_cast<int>(w.tensors.size());
    w.tensors.push_back(std::move(t));
  }
  for (size_t i = 0; i < specs.size(); ++i)
    if (specs[i].init == Init::Normal) {
      const int64_t n = static_cast<int64_t>(specs[i].rows) * specs[i].cols;
      normal_dst.push_back({w.tensors[i].data.empty() ? nullptr : w.tensors[i].data.data(), n});
      normal_sd.push_back(specs[i].stddev);
      n_normal += n;
    }
  const int64_t n_pairs = (n_normal + 1) / 2;
  const int64_t chunk_pairs = int64_t(1) << 21;
  const int64_t n_chunks = (n_pairs + chunk_pairs - 1) / chunk_pairs;
  std::vector<Rng> starts;
  starts.reserve(static_cast<size_t>(n_chunks));
  Rng rng(cfg.seed);
  for (int64_t ch = 0; ch < n_chunks; ++ch) {
    starts.push_back(rng);
    int64_t np = std::min(chunk_pairs, n_pairs - ch * chunk_pairs);
    for (int64_t i = 0; i < 2 * np; ++i) rng.next_u64();
  }
  // normal index -> tensor lookup via prefix offsets
  std::vector<int64_t> prefix(normal_dst.size() + 1, 0);
  for (size_t i = 0; i < normal_dst.size(); ++i) prefix[i + 1] = prefix[i] + normal_dst[i].second;
  bool retry_hit = false;
  auto work = [&](int64_t ch) {
    Rng r = starts[static_cast<size_t>(ch)];
    int64_t j0 = ch * chunk_pairs * 2, j1 = std::min(n_normal, j0 + chunk_pairs * 2);
    size_t ti = static_cast<size_t>(std::upper_bound(prefix.begin(), prefix.end(), j0) - prefix.begin() - 1);
    {  // skip chunks that only cover tensors this process does not keep
      bool any = false;
      for (size_t t2 = ti; t2 < normal_dst.size() && prefix[t2] < j1; ++t2) any = any || normal_dst[t2].first;
      if (!any) return;
    }
    for (int64_t j = j0; j < j1; j += 2) {
      double u1 = r.uniform();
      double u2 = r.uniform();
      if (u1 <= 0.0) {
        retry_hit = true;
        return;
      }
      double rad = std::sqrt(-2.0 * std::log(u1));
      double a = 2.0 * std::numbers::pi * u2;
      double v[2] = {rad * std::cos(a), rad * std::sin(a)};
      for (int q = 0; q < 2 && j + q < j1; ++q) {
        int64_t jj = j + q;
        while (jj >= prefix[ti + 1]) ++ti;
        if (normal_dst[ti].first) normal_dst[ti].first[jj - prefix[ti]] = static_cast<float>(0.0 + normal_sd[ti] * v[q]);
      }
    }
  };
  unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  std::atomic<int64_t> next{0};
  for (unsigned t = 0; t < nt; ++t)
    pool.emplace_back([&] {
      for (int64_t ch; (ch = next.fetch_add(1)) < n_chunks;) work(ch);
    });
  for (auto& th : pool) th.join();
  if (retry_hit) {  // u1 == 0 (p = 2^-53 per pair): fall back to the sequential stream
    Rng r(cfg.seed);
    for (size_t i = 0; i < normal_dst.size(); ++i)
      for (int64_t k = 0; k < normal_dst[i].second; ++k) {
        const float v = static_cast<float>(0.0 + normal_sd[i] * r.normal());
        if (normal_dst[i].first) normal_dst[i].first[k] = v;
      }
  }
  return w;
}

// ---- GRCP (policy.cpp:344-443; io.cpp:22-95) ---------------------------------------------

namespace {
struct Reader {
  std::ifstream in;
  std::string path;
  template <class T>
  T pod() {
    T v;
    in.read(reinterpret_cast<char*>(&v), sizeof v);
    if (!in) throw RuntimeError("truncated file: " + path);
    return v;
  }
  std::string str() {
    uint64_t n = pod<uint64_t>();
    std::string s(n, '\0');
    in.read(s.data(), static_cast<std::streamsize>(n));
    if (!in) throw RuntimeError("truncated file: " + path);
    return s;
  }
};
}  // namespace

HostWeights HostWeights::load_grcp(const std::string& path) {
  Reader r{std::ifstream(path, std::ios::binary), path};
  if (!r.in) throw RuntimeError("cannot open for reading: " + path);
  char magic[4];
  r.in.read(magic, 4);
  if (!r.in || memcmp(magic, "GRCP", 4) != 0) throw RuntimeError("bad magic bytes in " + path);
  uint32_t version = r.pod<uint32_t>();
  require(version == 1, "unsupported checkpoint version");
  HostWeights w;
  w.cfg = config_from_json(r.str());
  auto specs = param_specs(w.cfg);
  uint64_t count = r.pod<uint64_t>();
  require(count == specs.size(), "checkpoint parameter count mismatch");
  for (auto& s : specs) {
    Tensor t;
    t.name = s.name;
    t.rows = s.rows;
    t.cols = s.cols;
    w.index[s.name] = static_cast<int>(w.tensors.size());
    w.tensors.push_back(std::move(t));
  }
  std::vector<double> buf;
  std::vector<bool> seen(specs.size(), false);
  for (uint64_t i = 0; i < count; ++i) {
    std::string name = r.str();
    uint32_t nd = r.pod<uint32_t>();
    std::vector<uint32_t> dims(nd);
    for (auto& x : dims) x = r.pod<uint32_t>();
    auto it = w.index.find(name);
    require(it != w.index.end(), "checkpoint has unknown parameter: " + name);
    Tensor& t = w.tensors[static_cast<size_t>(it->second)];
    int64_t n = 1;
    for (auto x : dims) n *= x;
    bool same = (nd == 2 && int(dims[0]) == t.rows && int(dims[1]) == t.cols) ||
                (nd == 1 && t.rows == 1 && int(dims[0]) == t.cols);
    require(same, "checkpoint shape mismatch for " + name);
    buf.resize(static_cast<size_t>(n));
    r.in.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(n * 8));
    if (!r.in) throw RuntimeError("truncated file: " + path);
    t.data.resize(static_cast<size_t>(n));
    for (int64_t k = 0; k < n; ++k) {
      if (!std::isfinite(buf[static_cast<size_t>(k)])) throw RuntimeError("non-finite value in checkpoint: " + name);
      t.data[static_cast<size_t>(k)] = static_cast<float>(buf[static_cast<size_t>(k)]);
    }
    seen[static_cast<size_t>(it->second)] = true;
  }
  for (size_t i = 0; i < seen.size(); ++i) require(seen[i], "checkpoint lacks parameter " + specs[i].name);
  return w;
}

void HostWeights::save_grcp(const std::string& path) const {
  require(!partial, "cannot save an expert-parallel shard of the weights as a GRCP checkpoint");
  std::ofstream out(path, std::ios::binary);
  if (!out) throw RuntimeError("cannot open for writing: " + path);
  auto pod = [&](auto v) { out.write(reinterpret_cast<const char*>(&v), sizeof v); };
  auto str = [&](const std::string& s) {
    pod(static_cast<uint64_t>(s.size()));
    out.write(s.data(), static_cast<std::streamsize>(s.size()));
  };
  out.write("GRCP", 4);
  pod(static_cast<uint32_t>(1));
  str(config_to_json(cfg));
  pod(static_cast<uint64_t>(tensors.size()));
  std::vector<double> buf;
  for (auto& t : tensors) {
    str(t.name);
    pod(static_cast<uint32_t>(2));
    pod(static_cast<uint32_t>(t.rows));
    pod(static_cast<uint32_t>(t.cols));
    buf.assign(t.data.begin(), t.data.end());
    out.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(buf.size() * 8));
  }
  out.close();
  if (!out.good()) throw RuntimeError("write failed: " + path);
}

}  // namespace orx
