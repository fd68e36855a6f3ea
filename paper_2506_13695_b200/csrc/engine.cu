// Engine: device weights, activation arena and the per-batch forward flows.
//
//   encode        PolicyModel::encode (policy.cpp:254-265): pathway MLPs,
//                 lifelong QFormer, + pos_emb, L_enc pre-norm blocks.
//   decode_step   one beam position for all live rows: PolicyModel::decode
//                 (policy.cpp:267-288) with a per-position K/V cache for the
//                 causal self-attention and a per-user cross-K/V cache of
//                 z_enc computed once (nn.cpp:59-60 recomputes it per call),
//                 then position_logits (policy.cpp:290-295).
//   beam_search   generation.cpp:41-88 batched over users: decode_step ->
//                 row log-softmax + top-k -> per-user merge, depth times.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <type_traits>

#include "attention.cuh"
#include "beam.cuh"
#include "engine.hpp"
#include "ep_plan.hpp"
#include "nccl_dl.hpp"
#include "gemm.cuh"
#include "kernels.cuh"

namespace orx {

void launch_beam_init(int users, BeamState& st, cudaStream_t s);

namespace {

#define CUDA_CHECK(x)                                                                              \
  do {                                                                                             \
    cudaError_t e__ = (x);                                                                         \
    if (e__ != cudaSuccess) throw RuntimeError(std::string("CUDA: ") + cudaGetErrorString(e__) +  \
                                               " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

#define NCCL_CHECK(x)                                                                                      \
  do {                                                                                                     \
    ncclResult_t r__ = (x);                                                                                \
    if (r__ != ncclSuccess) throw RuntimeError(std::string("NCCL: ") + nccl().GetErrorString(r__) + " at " + \
                                               __FILE__ + ":" + std::to_string(__LINE__));                 \
  } while (0)

inline int rup(int x, int m) { return (x + m - 1) / m * m; }

template <class T>
T to_t(float v) {
  if constexpr (std::is_same_v<T, float>) return v;
  else return __float2bfloat16_rn(v);
}

// Device arena: one cudaMalloc per buffer, freed with the engine.
struct Arena {
  std::vector<void*> ptrs;
  template <class X>
  X* alloc(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    CUDA_CHECK(cudaMalloc(&p, n * sizeof(X)));
    ptrs.push_back(p);
    return static_cast<X*>(p);
  }
  void reset() {
    for (void* p : ptrs) cudaFree(p);
    ptrs.clear();
  }
  ~Arena() { reset(); }
};

template <class T>
struct Lin {  // y = x . W, W^T packed [N][K] (K padded to 8, zeros)
  const T* w = nullptr;
  int N = 0, K = 0;
  const float* bias = nullptr;
};

struct MoeW {
  const float* gate_t = nullptr;  // [E][d]
  const float* gate_gain = nullptr;  // [E][d] gate_t[e][c] * (pre-MoE RMSNorm gain)[c]
  const float* gate_sw = nullptr;    // gate_gain in moe_route4's swizzled shared-memory layout (E <= 24)
  const float* gate_hi = nullptr;    // bf16 engine: [32][d] tf32 hi / fp32 residual of gate_gain (route_tc.cu)
  const float* gate_lo = nullptr;
  const float* bias = nullptr;    // [E]
  const void* w13 = nullptr;      // bf16: [E][2h][d] interleaved per 128 rows; fp32: w1 [E][h][d]
  const void* w3 = nullptr;       // fp32 only: [E][h][d]
  const void* w2 = nullptr;       // [E][d][h]
  // expert parallelism: this MoE layer's placement tables (ep_plan.hpp) and
  // accumulated per-expert loads
  int li = 0;
  const int32_t* ep_owner = nullptr;  // [E]
  const int32_t* ep_slot = nullptr;   // [E]
  const int32_t* ep_list = nullptr;   // [W][C]
  long long* ep_load = nullptr;       // [E]
};

}  // namespace

void validate_batch(const orx_config& cfg, const orx_user_batch& b) {  // validate_context, policy.cpp:23-38
  require(b.n_users >= 0, "negative user count");
  // messages are only built on failure (this runs over every record of every request)
  auto fail = [](const char* name, const char* what) { throw InvalidArgument(std::string(name) + what); };
  const uint32_t label_limit = cfg.n_label_flags >= 32 ? 0u : (1u << cfg.n_label_flags);
  auto check = [&](const orx_records& r, int cap, const char* name) {
    if (b.n_users == 0) return;
    if (!r.offsets) fail(name, ": offsets required");
    if (r.offsets[0] != 0) fail(name, ": offsets must start at 0");
    for (int u = 0; u < b.n_users; ++u) {
      const int64_t s = r.offsets[u], e = r.offsets[u + 1];
      if (e < s) fail(name, ": offsets must be non-decreasing");
      if (e - s > cap) fail(name, " sequence exceeds its configured cap");
      for (int64_t i = s; i < e; ++i) {
        if (i > s && !(r.ts[i] >= r.ts[i - 1])) fail(name, " sequence not time-ordered");
        if (!(r.playtime[i] <= r.duration[i] * 1.0 + 1e-6)) throw InvalidArgument("playtime exceeds duration");
        if (label_limit && r.labels[i] >= label_limit) throw InvalidArgument("label bits outside defined flags");
        if (cfg.use_sid_history) {
          if (!r.sid) throw InvalidArgument("sid history enabled but record lacks semantic id codes");
          for (int l = 0; l < cfg.n_code_layers; ++l) {
            const int c = r.sid[i * cfg.n_code_layers + l];
            if (c < 0 || c >= cfg.codebook_size) throw InvalidArgument("sid code outside its layer vocabulary");
          }
        }
      }
    }
  };
  check(b.short_seq, cfg.short_len, "short");
  check(b.positive_seq, cfg.positive_len, "positive");
  check(b.lifelong_seq, cfg.lifelong_len, "lifelong");
}

namespace {

// The per-record part of validate_batch for users [u0, u1) of one sequence,
// as a non-throwing predicate (the request packers run it in parallel; on a
// failure the sequential validate_batch re-runs to raise the first error in
// the reference's order). Offsets must already be known to be valid.
bool records_ok(const orx_config& cfg, const orx_records& r, int u0, int u1) {
  const uint32_t label_limit = cfg.n_label_flags >= 32 ? 0u : (1u << cfg.n_label_flags);
  const int64_t i0 = r.offsets[u0], i1 = r.offsets[u1];
  bool ok = true;
  for (int u = u0; u < u1; ++u) {
    const int64_t s = r.offsets[u], e = r.offsets[u + 1];
    for (int64_t i = s + 1; i < e; ++i) ok &= r.ts[i] >= r.ts[i - 1];
  }
  for (int64_t i = i0; i < i1; ++i) {
    ok &= r.playtime[i] <= r.duration[i] * 1.0 + 1e-6;
    if (label_limit) ok &= static_cast<uint32_t>(r.labels[i]) < label_limit;
  }
  if (cfg.use_sid_history) {
    if (i1 > i0 && !r.sid) return false;
    const int L = cfg.n_code_layers;
    for (int64_t i = i0 * L; i < i1 * L; ++i) ok &= r.sid[i] >= 0 && r.sid[i] < cfg.codebook_size;
  }
  return ok;
}

// Write back and evict [p, p + n) from the CPU caches. The pinned stage is
// packed by many cores; a DMA read of lines still dirty in several cores'
// caches runs at ~6 GB/s on the B200 hosts, after a flush at ~53 GB/s
// (12.6 MB: 2.2 ms -> 0.24 ms, measured with profiles/h2d_flush_probe.cu).
#if defined(__x86_64__)
__attribute__((target("clflushopt"))) void flush_lines(const void* p, size_t n) {
  const char* c = static_cast<const char*>(p);
  const char* e = c + n;
  for (c = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(c) & ~uintptr_t(63)); c < e; c += 64)
    __builtin_ia32_clflushopt(c);
  __builtin_ia32_sfence();
}
#else
void flush_lines(const void*, size_t) {}
#endif

// hashed (policy.cpp:14-17): id mod vocab in [0, vocab)
inline int32_t host_hashed(int64_t id, int vocab) {
  const int64_t m = id % vocab;
  return static_cast<int32_t>(m < 0 ? m + vocab : m);
}

bool offsets_ok(const orx_config& cfg, const orx_user_batch& b) {
  const orx_records* rs[3] = {&b.short_seq, &b.positive_seq, &b.lifelong_seq};
  const int caps[3] = {cfg.short_len, cfg.positive_len, cfg.lifelong_len};
  for (int p = 0; p < 3; ++p) {
    const orx_records& r = *rs[p];
    if (!r.offsets || r.offsets[0] != 0) return false;
    for (int u = 0; u < b.n_users; ++u)
      if (r.offsets[u + 1] < r.offsets[u] || r.offsets[u + 1] - r.offsets[u] > caps[p]) return false;
  }
  return true;
}

// Persistent host workers for request packing (thread start-up would cost
// more than the packing slice of a small request).
class WorkerPool {
 public:
  explicit WorkerPool(int n) {
    for (int w = 1; w < n; ++w) threads_.emplace_back([this, w] { loop(w); });
    n_ = n;
  }
  ~WorkerPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  int size() const { return n_; }
  // fn(w) for w in [0, n) on n threads (the caller runs w = 0); returns when all are done
  void run(int n, const std::function<void(int)>& fn) {
    n = std::max(1, std::min(n, n_));
    {
      std::lock_guard<std::mutex> g(m_);
      fn_ = &fn;
      active_ = n;
      pending_ = n - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void loop(int w) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* fn;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        if (w >= active_) continue;
        fn = fn_;
      }
      (*fn)(w);
      std::lock_guard<std::mutex> g(m_);
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
  std::vector<std::thread> threads_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  uint64_t gen_ = 0;
  int n_ = 1, active_ = 0, pending_ = 0;
  bool stop_ = false;
};

}  // namespace

template <class T>
class EngineT final : public Engine {
  static constexpr bool kBf16 = std::is_same_v<T, __nv_bfloat16>;
  // Expert segments are padded to the grouped GEMM's M tile: 256 rows for the
  // tcgen05 CTA-pair kernel (both CTAs of a pair share one expert's B tile).
  static constexpr int kMoeTile = kBf16 ? 256 : 128;

 public:
  EngineT(const HostWeights& hw, int device, int max_users, int max_width, const EpConfig* ep)
      : cfg_(hw.cfg), dev_(device), maxU_(max_users), maxW_(max_width) {
    CUDA_CHECK(cudaSetDevice(dev_));
    CUDA_CHECK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    El_ = cfg_.moe_enabled ? cfg_.n_experts : 0;
    if (ep && ep->world > 1) {
      require(cfg_.moe_enabled, "expert parallelism needs a MoE config");
      require(ep->rank >= 0 && ep->rank < ep->world, "expert-parallel rank outside the world");
      require(!ep->owner.empty() || cfg_.n_experts % ep->world == 0,
              "expert count must divide evenly over the expert-parallel ranks");
      require(ep->owner.empty() || ep->owner.size() == static_cast<size_t>(moe_layers(cfg_)) * cfg_.n_experts,
              "expert placement must have moe_layers * n_experts entries");
      ep_rank_ = ep->rank;
      ep_world_ = ep->world;
      const int nml = moe_layers(cfg_);
      place_ = ep->owner.empty() ? EpPlacement::contiguous(nml, cfg_.n_experts, ep_world_) : EpPlacement{};
      if (!ep->owner.empty()) {
        place_.layers = nml, place_.E = cfg_.n_experts, place_.W = ep_world_;
        place_.owner = ep->owner;
      }
      place_.validate();
      El_ = place_.capacity();  // local expert slots per MoE layer (replicated + owned)
      ncclUniqueId id;
      static_assert(sizeof(id.internal) == 128, "ncclUniqueId size");
      memcpy(id.internal, ep->unique_id, 128);
      NCCL_CHECK(nccl().CommInitRank(&comm_, ep_world_, id, ep_rank_));
    }
    require(max_users >= 1 && max_width >= 1, "engine capacity must be positive");
    require(cfg_.n_code_layers <= 8, "n_code_layers above 8 is not supported");
    require(!cfg_.moe_enabled || cfg_.n_experts <= 32, "more than 32 experts is not supported");
    require(max_width <= 1024, "beam width above 1024 is not supported");
    if (kBf16) {
      require((cfg_.d_model / cfg_.n_heads) % 32 == 0 && cfg_.d_model / cfg_.n_heads <= 128,
              "bf16 mode needs head dim 32, 64 or 128");
      require(!cfg_.moe_enabled || expert_hidden(cfg_) % 128 == 0, "bf16 MoE needs expert hidden % 128 == 0");
    }
    if constexpr (kBf16) tc_attn_ = fmha_supported(cfg_.d_model / cfg_.n_heads) && !getenv("ORX_ATTN_MMA_SYNC");
    upload(hw);
    alloc_activations();
  }
  ~EngineT() override {
    cudaSetDevice(dev_);
    cudaStreamSynchronize(st_);
    report_routing();
    for (auto& g : graphs_) cudaGraphExecDestroy(g.exec);
    for (size_t p = 0; p < ep_peer_base_.size(); ++p)
      if (static_cast<int>(p) != ep_rank_ && ep_peer_base_[p]) cudaIpcCloseMemHandle(ep_peer_base_[p]);
    if (ep_region_) cudaFree(ep_region_);
    if (comm_) nccl().CommDestroy(comm_);
    for (int k = 0; k < 2; ++k) {
      if (host_stage_[k]) cudaFreeHost(host_stage_[k]);
      if (host_out_[k]) cudaFreeHost(host_out_[k]);
      cudaEventDestroy(h2d_done_[k]);
      cudaEventDestroy(dev_free_[k]);
      cudaEventDestroy(out_ready_[k]);
    }
    cudaStreamDestroy(cs_);
    cudaStreamDestroy(st_);
  }

  // The reference checks every tape value (tape.cpp:29); host outputs are
  // checked here, the beam search by its device flag (BeamState::nonfinite).
  template <class X>
  static void require_finite(const X* p, size_t n) {
    for (size_t i = 0; i < n; ++i)
      if (!std::isfinite(p[i])) throw RuntimeError("non-finite value produced on tape");
  }

  void expert_load(int64_t* out, bool reset) override {
    require_idle();
    const size_t E = cfg_.n_experts;
    if (moe_layers(cfg_) == 0) return;
    std::fill(out, out + static_cast<size_t>(moe_layers(cfg_)) * E, int64_t(0));
    CUDA_CHECK(cudaStreamSynchronize(st_));
    for (size_t li = 0; li < ep_loads_.size(); ++li) {
      static_assert(sizeof(long long) == sizeof(int64_t), "load counters are 64-bit");
      CUDA_CHECK(cudaMemcpy(out + li * E, ep_loads_[li], E * 8, cudaMemcpyDeviceToHost));
      if (reset) CUDA_CHECK(cudaMemset(ep_loads_[li], 0, E * 8));
    }
  }
  void* stream() override { return st_; }
  void require_idle() const override {
    require(pending_.empty(), "a submitted beam search is in flight: collect it before synchronous calls");
  }

  // ------------------------------------------------------------------------
  // weights
  // ------------------------------------------------------------------------
  const float* upload_f32(const float* src, size_t n) {
    float* d = ar_.alloc<float>(n);
    CUDA_CHECK(cudaMemcpy(d, src, n * 4, cudaMemcpyHostToDevice));
    return d;
  }
  const float* up(const HostWeights& hw, const std::string& name) {
    const Tensor& t = hw.get(name);
    return upload_f32(t.data.data(), t.data.size());
  }
  // Pack several (in, out) row-major weights side by side along N: W^T [sum N][Kp].
  Lin<T> pack(const HostWeights& hw, const std::vector<std::string>& names, const std::string& bias = "",
              const std::string& in_gain = "") {
    const Tensor& f = hw.get(names[0]);
    const float* gk = in_gain.empty() ? nullptr : hw.get(in_gain).data.data();  // RMSNorm gain folded into W rows
    int K = f.rows, N = 0;
    for (auto& n : names) {
      require(hw.get(n).rows == K, "pack: inner dims differ");
      N += hw.get(n).cols;
    }
    int Kp = rup(K, 8);
    std::vector<T> h(static_cast<size_t>(N) * Kp, to_t<T>(0.f));
    int n0 = 0;
    for (auto& n : names) {
      const Tensor& t = hw.get(n);
      for (int k = 0; k < K; ++k)
        for (int j = 0; j < t.cols; ++j)
          h[static_cast<size_t>(n0 + j) * Kp + k] = to_t<T>(gk ? gk[k] * t.data[(size_t)k * t.cols + j]
                                                               : t.data[(size_t)k * t.cols + j]);
      n0 += t.cols;
    }
    T* d = ar_.alloc<T>(h.size());
    CUDA_CHECK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    Lin<T> L;
    L.w = d;
    L.N = N;
    L.K = Kp;
    if (!bias.empty()) L.bias = up(hw, bias);
    return L;
  }
  // Lifelong keys only feed the QFormer's K / V projections (policy.cpp:233-238,
  // nn.cpp:97-100): K|V = (H W2 + b2) Wkv = H (W2 Wkv) + b2 Wkv, H the pathway's
  // LeakyReLU hidden rows. W2 Wkv is formed once here (fp32 SIMT GEMM, one bf16
  // rounding), so the pathway's fc2 GEMM and its key rows disappear from the
  // encoder; empty-history users' pad key (pad.lifelong, not an fc2 output) gets
  // pad Wkv written by launch_fill_kv_pad.
  void build_kv_fold(const HostWeights& hw, const std::vector<std::string>& kv) {
    const int d = cfg_.d_model, nkv = static_cast<int>(kv.size()) * d;
    const Tensor& W2 = hw.get("pathway.lifelong.fc2.w");  // (in, out) = [d][d]
    const Tensor& b2 = hw.get("pathway.lifelong.fc2.b");
    const Tensor& pad = hw.get("pad.lifelong");
    require(W2.rows == d && W2.cols == d, "kv fold: unexpected fc2 shape");
    std::vector<float> at(static_cast<size_t>(nkv) * d);  // Wkv^T [nkv][d]
    std::vector<double> c(nkv, 0.0), pk(nkv, 0.0);
    int n0 = 0;
    for (const auto& name : kv) {
      const Tensor& t = hw.get(name);  // (in, out) = [d][d]
      for (int k = 0; k < d; ++k)
        for (int j = 0; j < t.cols; ++j) {
          const float w = t.data[(size_t)k * t.cols + j];
          at[(size_t)(n0 + j) * d + k] = w;
          c[n0 + j] += double(b2.data[k]) * w;
          pk[n0 + j] += double(pad.data[k]) * w;
        }
      n0 += t.cols;
    }
    float* dA = ar_.alloc<float>(at.size());
    float* dB = ar_.alloc<float>(W2.data.size());
    float* dC = ar_.alloc<float>(static_cast<size_t>(nkv) * d);
    CUDA_CHECK(cudaMemcpy(dA, at.data(), at.size() * 4, cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(dB, W2.data.data(), W2.data.size() * 4, cudaMemcpyHostToDevice));
    Epi ef;
    ef.out = dC;
    ef.ldo = d;
    ef.n_out = d;
    ef.m_valid = nkv;
    gemm_f32(dA, d, dB, d, nkv, d, d, ef, nullptr, st_);  // C[m][n] = sum_k Wkv[k][m] W2[n][k] = (W2 Wkv)^T
    T* w = ar_.alloc<T>(static_cast<size_t>(nkv) * d);
    launch_convert<T>(nkv, d, dC, d, w, d, st_);
    CUDA_CHECK(cudaStreamSynchronize(st_));
    kvf_.w = w;
    kvf_.N = nkv;
    kvf_.K = d;
    std::vector<float> cf(c.begin(), c.end()), pf(pk.begin(), pk.end());
    kvf_.bias = upload_f32(cf.data(), cf.size());
    kv_pad_ = upload_f32(pf.data(), pf.size());
    kv_fold_ = true;
  }

  MoeW pack_moe(const HostWeights& hw, const std::string& n, const std::string& gain_name) {
    const int d = cfg_.d_model, E = cfg_.n_experts, El = El_, h = expert_hidden(cfg_);
    MoeW m;
    const Tensor& g = hw.get(n + ".gate.w");  // (d, E)
    std::vector<float> gt(static_cast<size_t>(E) * d);
    for (int k = 0; k < d; ++k)
      for (int e = 0; e < E; ++e) gt[(size_t)e * d + k] = g.data[(size_t)k * E + e];
    m.gate_t = upload_f32(gt.data(), gt.size());
    const Tensor& gain = hw.get(gain_name);
    for (int e = 0; e < E; ++e)
      for (int k = 0; k < d; ++k) gt[(size_t)e * d + k] *= gain.data[k];
    m.gate_gain = upload_f32(gt.data(), gt.size());
    if (E <= 24 && d % 128 == 0) {  // moe_route4's swizzled shared-memory layout
      std::vector<float> sw(static_cast<size_t>(d) * 24);
      gate_route4_layout(gt.data(), E, d, sw.data());
      m.gate_sw = upload_f32(sw.data(), sw.size());
    }
    if (kBf16 && moe_route_tc_supported(d, E, cfg_.experts_active, d) && !getenv("ORX_ROUTE_SIMT")) {
      // 3xTF32 gate for the tensor-pipe router: tf32-exact hi part and the fp32 residual, 32 expert rows
      std::vector<float> hi(static_cast<size_t>(32) * d), lo(static_cast<size_t>(32) * d);
      gate_tf32_split(gt.data(), E, d, hi.data(), lo.data());
      m.gate_hi = upload_f32(hi.data(), hi.size());
      m.gate_lo = upload_f32(lo.data(), lo.size());
    }
    m.bias = up(hw, n + ".routing_bias");
    const int dp = rup(d, 8), hp = rup(h, 8);
    // this rank's expert slots (all experts without expert parallelism): slot e -> global expert
    m.li = n_moe_++;
    std::vector<int> glob(static_cast<size_t>(El));
    if (ep_world_ > 1) {
      const std::vector<int> l = place_.local(m.li, ep_rank_);
      for (int e = 0; e < El; ++e) glob[e] = e < static_cast<int>(l.size()) ? l[e] : -1;
      std::vector<int32_t> list, slot;
      place_.tables(El, list, slot);
      const size_t W = ep_world_;
      int32_t* t = ar_.alloc<int32_t>(2 * static_cast<size_t>(E) + W * El);
      CUDA_CHECK(cudaMemcpy(t, place_.owner.data() + static_cast<size_t>(m.li) * E, E * 4, cudaMemcpyHostToDevice));
      CUDA_CHECK(cudaMemcpy(t + E, slot.data() + static_cast<size_t>(m.li) * E, E * 4, cudaMemcpyHostToDevice));
      CUDA_CHECK(cudaMemcpy(t + 2 * E, list.data() + static_cast<size_t>(m.li) * W * El, W * El * 4,
                            cudaMemcpyHostToDevice));
      m.ep_owner = t, m.ep_slot = t + E, m.ep_list = t + 2 * E;
      m.ep_load = ar_.alloc<long long>(E);
      CUDA_CHECK(cudaMemset(m.ep_load, 0, E * sizeof(long long)));
      ep_loads_.push_back(m.ep_load);
    } else {
      for (int e = 0; e < El; ++e) glob[e] = e;
    }
    auto ex = [&](int e, const char* w) -> const Tensor& {  // empty slots (glob < 0) stay zero
      return hw.get(n + ".expert" + std::to_string(glob[e]) + "." + w + ".w");
    };
    if (kBf16) {
      // folded RMSNorm (fold_norm_): the pre-MoE norm's gain goes into W1|W3's input
      // rows; the tokens arrive un-normalised (or gain-free normalised) and are scaled
      // per row in the SwiGLU epilogue (Epi::row_rsq) or by an explicit ones-gain norm
      std::vector<float> g(static_cast<size_t>(d), 1.f);
      if (fold_norm_) g.assign(gain.data.begin(), gain.data.end());
      std::vector<T> w13(static_cast<size_t>(El) * 2 * h * dp, to_t<T>(0.f));
      for (int e = 0; e < El; ++e) {
        if (glob[e] < 0) continue;
        const Tensor& w1 = ex(e, "w1");
        const Tensor& w3 = ex(e, "w3");
        for (int j = 0; j < h; ++j) {
          // output column j -> block j/128; W1 rows first, then W3 rows, per 256-row tile
          size_t r1 = (size_t)e * 2 * h + (j / 128) * 256 + (j % 128);
          size_t r3 = r1 + 128;
          for (int k = 0; k < d; ++k) {
            w13[r1 * dp + k] = to_t<T>(w1.data[(size_t)k * h + j] * g[k]);
            w13[r3 * dp + k] = to_t<T>(w3.data[(size_t)k * h + j] * g[k]);
          }
        }
      }
      T* p = ar_.alloc<T>(w13.size());
      CUDA_CHECK(cudaMemcpy(p, w13.data(), w13.size() * sizeof(T), cudaMemcpyHostToDevice));
      m.w13 = p;
    } else {
      for (int which = 0; which < 2; ++which) {
        std::vector<T> w(static_cast<size_t>(El) * h * dp, to_t<T>(0.f));
        for (int e = 0; e < El; ++e) {
          if (glob[e] < 0) continue;
          const Tensor& t = ex(e, which == 0 ? "w1" : "w3");
          for (int j = 0; j < h; ++j)
            for (int k = 0; k < d; ++k) w[((size_t)e * h + j) * dp + k] = to_t<T>(t.data[(size_t)k * h + j]);
        }
        T* p = ar_.alloc<T>(w.size());
        CUDA_CHECK(cudaMemcpy(p, w.data(), w.size() * sizeof(T), cudaMemcpyHostToDevice));
        (which == 0 ? m.w13 : m.w3) = p;
      }
    }
    std::vector<T> w2(static_cast<size_t>(El) * d * hp, to_t<T>(0.f));
    for (int e = 0; e < El; ++e) {
      if (glob[e] < 0) continue;
      const Tensor& t = ex(e, "w2");  // (h, d)
      for (int k = 0; k < h; ++k)
        for (int j = 0; j < d; ++j) w2[((size_t)e * d + j) * hp + k] = to_t<T>(t.data[(size_t)k * d + j]);
    }
    T* p = ar_.alloc<T>(w2.size());
    CUDA_CHECK(cudaMemcpy(p, w2.data(), w2.size() * sizeof(T), cudaMemcpyHostToDevice));
    m.w2 = p;
    return m;
  }

  struct Mlp { Lin<T> fc1, fc2; };
  // tc_attn_ (bf16, head dim 64/128): V is projected by its own GEMM whose
  // epilogue writes it transposed per (user, head) for the tcgen05 attention
  struct QBlock { Lin<T> wq, wkv, wo, fc1, fc2; const float* gain; };
  struct EncL { const float *n1, *n2; Lin<T> wqkv, wo, fc1, fc2; MoeW moe; };
  struct DecL { const float *n1, *n2, *n3; Lin<T> sqkv, so, cq, co, fc1, fc2; MoeW moe; };

  // fc1 of a record pathway is linear in each feature section (policy.cpp:139-216):
  //   features(r) . W1 = vid_row . W1[0:d] + aid_row . W1[d:d+ad]
  //                    + sum_f (x_f w_f + b_f) . W1[sec_f] + sum_b lab_b label_b . W1[sec_lab]
  // so the vid / aid products become [vocab][d] tables (two GEMMs over the
  // bf16 tables, once per engine) and the scalar / label sections d-vectors
  // (f64 on the host). The per-record fc1 GEMM and the n x 2.125d feature rows
  // are replaced by a gather-add (launch_fold_features).
  FoldTables build_fold(const HostWeights& hw, const std::string& n, const Mlp& m) {
    const orx_config& c = cfg_;
    const int d = c.d_model, ad = aid_dim(c), mn = minor_dim(c), nf = c.n_label_flags;
    const Tensor& W = hw.get(n + ".fc1.w");  // [F][d] (in, out)
    require(W.cols == d && W.rows == d + ad + 5 * mn && m.fc1.K >= d + ad, "fold: unexpected fc1 shape");
    const int nvid = hw.get("emb.vid").rows, naid = hw.get("emb.aid").rows;
    FoldTables f;
    f.d = d;
    f.n_flags = nf;
    float* pv = ar_.alloc<float>(static_cast<size_t>(nvid) * d);
    float* pa = ar_.alloc<float>(static_cast<size_t>(naid) * d);
    Epi ev = epi(pv, d, true);
    ev.n_out = d;
    ev.m_valid = nvid;
    gemm_bf16(t_vid16_, d, m.fc1.w, m.fc1.K, nvid, d, d, ev, nullptr, st_);
    Epi ea = epi(pa, d, true);
    ea.n_out = d;
    ea.m_valid = naid;
    gemm_bf16(t_aid16_, ad, m.fc1.w + d, m.fc1.K, naid, d, ad, ea, nullptr, st_);
    std::vector<double> u(static_cast<size_t>(4) * d, 0.0), c0(d, 0.0), lab(static_cast<size_t>(nf) * d, 0.0);
    auto axpy = [&](double a, int k, double* y) {
      const float* r = W.data.data() + static_cast<size_t>(k) * d;
      for (int j = 0; j < d; ++j) y[j] += a * r[j];
    };
    const char* sec[4] = {"emb.tag", "emb.ts", "emb.playtime", "emb.duration"};
    for (int s = 0; s < 4; ++s) {
      const Tensor& t = hw.get(sec[s]);  // [2][minor]: w row, b row
      for (int j = 0; j < mn; ++j) {
        axpy(t.data[j], d + ad + s * mn + j, u.data() + static_cast<size_t>(s) * d);
        axpy(t.data[mn + j], d + ad + s * mn + j, c0.data());
      }
    }
    const Tensor& L = hw.get("emb.label");  // [n_flags][minor]
    for (int b = 0; b < nf; ++b)
      for (int j = 0; j < mn; ++j)
        axpy(L.data[static_cast<size_t>(b) * mn + j], d + ad + 4 * mn + j, lab.data() + static_cast<size_t>(b) * d);
    const Tensor& bias = hw.get(n + ".fc1.b");
    for (int j = 0; j < d; ++j) c0[j] += bias.data[j];
    // every label combination (labels < 2^n_flags, policy.cpp:33) with the constant part folded in
    std::vector<float> pl(static_cast<size_t>(d) << nf);
    for (int m = 0; m < (1 << nf); ++m)
      for (int j = 0; j < d; ++j) {
        double acc = c0[j];
        for (int b = 0; b < nf; ++b)
          if ((m >> b) & 1) acc += lab[static_cast<size_t>(b) * d + j];
        pl[static_cast<size_t>(m) * d + j] = static_cast<float>(acc);
      }
    std::vector<float> uf(u.begin(), u.end());
    f.pv = pv;
    f.pa = pa;
    f.pl = upload_f32(pl.data(), pl.size());
    f.u = upload_f32(uf.data(), uf.size());
    // aid x label-combination rows pre-added (<= 64 MB): one L2 gather less per record
    const size_t pal_rows = static_cast<size_t>(naid) << nf;
    if (pal_rows * d * 4 <= (size_t(64) << 20) && !getenv("ORX_NO_FOLD_PAL")) {
      float* pal = ar_.alloc<float>(pal_rows * d);
      launch_fold_pal(naid, nf, d, pa, f.pl, pal, st_);
      CUDA_CHECK(cudaGetLastError());
      f.pal = pal;
    }
    CUDA_CHECK(cudaStreamSynchronize(st_));
    return f;
  }

  void upload(const HostWeights& hw) {
    const orx_config& c = cfg_;
    if constexpr (kBf16) fold_norm_ = c.d_model % 256 == 0 && !getenv("ORX_NO_NORM_FOLD");
    if (fold_norm_) {
      std::vector<float> ones(c.d_model, 1.f);
      ones_ = upload_f32(ones.data(), ones.size());
    }
    auto mlp = [&](const std::string& n) {
      return Mlp{pack(hw, {n + ".fc1.w"}, n + ".fc1.b"), pack(hw, {n + ".fc2.w"}, n + ".fc2.b")};
    };
    t_uid_ = up(hw, "emb.uid");
    t_gender_ = up(hw, "emb.gender");
    t_age_ = up(hw, "emb.age");
    t_vid_ = up(hw, "emb.vid");
    t_aid_ = up(hw, "emb.aid");
    if constexpr (kBf16) {  // bf16 copies for the feature-row gathers
      auto up16 = [&](const std::string& n) {
        const Tensor& t = hw.get(n);
        std::vector<T> h(t.data.size());
        for (size_t i = 0; i < h.size(); ++i) h[i] = to_t<T>(t.data[i]);
        T* p = ar_.alloc<T>(h.size());
        CUDA_CHECK(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
        return p;
      };
      t_vid16_ = up16("emb.vid");
      t_aid16_ = up16("emb.aid");
    }
    t_label_ = up(hw, "emb.label");
    t_tag_ = up(hw, "emb.tag");
    t_ts_ = up(hw, "emb.ts");
    t_play_ = up(hw, "emb.playtime");
    t_dur_ = up(hw, "emb.duration");
    pad_s_ = up(hw, "pad.short");
    pad_p_ = up(hw, "pad.positive");
    pad_l_ = up(hw, "pad.lifelong");
    pos_ = up(hw, "emb.pos");
    bos_ = up(hw, "dec.bos");
    for (int l = 0; l < c.n_code_layers; ++l) {
      tokens_.push_back(up(hw, "dec.tokens" + std::to_string(l)));
      heads_.push_back(pack(hw, {"dec.head" + std::to_string(l) + ".w"}));
    }
    p_static_ = mlp("pathway.static");
    p_short_ = mlp("pathway.short");
    p_pos_ = mlp("pathway.positive");
    p_life_ = mlp("pathway.lifelong");
    if constexpr (kBf16) {
      // The fold pays only while one pathway's folded vid/aid tables stay
      // L2-resident (126 MB L2): above a 48 MB budget per pathway (e.g. a
      // production-size vid vocabulary) the explicit feature rows + fc1 GEMM
      // path is used instead.
      const double fold_bytes = double(c.vid_vocab + c.aid_vocab) * c.d_model * 4.0;
      fold_on_ = !c.use_sid_history && !c.vid_only_features && aid_dim(c) % 8 == 0 &&
                 fold_features_supported(c.d_model, c.n_label_flags) && fold_bytes <= 48.0 * (1 << 20) &&
                 !getenv("ORX_NO_FEATURE_FOLD");
      if (getenv("ORX_VERBOSE"))
        fprintf(stderr, "orx: pathway fc1 fold %s (folded tables %.1f MB per pathway)\n", fold_on_ ? "on" : "off",
                fold_bytes / (1 << 20));
      if (fold_on_) {
        fold_[0] = build_fold(hw, "pathway.short", p_short_);
        fold_[1] = build_fold(hw, "pathway.positive", p_pos_);
        fold_[2] = build_fold(hw, "pathway.lifelong", p_life_);
      }
    }
    {  // lifelong.queries as a GEMM operand [Nq][d]
      const Tensor& q = hw.get("lifelong.queries");
      std::vector<T> h(q.data.size());
      for (size_t i = 0; i < h.size(); ++i) h[i] = to_t<T>(q.data[i]);
      T* p = ar_.alloc<T>(h.size());
      CUDA_CHECK(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
      queries_ = p;
    }
    for (int b = 0; b < c.lifelong_blocks; ++b) {
      std::string n = "lifelong.block" + std::to_string(b);
      QBlock q;
      q.wq = pack(hw, {n + ".attn.wq.w"});
      if (!tc_attn_) q.wkv = pack(hw, {n + ".attn.wk.w", n + ".attn.wv.w"});
      q.wo = pack(hw, {n + ".attn.wo.w"});
      q.gain = up(hw, n + ".norm.gain");
      q.fc1 = pack(hw, {n + ".ffn.fc1.w"}, n + ".ffn.fc1.b", fold_norm_ ? n + ".norm.gain" : "");
      q.fc2 = pack(hw, {n + ".ffn.fc2.w"}, n + ".ffn.fc2.b");
      qblocks_.push_back(q);
    }
    if (tc_attn_ && c.lifelong_blocks > 0) {  // the keys are the same for every block: one K|V GEMM for all
      std::vector<std::string> kv;
      for (int b = 0; b < c.lifelong_blocks; ++b) kv.push_back("lifelong.block" + std::to_string(b) + ".attn.wk.w");
      for (int b = 0; b < c.lifelong_blocks; ++b) kv.push_back("lifelong.block" + std::to_string(b) + ".attn.wv.w");
      qkv_all_ = pack(hw, kv);
      if constexpr (kBf16) {
        if (!getenv("ORX_NO_KV_FOLD")) build_kv_fold(hw, kv);
      }
    }
    for (int l = 0; l < enc_layers(c); ++l) {
      std::string n = "enc" + std::to_string(l);
      EncL e;
      e.n1 = up(hw, n + ".n1.gain");
      e.n2 = up(hw, n + ".n2.gain");
      e.wqkv = pack(hw, {n + ".attn.wq.w", n + ".attn.wk.w", n + ".attn.wv.w"}, "",
                    fold_norm_ ? n + ".n1.gain" : "");  // tcgen05 path: V transposed
      e.wo = pack(hw, {n + ".attn.wo.w"});
      if (enc_moe(c)) e.moe = pack_moe(hw, n + ".moe", n + ".n2.gain");
      else {
        e.fc1 = pack(hw, {n + ".ffn.fc1.w"}, n + ".ffn.fc1.b", fold_norm_ ? n + ".n2.gain" : "");
        e.fc2 = pack(hw, {n + ".ffn.fc2.w"}, n + ".ffn.fc2.b");
      }
      enc_.push_back(e);
    }
    std::vector<std::string> xkv;
    for (int l = 0; l < dec_layers(c); ++l) {
      std::string n = "dec" + std::to_string(l);
      DecL e;
      e.n1 = up(hw, n + ".n1.gain");
      e.n2 = up(hw, n + ".n2.gain");
      e.n3 = up(hw, n + ".n3.gain");
      e.sqkv = pack(hw, {n + ".self.wq.w", n + ".self.wk.w", n + ".self.wv.w"});
      e.so = pack(hw, {n + ".self.wo.w"});
      e.cq = pack(hw, {n + ".cross.wq.w"}, "", fold_norm_ ? n + ".n2.gain" : "");
      e.co = pack(hw, {n + ".cross.wo.w"});
      xkv.push_back(n + ".cross.wk.w");
      xkv.push_back(n + ".cross.wv.w");
      if (c.moe_enabled) e.moe = pack_moe(hw, n + ".moe", n + ".n3.gain");
      else {
        e.fc1 = pack(hw, {n + ".ffn.fc1.w"}, n + ".ffn.fc1.b", fold_norm_ ? n + ".n3.gain" : "");
        e.fc2 = pack(hw, {n + ".ffn.fc2.w"}, n + ".ffn.fc2.b");
      }
      dec_.push_back(e);
    }
    if (tc_attn_) {  // one GEMM: all layers' cross K, then all layers' cross V (stored transposed)
      std::vector<std::string> kv;
      for (size_t i = 0; i < xkv.size(); i += 2) kv.push_back(xkv[i]);
      for (size_t i = 1; i < xkv.size(); i += 2) kv.push_back(xkv[i]);
      xkv_w_ = pack(hw, kv);
    } else {
      xkv_w_ = pack(hw, xkv);  // all decoder layers' cross K|V in one GEMM
    }
  }

  // ------------------------------------------------------------------------
  // activations
  // ------------------------------------------------------------------------
  void alloc_activations() {
    const orx_config& c = cfg_;
    const int d = c.d_model, U = maxU_, Tn = enc_seq_len(c), Nq = c.n_queries, L = c.n_code_layers;
    const int Ld = dec_layers(c);
    Rd_ = static_cast<int64_t>(U) * maxW_;
    const int64_t rec_max = static_cast<int64_t>(U) * std::max({c.short_len, c.positive_len, c.lifelong_len, 1});
    const int64_t keys_max = static_cast<int64_t>(U) * std::max(c.lifelong_len, 1);
    const int64_t rows_enc = static_cast<int64_t>(U) * Tn;
    const int64_t rows_big = std::max<int64_t>({rows_enc, Rd_, static_cast<int64_t>(U) * Nq});
    Fp_ = rup(feat_dim(c), 8);
    Sp_ = rup(3 * static_dim(c), 8);
    feat_ = ar_.alloc<T>(static_cast<size_t>(std::max<int64_t>(rec_max, U)) * std::max(Fp_, Sp_));
    hid_ = ar_.alloc<T>(static_cast<size_t>(std::max<int64_t>(rec_max, U)) * d);
    keys_ = ar_.alloc<T>(static_cast<size_t>(keys_max) * d);
    const int nqb = std::max(c.lifelong_blocks, 1);
    kvl_ = ar_.alloc<T>(static_cast<size_t>(keys_max) * std::max(2, nqb) * d);  // tcgen05: K of every QFormer block
    z_ = ar_.alloc<float>(static_cast<size_t>(rows_enc) * d);
    xn_ = ar_.alloc<T>(static_cast<size_t>(rows_big) * d);
    if (fold_norm_) {  // per-row sum-of-squares partials of the folded RMSNorms: 2 per 256 output columns
      ssq_ld_ = rows_big;
      ssq_ = ar_.alloc<float>(static_cast<size_t>(2 * d / 256) * rows_big);
    }
    qkv_ = ar_.alloc<T>(static_cast<size_t>(rows_big) * 3 * d);
    att_ = ar_.alloc<T>(static_cast<size_t>(rows_big) * d);
    ffh_ = ar_.alloc<T>(static_cast<size_t>(rows_big) * c.ffn_hidden);
    qproj_ = ar_.alloc<T>(static_cast<size_t>(U) * Nq * d);
    qo_ = ar_.alloc<float>(static_cast<size_t>(U) * Nq * d);
    qcur_ = ar_.alloc<T>(static_cast<size_t>(U) * Nq * d);
    zt_ = kBf16 ? ar_.alloc<T>(static_cast<size_t>(rows_enc) * d) : reinterpret_cast<T*>(z_);
    xkv_ = ar_.alloc<T>(static_cast<size_t>(rows_enc) * 2 * d * Ld);
    if (tc_attn_) {  // transposed V operands, zero padding columns stay finite
      Tpad_ = rup(Tn, 8);
      Lpad_ = rup(std::max(c.lifelong_len, 1), 8);
      vt_enc_ = ar_.alloc<T>(static_cast<size_t>(U) * d * Tpad_);
      vt_q_ = ar_.alloc<T>(static_cast<size_t>(nqb) * U * d * Lpad_);  // V^T of every QFormer block
      vt_x_ = ar_.alloc<T>(static_cast<size_t>(Ld) * U * d * Tpad_);
      CUDA_CHECK(cudaMemset(vt_enc_, 0, static_cast<size_t>(U) * d * Tpad_ * sizeof(T)));
      CUDA_CHECK(cudaMemset(vt_q_, 0, static_cast<size_t>(nqb) * U * d * Lpad_ * sizeof(T)));
      CUDA_CHECK(cudaMemset(vt_x_, 0, static_cast<size_t>(Ld) * U * d * Tpad_ * sizeof(T)));
    }
    h_ = ar_.alloc<float>(static_cast<size_t>(Rd_) * d);
    // self-attention K/V cache: each (position, layer) keeps its own QKV GEMM output
    // [rows][3d]; later positions read the K|V columns of their ancestor rows there
    for (int p = 0; p < L * Ld; ++p) kvpos_.push_back(ar_.alloc<T>(static_cast<size_t>(Rd_) * 3 * d));
    kvpos_ptrs_ = ar_.alloc<T*>(static_cast<size_t>(L) * Ld);
    CUDA_CHECK(cudaMemcpy(kvpos_ptrs_, kvpos_.data(), static_cast<size_t>(L) * Ld * sizeof(T*), cudaMemcpyHostToDevice));
    logits_ = ar_.alloc<float>(static_cast<size_t>(Rd_) * c.codebook_size);
    const int ksel = std::min(maxW_, c.codebook_size);
    cand_ = ar_.alloc<uint64_t>(static_cast<size_t>(Rd_) * ksel);
    lse_ = ar_.alloc<float>(Rd_);
    if constexpr (kBf16) {  // fused log-softmax + beam selection from the head GEMM's chunk statistics
      fused_select_ = c.codebook_size % 256 == 0 && maxW_ <= 1024 && !getenv("ORX_NO_FUSED_SELECT");
      if (fused_select_) {
        head_stats_ = ar_.alloc<float2>(static_cast<size_t>(Rd_) * (c.codebook_size / 32));
        const size_t words = beam_select_scratch_words(std::min(maxW_, c.codebook_size), c.codebook_size);
        if (words) sel_scratch_ = ar_.alloc<uint32_t>(words * maxU_);
      }
    }
    topk_fail_ = ar_.alloc<int32_t>(Rd_ + 1);
    for (int s = 0; s < 2; ++s) {
      bs_[s].codes = ar_.alloc<int32_t>(static_cast<size_t>(Rd_) * L);
      bs_[s].score = ar_.alloc<float>(Rd_);
      bs_[s].score64 = ar_.alloc<double>(Rd_);
      bs_[s].lexrank = ar_.alloc<int32_t>(Rd_);
      bs_[s].lex2beam = ar_.alloc<int32_t>(Rd_);
      bs_[s].anc = ar_.alloc<int32_t>(static_cast<size_t>(Rd_) * L);
      node_[s] = ar_.alloc<int32_t>(Rd_);
    }
    nonfinite_ = ar_.alloc<int32_t>(4);
    bs_[0].nonfinite = bs_[1].nonfinite = nonfinite_;
    tf_anc_ = ar_.alloc<int32_t>(static_cast<size_t>(Rd_) * L);
    seq_acc_ = ar_.alloc<double>(Rd_);
    tf_codes_ = ar_.alloc<int32_t>(static_cast<size_t>(Rd_) * L);
    grp_start_ = ar_.alloc<int32_t>(Rd_ + 1);
    grp_len_ = ar_.alloc<int32_t>(Rd_ + 1);
    grp_kstart_ = ar_.alloc<int32_t>(Rd_ + 1);
    grp_user_ = ar_.alloc<int32_t>(Rd_ + 1);
    if (c.moe_enabled) {
      const int E = c.n_experts, k = c.experts_active, h = expert_hidden(c);
      const int64_t mrows = std::max(rows_enc, Rd_);
      // grouped rows: this rank's own (token, expert) pairs, or with expert
      // parallelism everything any rank may send here, + per-expert padding
      const int64_t grouped = mrows * k * ep_world_;
      S_ = grouped + static_cast<int64_t>(El_) * kMoeTile;
      max_tiles_ = static_cast<int>(S_ / kMoeTile + 1);
      sel_ = ar_.alloc<int32_t>(mrows * k);
      wts_ = ar_.alloc<float>(mrows * k);
      slot_ = ar_.alloc<int32_t>(mrows * k);
      // routing histogram | scatter fill counters | the split-K router's per-tile tickets,
      // zeroed together once per forward pass (zero_moe_counters)
      n_route_tickets_ = kBf16 ? static_cast<int>((mrows + 127) / 128) : 0;
      counts_ = ar_.alloc<int32_t>(2 * static_cast<size_t>(E) + n_route_tickets_);
      CUDA_CHECK(cudaMemset(counts_, 0, (2 * static_cast<size_t>(E) + n_route_tickets_) * 4));
      if constexpr (kBf16) {  // split-K tensor-pipe router: per-(tile, K half) partials
        route_part_ = ar_.alloc<float>(moe_route_tc_scratch_floats(static_cast<int>(mrows)));
        route_ticket_ = counts_ + 2 * E;
      }
      cursor_ = ar_.alloc<int32_t>(E);
      tile_expert_ = ar_.alloc<int32_t>(max_tiles_);
      n_mtiles_ = ar_.alloc<int32_t>(1);
      row_scale_ = ar_.alloc<float>(S_);
      if (fold_norm_) row_rsq_ = ar_.alloc<float>(S_);
      xg_ = ar_.alloc<T>(static_cast<size_t>(S_) * d);
      hg_ = ar_.alloc<T>(static_cast<size_t>(S_) * rup(h, 8));
      yg_ = ar_.alloc<T>(static_cast<size_t>(S_) * d);
      CUDA_CHECK(cudaMemset(xg_, 0, static_cast<size_t>(S_) * d * sizeof(T)));
      if (!kBf16) {
        ga_ = ar_.alloc<float>(static_cast<size_t>(S_) * h);
        gb_ = ar_.alloc<float>(static_cast<size_t>(S_) * h);
      }
      if (ep_world_ > 1) setup_ep_exchange(mrows * k, S_);
    }
    // user batch staging: two slots (pinned host + device), grown on demand; a
    // copy stream moves slot s while the compute stream still runs the other
    CUDA_CHECK(cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      CUDA_CHECK(cudaEventCreateWithFlags(&h2d_done_[k], cudaEventDisableTiming));
      CUDA_CHECK(cudaEventCreateWithFlags(&dev_free_[k], cudaEventDisableTiming));
      CUDA_CHECK(cudaEventCreateWithFlags(&out_ready_[k], cudaEventDisableTiming));
    }
  }

  // ------------------------------------------------------------------------
  // GEMM helper
  // ------------------------------------------------------------------------
  Epi epi(void* out, int ldo, bool out_f32) {
    Epi e;
    e.out = out;
    e.ldo = ldo;
    e.out_bf16 = (!out_f32 && kBf16) ? 1 : 0;
    return e;
  }
  // epilogue writing V transposed per (user, head) for the tcgen05 attention:
  // vt[layer][u][c][t] with t the key position (rows r -> (r / T, r % T) or maps)
  Epi vt_epi(T* vt, int ld, int T_rows, const int32_t* row_user, const int32_t* row_pos, long long layer_stride) {
    Epi e;
    e.vt = vt;
    e.vt_ld = ld;
    e.vt_T = T_rows;
    e.vt_cols = cfg_.d_model;
    e.vt_user_stride = static_cast<long long>(cfg_.d_model) * ld;
    e.vt_layer_stride = layer_stride;
    e.vt_row_user = row_user;
    e.vt_row_pos = row_pos;
    e.out_bf16 = 1;
    return e;
  }
  // split K|V GEMM: columns [0, vt_col0) to out (ldo), the rest transposed as in `vt`
  static Epi split_epi(Epi vt, void* out, int ldo, int vt_col0) {
    vt.out = out;
    vt.ldo = ldo;
    vt.vt_col0 = vt_col0;
    return vt;
  }
  FmhaArgs fmha(int B, int max_q, const T* Q, long long q_rows, int ldq, const T* K, long long k_rows, int ldk,
                int k_col0, const T* Vt, int vt_users, int vt_ld, const int32_t* vt_user, Seg q, Seg k, Seg o,
                double flops) {
    FmhaArgs f;
    f.B = B;
    f.max_q = max_q;
    f.heads = cfg_.n_heads;
    f.dh = cfg_.d_model / cfg_.n_heads;
    f.Q = Q;
    f.q_rows = q_rows;
    f.ldq = ldq;
    f.K = K;
    f.k_rows = k_rows;
    f.ldk = ldk;
    f.k_col0 = k_col0;
    f.Vt = Vt;
    f.vt_rows = static_cast<long long>(vt_users) * cfg_.d_model;
    f.vt_cols = vt_ld;
    f.vt_ld = vt_ld;
    f.vt_user = vt_user;
    f.O = att_;
    f.ldo = cfg_.d_model;
    f.q = q;
    f.k = k;
    f.o = o;
    f.flops = flops;
    return f;
  }
  void gemm(const T* A, int lda, const Lin<T>& W, int M, Epi e) {
    if (M <= 0) return;
    if (!e.n_out) e.n_out = W.N;
    if (!e.m_valid) e.m_valid = M;
    if (!e.bias) e.bias = W.bias;
    if constexpr (kBf16) gemm_bf16(A, lda, W.w, W.K, M, W.N, W.K, e, nullptr, st_);
    else gemm_f32(A, lda, W.w, W.K, M, W.N, W.K, e, nullptr, st_);
  }

  // ------------------------------------------------------------------------
  // user batch staging: one pinned arena, one H2D copy
  // ------------------------------------------------------------------------
  struct Stage {
    int U = 0;
    int n_rec[3] = {0, 0, 0};  // short, positive, lifelong
    int n_keys = 0;
    int n_pad_keys = 0;
    size_t off_uid, off_gender, off_age, off_ns, off_np, off_kstart, off_klen, off_static_map, off_life_map,
        off_pad_keys, off_key_user, off_key_pos;
    size_t off_vid[3], off_aid[3], off_tag[3], off_ts[3], off_play[3], off_dur[3], off_lab[3], off_sid[3],
        off_map[3];
    size_t bytes = 0;
  } sg_;

  void stage_batch(const orx_user_batch& b) override {
    const auto t_enter = std::chrono::steady_clock::now();
    const orx_config& c = cfg_;
    require(b.n_users >= 0, "negative user count");
    // offsets first (O(users), sequential): the packers below index by them;
    // the per-record checks run inside the packers
    if (!offsets_ok(c, b)) validate_batch(c, b);  // raises the first error in reference order
    require(b.n_users >= 1 && b.n_users <= maxU_, "batch size outside the engine capacity");
    // a slot no submitted (uncollected) request holds; with none in flight,
    // the one not used by the most recent request
    int ss = stage_slot_ ^ 1;
    for (const Pending& p : pending_) ss = p.slot ^ 1;
    require(pending_.size() < 2, "both staging slots hold submitted searches");
    CUDA_CHECK(cudaEventSynchronize(h2d_done_[ss]));  // its previous H2D has read the pinned buffer
    const auto t_synced = std::chrono::steady_clock::now();
    CUDA_CHECK(cudaSetDevice(dev_));
    Stage s;
    s.U = b.n_users;
    const orx_records* rs[3] = {&b.short_seq, &b.positive_seq, &b.lifelong_seq};
    for (int p = 0; p < 3; ++p) s.n_rec[p] = static_cast<int>(rs[p]->offsets[s.U]);
    const int Tn = enc_seq_len(c), Nq = c.n_queries, L = c.n_code_layers;
    size_t off = 0;
    auto take = [&](size_t bytes) {
      size_t o = off;
      off += (bytes + 15) / 16 * 16;
      return o;
    };
    s.off_uid = take(4 * s.U);
    s.off_gender = take(4 * s.U);
    s.off_age = take(4 * s.U);
    s.off_ns = take(4 * s.U);
    s.off_np = take(4 * s.U);
    s.off_kstart = take(4 * s.U);
    s.off_klen = take(4 * s.U);
    s.off_static_map = take(4 * s.U);
    s.off_life_map = take(4 * static_cast<size_t>(s.U) * Nq);
    s.off_pad_keys = take(4 * s.U);
    int64_t n_keys_total = 0;
    for (int u = 0; u < s.U; ++u)
      n_keys_total += std::max<int64_t>(b.lifelong_seq.offsets[u + 1] - b.lifelong_seq.offsets[u], 1);
    s.off_key_user = take(4 * n_keys_total);  // lifelong key row -> (user, position)
    s.off_key_pos = take(4 * n_keys_total);
    for (int p = 0; p < 3; ++p) {
      size_t n = s.n_rec[p];
      s.off_vid[p] = take(4 * n);  // hashed vid row index (policy.cpp:14-17), int32
      s.off_aid[p] = take(4 * n);
      s.off_tag[p] = take(4 * n);
      s.off_ts[p] = take(4 * n);
      s.off_play[p] = take(4 * n);
      s.off_dur[p] = take(4 * n);
      s.off_lab[p] = take(4 * n);
      s.off_sid[p] = take(c.use_sid_history ? 4 * n * L : 0);
      s.off_map[p] = take(4 * n);
    }
    s.bytes = off;
    if (s.bytes > stage_cap_[ss]) {
      if (host_stage_[ss]) cudaFreeHost(host_stage_[ss]);
      CUDA_CHECK(cudaMallocHost(&host_stage_[ss], s.bytes));
      dev_stage_[ss] = ar_.alloc<uint8_t>(s.bytes);
      stage_cap_[ss] = s.bytes;
    }
    uint8_t* H = static_cast<uint8_t*>(host_stage_[ss]);
    auto I32 = [&](size_t o) { return reinterpret_cast<int32_t*>(H + o); };
    auto F32 = [&](size_t o) { return reinterpret_cast<float*>(H + o); };
    for (int u = 0; u < s.U; ++u) {
      I32(s.off_uid)[u] = b.uid[u];
      I32(s.off_gender)[u] = b.gender[u];
      I32(s.off_age)[u] = b.age_bucket[u];
      I32(s.off_ns)[u] = static_cast<int32_t>(b.short_seq.offsets[u + 1] - b.short_seq.offsets[u]);
      I32(s.off_np)[u] = static_cast<int32_t>(b.positive_seq.offsets[u + 1] - b.positive_seq.offsets[u]);
      I32(s.off_static_map)[u] = u * Tn;
      for (int q = 0; q < Nq; ++q) I32(s.off_life_map)[u * Nq + q] = u * Tn + 1 + c.short_len + c.positive_len + q;
    }
    // lifelong key rows: user u owns [kstart, kstart + max(1, n)); empty -> one pad key (policy.cpp:205-207)
    int kpos = 0, npad = 0;
    for (int u = 0; u < s.U; ++u) {
      int n = static_cast<int>(b.lifelong_seq.offsets[u + 1] - b.lifelong_seq.offsets[u]);
      I32(s.off_kstart)[u] = kpos;
      I32(s.off_klen)[u] = std::max(n, 1);
      if (n == 0) I32(s.off_pad_keys)[npad++] = kpos;
      kpos += std::max(n, 1);
    }
    s.n_keys = kpos;
    s.n_pad_keys = npad;
    // Record copy / conversion and row maps, split over user ranges on worker
    // threads (this host packing sits inside every end-to-end request).
    auto pack_users = [&](int u0, int u1) {
      for (int u = u0; u < u1; ++u) {  // key row -> (user, position)
        const int k0 = I32(s.off_kstart)[u], kn = I32(s.off_klen)[u];
        for (int t = 0; t < kn; ++t) {
          I32(s.off_key_user)[k0 + t] = u;
          I32(s.off_key_pos)[k0 + t] = t;
        }
      }
      for (int p = 0; p < 3; ++p) {
        const orx_records& r = *rs[p];
        if (s.n_rec[p] == 0) continue;
        const int64_t i0 = r.offsets[u0], i1 = r.offsets[u1], n = i1 - i0;
        if (n == 0) continue;
        // embedding-row indices hashed here (the 64-bit modulo per record
        // was a third of the device feature kernel's instructions)
        int32_t* vi = I32(s.off_vid[p]);
        int32_t* ai = I32(s.off_aid[p]);
        for (int64_t i = i0; i < i1; ++i) {
          vi[i] = c.use_sid_history ? 0 : host_hashed(r.vid[i], c.vid_vocab);
          ai[i] = host_hashed(r.aid[i], c.aid_vocab);
        }
        memcpy(H + s.off_lab[p] + 4 * i0, r.labels + i0, 4 * n);
        float *tg = F32(s.off_tag[p]), *ts = F32(s.off_ts[p]), *pl = F32(s.off_play[p]), *du = F32(s.off_dur[p]);
        for (int64_t i = i0; i < i1; ++i) {
          tg[i] = static_cast<float>(r.tag[i]);
          ts[i] = static_cast<float>(r.ts[i]);
          pl[i] = static_cast<float>(r.playtime[i]);
          du[i] = static_cast<float>(r.duration[i]);
        }
        if (c.use_sid_history) memcpy(H + s.off_sid[p] + 4 * i0 * L, r.sid + i0 * L, 4 * n * L);
        int32_t* map = I32(s.off_map[p]);
        for (int u = u0; u < u1; ++u) {
          const int64_t b0 = r.offsets[u], e0 = r.offsets[u + 1];
          const int cnt = static_cast<int>(e0 - b0);
          for (int64_t i = b0; i < e0; ++i) {
            const int j = static_cast<int>(i - b0);
            if (p == 0) map[i] = u * Tn + 1 + (c.short_len - cnt) + j;  // left padding, policy.cpp:209-215
            else if (p == 1) map[i] = u * Tn + 1 + c.short_len + (c.positive_len - cnt) + j;
            else map[i] = I32(s.off_kstart)[u] + j;
          }
        }
      }
    };
    const int64_t total_rec = static_cast<int64_t>(s.n_rec[0]) + s.n_rec[1] + s.n_rec[2];
    const auto t_pack0 = std::chrono::steady_clock::now();
    const int n_workers = static_cast<int>(
        std::min<int64_t>({pool_.size(), std::max<int64_t>(1, total_rec / 16384), s.U}));
    std::atomic<bool> rec_ok{true};
    pool_.run(n_workers, [&](int w) {
      const int u0 = s.U * w / n_workers, u1 = s.U * (w + 1) / n_workers;
      bool ok = true;
      for (int p = 0; p < 3; ++p) ok &= records_ok(c, *rs[p], u0, u1);
      if (!ok) {
        rec_ok = false;
        return;
      }
      pack_users(u0, u1);
    });
    if (!rec_ok) validate_batch(c, b);  // raises the first error in reference order
    const int n_flush = static_cast<int>(std::min<int64_t>(pool_.size(), std::max<size_t>(1, s.bytes >> 19)));
    pool_.run(n_flush, [&](int w) {  // stage lines out of the CPU caches before the DMA reads them
      const size_t a = (s.bytes * w / n_flush) & ~size_t(63), e = w + 1 == n_flush ? s.bytes : (s.bytes * (w + 1) / n_flush) & ~size_t(63);
      flush_lines(H + a, e - a);
    });
    static const bool timing = getenv("ORX_STAGE_TIMING") != nullptr;
    if (timing) {
      const auto now = std::chrono::steady_clock::now();
      auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      fprintf(stderr, "stage: validate+sync %.3f ms, layout %.3f ms, %d workers pack %.3f ms\n",
              ms(t_enter, t_synced), ms(t_synced, t_pack0), n_workers, ms(t_pack0, now));
    }
    const auto t_copy0 = std::chrono::steady_clock::now();
    // copy stream: wait until the compute stream no longer reads this slot, copy, and
    // make the compute stream wait for the copy (the other slot's work overlaps it)
    CUDA_CHECK(cudaStreamWaitEvent(cs_, dev_free_[ss], 0));
    CUDA_CHECK(cudaMemcpyAsync(dev_stage_[ss], host_stage_[ss], s.bytes, cudaMemcpyHostToDevice, cs_));
    CUDA_CHECK(cudaEventRecord(h2d_done_[ss], cs_));
    CUDA_CHECK(cudaStreamWaitEvent(st_, h2d_done_[ss], 0));
    if (timing) {
      const auto t1 = std::chrono::steady_clock::now();
      CUDA_CHECK(cudaStreamSynchronize(cs_));
      const auto t2 = std::chrono::steady_clock::now();
      auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      cudaPointerAttributes pa{};
      cudaPointerGetAttributes(&pa, host_stage_[ss]);
      fprintf(stderr, "stage: H2D %zu B issue %.3f ms, complete %.3f ms (host type %d)\n", s.bytes, ms(t_copy0, t1),
              ms(t1, t2), int(pa.type));
    }
    h2d_bytes += static_cast<int64_t>(s.bytes);
    sg_ = s;
    stage_slot_ = ss;
    staged_ = true;
  }
  template <class X>
  const X* dp(size_t off) const {
    return reinterpret_cast<const X*>(dev_stage_[stage_slot_] + off);
  }
  RecordsDev recs(int p) const {
    RecordsDev r;
    r.n = sg_.n_rec[p];
    r.vid = dp<int32_t>(sg_.off_vid[p]);
    r.aid = dp<int32_t>(sg_.off_aid[p]);
    r.tag = dp<float>(sg_.off_tag[p]);
    r.ts = dp<float>(sg_.off_ts[p]);
    r.play = dp<float>(sg_.off_play[p]);
    r.dur = dp<float>(sg_.off_dur[p]);
    r.labels = dp<uint32_t>(sg_.off_lab[p]);
    r.sid = cfg_.use_sid_history ? dp<int32_t>(sg_.off_sid[p]) : nullptr;
    return r;
  }
  FeatureTables tables() const {
    const orx_config& c = cfg_;
    FeatureTables t{};
    t.vid = t_vid_;
    t.aid = t_aid_;
    t.tag = t_tag_;
    t.ts = t_ts_;
    t.play = t_play_;
    t.dur = t_dur_;
    t.label = t_label_;
    if constexpr (kBf16) {
      t.vid16 = t_vid16_;
      t.aid16 = t_aid16_;
    }
    for (int l = 0; l < c.n_code_layers && l < 8; ++l) t.tokens[l] = tokens_[l];
    t.d = c.d_model;
    t.aid_dim = aid_dim(c);
    t.minor = minor_dim(c);
    t.vid_vocab = c.vid_vocab;
    t.aid_vocab = c.aid_vocab;
    t.n_flags = c.n_label_flags;
    t.n_code_layers = c.n_code_layers;
    t.use_sid = c.use_sid_history;
    t.vid_only = c.vid_only_features;
    return t;
  }

  // ------------------------------------------------------------------------
  // encode (policy.cpp:254-265)
  // ------------------------------------------------------------------------
  // MoE routing counters to zero at the start of a forward pass (each MoE
  // combine re-zeroes them for the next layer; this also recovers from an
  // interrupted pass)
  void zero_moe_counters() {
    if (counts_)
      CUDA_CHECK(cudaMemsetAsync(counts_, 0, (2 * static_cast<size_t>(cfg_.n_experts) + n_route_tickets_) * 4, st_));
  }
  void run_encode() {
    require(staged_, "no user batch staged");
    const orx_config& c = cfg_;
    if (enc_moe(c)) zero_moe_counters();
    const int d = c.d_model, U = sg_.U, Tn = enc_seq_len(c), Nq = c.n_queries, H = c.n_heads, dh = d / H;
    launch_z_init(U, Tn, d, pos_, pad_s_, pad_p_, dp<int32_t>(sg_.off_ns), dp<int32_t>(sg_.off_np), c.short_len,
                  c.positive_len, z_, st_);
    // static pathway (policy.cpp:218-223): [uid|gender|age] -> MLP -> row 0
    launch_static_features<T>(U, dp<int32_t>(sg_.off_uid), dp<int32_t>(sg_.off_gender), dp<int32_t>(sg_.off_age),
                              t_uid_, t_gender_, t_age_, static_dim(c), c.uid_vocab, c.gender_vocab, c.age_vocab,
                              feat_, Sp_, st_);
    mlp_into_z(p_static_, feat_, Sp_, U, dp<int32_t>(sg_.off_static_map));
    // short / positive pathways: MLP rows land left-padded inside z
    const FeatureTables tb = tables();
    for (int p = 0; p < 2; ++p) {
      if (!sg_.n_rec[p]) continue;
      if (fold_on_) {
        if constexpr (kBf16) launch_fold_features(recs(p), fold_[p], hid_, d, st_);
        fc2_into_z(p == 0 ? p_short_ : p_pos_, sg_.n_rec[p], dp<int32_t>(sg_.off_map[p]));
        continue;
      }
      launch_features<T>(recs(p), tb, feat_, Fp_, st_);
      mlp_into_z(p == 0 ? p_short_ : p_pos_, feat_, Fp_, sg_.n_rec[p], dp<int32_t>(sg_.off_map[p]));
    }
    // lifelong pathway -> keys (policy.cpp:233-238)
    if (sg_.n_rec[2]) {
      const Mlp& m = p_life_;
      if (fold_on_) {
        if constexpr (kBf16) launch_fold_features(recs(2), fold_[2], hid_, d, st_);
      } else {
        launch_features<T>(recs(2), tb, feat_, Fp_, st_);
        Epi e1 = epi(hid_, d, false);
        e1.act = ACT_LEAKY;
        gemm(feat_, Fp_, m.fc1, sg_.n_rec[2], e1);
      }
      if (kv_fold_) {  // K|V of every QFormer block straight from the hidden rows (build_kv_fold)
        const int nb = static_cast<int>(qblocks_.size());
        Epi ek = split_epi(vt_epi(vt_q_, Lpad_, 0, dp<int32_t>(sg_.off_key_user), dp<int32_t>(sg_.off_key_pos),
                                  static_cast<long long>(maxU_) * d * Lpad_),
                           kvl_, nb * d, nb * d);
        ek.row_map = dp<int32_t>(sg_.off_map[2]);
        gemm(hid_, d, kvf_, sg_.n_rec[2], ek);
      } else {
        Epi e2 = epi(keys_, d, false);
        e2.row_map = dp<int32_t>(sg_.off_map[2]);
        gemm(hid_, d, m.fc2, sg_.n_rec[2], e2);
      }
    }
    if (sg_.n_pad_keys) {
      if (kv_fold_) {
        const int nb = static_cast<int>(qblocks_.size());
        launch_fill_kv_pad<T>(sg_.n_pad_keys, dp<int32_t>(sg_.off_pad_keys), dp<int32_t>(sg_.off_key_user),
                              dp<int32_t>(sg_.off_key_pos), kv_pad_, nb * d, kvl_, nb * d, vt_q_, Lpad_,
                              static_cast<long long>(d) * Lpad_, static_cast<long long>(maxU_) * d * Lpad_, d, st_);
      } else {
        launch_fill_rows<T>(sg_.n_pad_keys, d, pad_l_, keys_, d, dp<int32_t>(sg_.off_pad_keys), st_);
      }
    }
    // QFormer blocks, no residual (nn.cpp:97-100)
    for (size_t b = 0; b < qblocks_.size(); ++b) {
      const QBlock& q = qblocks_[b];
      const bool first = b == 0, last = b + 1 == qblocks_.size();
      if (first) gemm(queries_, rup(d, 8), q.wq, Nq, epi(qproj_, d, false));  // user-independent
      else gemm(qcur_, d, q.wq, U * Nq, epi(qproj_, d, false));
      Seg qs;
      qs.stride = first ? 0 : Nq;
      qs.fixed_len = Nq;
      Seg ks;
      ks.start = dp<int32_t>(sg_.off_kstart);
      ks.len = dp<int32_t>(sg_.off_klen);
      Seg os;
      os.stride = Nq;
      os.fixed_len = Nq;
      const double aflops = 4.0 * Nq * sg_.n_keys * d;
      if (tc_attn_) {
        const int nb = static_cast<int>(qblocks_.size());
        const long long vt_layer = static_cast<long long>(maxU_) * d * Lpad_;
        if (first && !kv_fold_)  // K of every block | V^T of every block, keys_ read once
          gemm(keys_, d, qkv_all_, sg_.n_keys,
               split_epi(vt_epi(vt_q_, Lpad_, 0, dp<int32_t>(sg_.off_key_user), dp<int32_t>(sg_.off_key_pos), vt_layer),
                         kvl_, nb * d, nb * d));
        FmhaArgs f = fmha(U, Nq, qproj_, first ? Nq : U * Nq, d, kvl_, sg_.n_keys, nb * d, static_cast<int>(b) * d,
                          vt_q_ + b * vt_layer, U, Lpad_, nullptr, qs, ks, os, aflops);
        launch_fmha_tc(f, st_);
      } else {
        gemm(keys_, d, q.wkv, sg_.n_keys, epi(kvl_, 2 * d, false));
        launch_attention<T>(U, Nq, H, dh, qproj_, d, kvl_, 2 * d, kvl_ + d, 2 * d, att_, d, qs, ks, os, st_, aflops);
      }
      // folded norm (fc1 carries the gain) when the GEMMs run on the CTA-pair kernel
      const bool nfq = fold_norm_ && U * Nq > 128;
      Epi eo = epi(qo_, d, true);
      if (nfq) norm_out(eo);
      gemm(att_, d, q.wo, U * Nq, eo);
      if (!nfq) launch_rmsnorm<T>(U * Nq, d, qo_, d, fold_norm_ ? ones_ : q.gain, xn_, d, st_);
      Epi e1 = epi(ffh_, c.ffn_hidden, false);
      e1.act = ACT_SILU;
      if (nfq) norm_in(e1);
      gemm(xn_, d, q.fc1, U * Nq, e1);
      if (last) {
        Epi e2 = epi(z_, d, true);
        pos_resid(e2);
        e2.row_map = dp<int32_t>(sg_.off_life_map);
        gemm(ffh_, c.ffn_hidden, q.fc2, U * Nq, e2);
      } else {
        gemm(ffh_, c.ffn_hidden, q.fc2, U * Nq, epi(qcur_, d, false));
      }
    }
    // encoder blocks (policy.cpp:259-263)
    const int R = U * Tn;
    // folded RMSNorm (dense FFN encoder, bf16): each residual GEMM also writes
    // bf16(z) and its sums of squares; QKV / fc1 carry the gains and scale rows
    const bool nf = fold_norm_ && !enc_moe(c);
    for (size_t li = 0; li < enc_.size(); ++li) {
      const EncL& l = enc_[li];
      const bool nf_in = nf && li > 0;  // layer 0's input is assembled by many producers: explicit norm
      if (!nf_in) launch_rmsnorm<T>(R, d, z_, d, nf ? ones_ : l.n1, xn_, d, st_);
      Seg s;
      s.stride = Tn;
      s.fixed_len = Tn;
      if (tc_attn_) {
        Epi eq = split_epi(vt_epi(vt_enc_, Tpad_, Tn, nullptr, nullptr, 0), qkv_, 2 * d, 2 * d);
        if (nf_in) norm_in(eq);
        gemm(xn_, d, l.wqkv, R, eq);
        FmhaArgs f = fmha(U, Tn, qkv_, R, 2 * d, qkv_, R, 2 * d, d, vt_enc_, U, Tpad_, nullptr, s, s, s,
                          4.0 * U * Tn * Tn * d);
        launch_fmha_tc(f, st_);
      } else {
        Epi eq = epi(qkv_, 3 * d, false);
        if (nf_in) norm_in(eq);
        gemm(xn_, d, l.wqkv, R, eq);
        launch_attention<T>(U, Tn, H, dh, qkv_, 3 * d, qkv_ + d, 3 * d, qkv_ + 2 * d, 3 * d, att_, d, s, s, s, st_,
                            4.0 * U * Tn * Tn * d);
      }
      Epi eo = epi(z_, d, true);
      eo.resid = z_;
      eo.ld_resid = d;
      if (nf) norm_out(eo);
      gemm(att_, d, l.wo, R, eo);
      if (!nf) launch_rmsnorm<T>(R, d, z_, d, enc_moe(c) && fold_norm_ ? ones_ : l.n2, xn_, d, st_);
      if (enc_moe(c)) {
        // the last layer's combine also writes bf16(z): the decoder's cross K|V GEMM operand
        if (kBf16 && li + 1 == enc_.size()) zt_fresh_ = moe(l.moe, xn_, R, z_, l.n2, zt_, nullptr);
        else moe(l.moe, xn_, R, z_, l.n2);
      } else {
        const bool last = li + 1 == enc_.size();
        // the last fc2 also writes bf16(z) for the decoder's cross K|V GEMM (XSSQ epilogue,
        // sums of squares unused) instead of a separate conversion pass
        ffn(l.fc1, l.fc2, xn_, R, z_, nf, nf && !last, nf && last ? zt_ : nullptr);
        zt_fresh_ = nf && last;
      }
    }
  }

  // The pathway outputs land in z on top of the position embedding: the
  // residual operand is the [Tn][d] position table, indexed by z row % Tn (it
  // stays in L2), so z itself is initialised only at left-padding rows
  // (launch_z_init) instead of being written once and read back.
  void pos_resid(Epi& e) {
    e.resid = pos_;
    e.ld_resid = cfg_.d_model;
    e.resid_mod = enc_seq_len(cfg_);
  }
  void fc2_into_z(const Mlp& m, int rows, const int32_t* map) {
    const int d = cfg_.d_model;
    Epi e2 = epi(z_, d, true);
    pos_resid(e2);
    e2.row_map = map;
    gemm(hid_, d, m.fc2, rows, e2);
  }
  void mlp_into_z(const Mlp& m, const T* x, int ldx, int rows, const int32_t* map) {
    const int d = cfg_.d_model;
    Epi e1 = epi(hid_, d, false);
    e1.act = ACT_LEAKY;
    gemm(x, ldx, m.fc1, rows, e1);
    Epi e2 = epi(z_, d, true);
    pos_resid(e2);
    e2.row_map = map;
    gemm(hid_, d, m.fc2, rows, e2);
  }
  // h += fc2(silu(fc1(x)))  (ffn, nn.cpp:71-73)
  // fold_in: x is the un-normalised bf16 row (fc1 carries the RMSNorm gain;
  // scales from ssq_); fold_out: fc2 also writes bf16(h) to xn_ and its sums
  // of squares to ssq_ for the next folded RMSNorm.
  void ffn(const Lin<T>& fc1, const Lin<T>& fc2, const T* x, int rows, float* h, bool fold_in = false,
           bool fold_out = false, T* copy_out = nullptr) {
    const int d = cfg_.d_model;
    Epi e1 = epi(ffh_, cfg_.ffn_hidden, false);
    e1.act = ACT_SILU;
    if (fold_in) norm_in(e1);
    gemm(x, d, fc1, rows, e1);
    Epi e2 = epi(h, d, true);
    e2.resid = h;
    e2.ld_resid = d;
    if (fold_out) norm_out(e2);
    if (copy_out) {  // bf16 copy of the updated rows (the folded-norm epilogue; its sums of squares unused)
      norm_out(e2);
      e2.out2 = copy_out;
    }
    gemm(ffh_, cfg_.ffn_hidden, fc2, rows, e2);
  }
  // RMSNorm folded into the GEMMs around it (Epi::out2 / ssq / rsq, fold_norm_)
  void norm_out(Epi& e) {
    e.out2 = xn_;
    e.ldo2 = cfg_.d_model;
    e.ssq = ssq_;
    e.ssq_ld = ssq_ld_;
  }
  void norm_in(Epi& e) {
    e.rsq = ssq_;
    e.rsq_ld = ssq_ld_;
    e.rsq_n = 2 * cfg_.d_model / 256;
    e.rsq_inv_d = 1.f / cfg_.d_model;
  }
  // h += MoE(x)  (moe_forward, nn.cpp:117-172)
  // post: when non-null the bf16 engine also writes the NEXT op's input from the
  // updated h in the combine pass: RMSNorm(h) with gain `post_gain` into `post`,
  // or a plain bf16 copy when post_gain is null. Returns whether it did.
  bool moe(const MoeW& m, const T* x, int rows, float* h, const float* norm_gain, T* post = nullptr,
           const float* post_gain = nullptr, bool x_unnormed = false) {
    const orx_config& c = cfg_;
    const int d = c.d_model, E = c.n_experts, k = c.experts_active;
    // counts_ (histogram | scatter fill) is zero here: zeroed once per forward pass
    // (zero_moe_counters) and by every MoE combine for the next layer
    // tensor-pipe router for large row counts (one 128-row tile per SM is latency-bound: the SIMT
    // router is faster below a few thousand rows)
    if (m.gate_hi && rows >= 4096)
      launch_moe_route_tc(rows, d, E, k, h, d, m.gate_hi, m.gate_lo, m.bias, sel_, wts_, counts_, route_part_,
                          route_ticket_, st_);
    else
      launch_moe_route(rows, d, E, k, h, d, norm_gain, m.gate_t, m.gate_gain, m.bias, sel_, wts_, counts_, st_,
                       m.gate_sw);
    if (route_stats_) record_routing(rows);
    if (ep_world_ > 1) return moe_ep(m, x, rows, h, post, post_gain);
    MoePlan plan;
    plan.counts = counts_;
    plan.fill = counts_ + E;
    plan.tile_expert = tile_expert_;
    plan.n_mtiles = n_mtiles_;
    plan.max_tiles = max_tiles_;
    plan.tile_rows = kMoeTile;
    plan.E = E;
    if (x_unnormed) {  // x = bf16(h) with ssq_ partials (norm_out): per-grouped-row scales for W1|W3
      plan.ssq = ssq_;
      plan.ssq_ld = ssq_ld_;
      plan.ssq_n = 2 * d / 256;
      plan.inv_d = 1.f / d;
      plan.row_rsq = row_rsq_;
    }
    launch_moe_scatter<T>(rows, k, d, x, d, sel_, wts_, plan, slot_, xg_, row_scale_, st_);
    expert_ffn(m, static_cast<int>(S_), static_cast<long long>(rows) * k, false, x_unnormed ? row_rsq_ : nullptr);
    if constexpr (kBf16) {
      if (post && launch_moe_combine_norm(rows, k, d, yg_, slot_, h, d, post_gain, post, d, st_, counts_, 2 * E))
        return true;
    }
    launch_moe_combine(rows, k, d, yg_, slot_, h, d, st_, counts_, 2 * E);
    return false;
  }

  // ORX_ROUTE_STATS (diagnostic, graphs off): per-expert token counts of every
  // MoE call with >= 4096 rows, summarised at engine teardown as the rank-load
  // imbalance an expert-parallel split of the experts would see.
  void record_routing(int rows) {
    if (rows < 4096) return;
    std::vector<int32_t> h(cfg_.n_experts);
    CUDA_CHECK(cudaMemcpyAsync(h.data(), counts_, h.size() * 4, cudaMemcpyDeviceToHost, st_));
    CUDA_CHECK(cudaStreamSynchronize(st_));
    route_hist_.push_back(std::move(h));
  }
  void report_routing() const {
    if (route_hist_.empty()) return;
    const int E = cfg_.n_experts;
    std::vector<double> share(E, 0.0);
    double imb[4] = {0, 0, 0, 0};
    for (const auto& h : route_hist_) {
      double tot = 0;
      for (int e = 0; e < E; ++e) tot += h[e];
      for (int e = 0; e < E; ++e) share[e] += h[e] / tot / route_hist_.size();
      for (int wi = 0; wi < 4; ++wi) {
        const int W = 1 << wi;
        if (E % W) continue;
        double mx = 0;
        for (int r = 0; r < W; ++r) {
          double s = 0;
          for (int e = r * E / W; e < (r + 1) * E / W; ++e) s += h[e];
          mx = std::max(mx, s);
        }
        imb[wi] += mx / (tot / W) / route_hist_.size();
      }
    }
    fprintf(stderr, "[orx route] calls %zu; max/mean rank load at EP2 %.3f EP4 %.3f EP8 %.3f; expert shares:",
            route_hist_.size(), imb[1], imb[2], imb[3]);
    for (int e = 0; e < E; ++e) fprintf(stderr, " %.3f", share[e]);
    fprintf(stderr, "\n");
  }

  // Grouped expert FFNs over xg_ (expert per M tile: tile_expert_ / n_mtiles_):
  // yg_ = row_scale * W2(silu(W1 x) * W3 x)  (swiglu, nn.cpp:75-86; weight nn.cpp:167-168)
  // peer: expert-parallel (bf16) -- the W2 epilogue stores every output row
  // straight into its token rank's return buffer (ep_.src codes, ep_.yr views).
  void expert_ffn(const MoeW& m, int M, long long algo_rows, bool peer = false, const float* row_rsq = nullptr) {
    const orx_config& c = cfg_;
    const int d = c.d_model, he = expert_hidden(c), hp = rup(he, 8);
    Grouped g;
    g.tile_expert = tile_expert_;
    g.n_mtiles = n_mtiles_;
    g.n_groups = El_;
    g.tile_rows = kMoeTile;
    g.algo_rows = algo_rows;
    if constexpr (kBf16) {
      Epi e1 = epi(hg_, hp, false);
      e1.swiglu = 1;
      e1.row_rsq = row_rsq;
      e1.n_out = he;
      e1.m_valid = M;
      g.b_rows_per_expert = 2 * he;
      gemm_bf16(xg_, d, m.w13, rup(d, 8), M, 2 * he, rup(d, 8), e1, &g, st_);
      Epi e2 = epi(yg_, d, false);
      e2.row_scale = row_scale_;
      e2.n_out = d;
      e2.m_valid = M;
      if (peer) {
        e2.peer_code = ep_.src[ep_rank_];
        for (int p = 0; p < ep_world_; ++p) e2.peer_out[p] = ep_.yr[p];
      }
      g.b_rows_per_expert = d;
      gemm_bf16(hg_, hp, m.w2, hp, M, d, hp, e2, &g, st_);
    } else {
      g.b_rows_per_expert = he;
      Epi ea = epi(ga_, he, true);
      ea.n_out = he;
      ea.m_valid = M;
      gemm_f32(reinterpret_cast<const float*>(xg_), d, static_cast<const float*>(m.w13), rup(d, 8), M, he, rup(d, 8),
               ea, &g, st_);
      Epi eb = ea;
      eb.out = gb_;
      gemm_f32(reinterpret_cast<const float*>(xg_), d, static_cast<const float*>(m.w3), rup(d, 8), M, he, rup(d, 8),
               eb, &g, st_);
      launch_swiglu_mul(static_cast<long long>(M) * he, ga_, gb_, reinterpret_cast<float*>(hg_), st_);
      Epi e2 = epi(yg_, d, true);
      e2.row_scale = row_scale_;
      e2.n_out = d;
      e2.m_valid = M;
      g.b_rows_per_expert = d;
      gemm_f32(reinterpret_cast<const float*>(hg_), he, static_cast<const float*>(m.w2), hp, M, d, he, e2, &g, st_);
    }
  }

  // Symmetric exchange region of an expert-parallel engine: one cudaMalloc per
  // rank, same layout on every rank, mapped into every peer by CUDA IPC (the
  // handles travel once, at engine creation, over the NCCL communicator).
  void setup_ep_exchange(int64_t send_cap, int64_t recv_cap) {
    const int d = cfg_.d_model, E = cfg_.n_experts, W = ep_world_;
    require(W <= kEpMaxWorld, "expert parallelism supports at most 8 ranks");
    require(send_cap < (1 << 24) && recv_cap < (int64_t(1) << 31), "expert-parallel exchange too large");
    size_t off = 0;
    auto take = [&](size_t bytes) {
      const size_t o = off;
      off += (bytes + 255) / 256 * 256;
      return o;
    };
    const size_t o_xr = take(static_cast<size_t>(recv_cap) * d * sizeof(T));
    const size_t o_wr = take(static_cast<size_t>(recv_cap) * 4);
    const size_t o_src = take(static_cast<size_t>(recv_cap) * 4);
    const size_t o_yr = take(static_cast<size_t>(send_cap) * d * sizeof(T));
    const size_t o_cnt = take(static_cast<size_t>(W) * E * 4);
    const size_t o_flag = take(static_cast<size_t>(3) * W * 4);
    CUDA_CHECK(cudaMalloc(&ep_region_, off));
    CUDA_CHECK(cudaMemset(ep_region_, 0, off));
    struct Hello {  // what every rank publishes once: its region and its expert placement
      cudaIpcMemHandle_t h;
      uint64_t placement;
    } mine{};
    CUDA_CHECK(cudaIpcGetMemHandle(&mine.h, ep_region_));
    mine.placement = 1469598103934665603ull;  // FNV-1a over the owner table
    for (int32_t o : place_.owner) mine.placement = (mine.placement ^ static_cast<uint32_t>(o)) * 1099511628211ull;
    // all-gather (NCCL moves device memory)
    uint8_t* dh = nullptr;
    CUDA_CHECK(cudaMalloc(&dh, static_cast<size_t>(W) * sizeof(mine)));
    CUDA_CHECK(cudaMemcpy(dh + static_cast<size_t>(ep_rank_) * sizeof(mine), &mine, sizeof(mine),
                          cudaMemcpyHostToDevice));
    NCCL_CHECK(nccl().AllGather(dh + static_cast<size_t>(ep_rank_) * sizeof(mine), dh, sizeof(mine), ncclUint8,
                                comm_, st_));
    std::vector<Hello> all(static_cast<size_t>(W));
    CUDA_CHECK(cudaStreamSynchronize(st_));
    CUDA_CHECK(cudaMemcpy(all.data(), dh, static_cast<size_t>(W) * sizeof(mine), cudaMemcpyDeviceToHost));
    CUDA_CHECK(cudaFree(dh));
    for (int p = 0; p < W; ++p)
      require(all[p].placement == mine.placement, "expert-parallel ranks were created with different expert placements");
    ep_peer_base_.assign(static_cast<size_t>(W), nullptr);
    for (int p = 0; p < W; ++p) {
      if (p == ep_rank_) {
        ep_peer_base_[p] = ep_region_;
      } else {
        CUDA_CHECK(cudaIpcOpenMemHandle(&ep_peer_base_[p], all[p].h, cudaIpcMemLazyEnablePeerAccess));
      }
      uint8_t* b = static_cast<uint8_t*>(ep_peer_base_[p]);
      ep_.xr[p] = b + o_xr;
      ep_.wr[p] = reinterpret_cast<float*>(b + o_wr);
      ep_.src[p] = reinterpret_cast<int32_t*>(b + o_src);
      ep_.yr[p] = b + o_yr;
      ep_.cnt[p] = reinterpret_cast<int32_t*>(b + o_cnt);
      ep_.flag[p] = reinterpret_cast<uint32_t*>(b + o_flag);
    }
    ep_.me = ep_rank_;
    ep_.world = W;
    ep_.recv_cap = static_cast<int>(recv_cap);
    ep_.epoch = ar_.alloc<uint32_t>(4);
    ep_.err = ar_.alloc<int32_t>(1);
    CUDA_CHECK(cudaMemset(ep_.epoch, 0, 16));
    CUDA_CHECK(cudaMemset(ep_.err, 0, 4));
    ep_seg_ = ar_.alloc<int32_t>(2 * El_);
    ep_tiles_ = ar_.alloc<int32_t>(max_tiles_);
    ep_ntiles_ = ar_.alloc<int32_t>(1);
    CUDA_CHECK(cudaDeviceSynchronize());
  }

  // Expert-parallel MoE: every rank routes its own tokens
  // and writes each (token, expert) row with its gate weight straight into the
  // expert owner's grouped GEMM buffer over NVLink (peer stores at offsets the
  // device plans from the all-gathered histograms); each rank runs the grouped
  // GEMMs of its local experts on what arrived and writes every weighted
  // output back into the token rank's return buffer; the combine (ascending
  // expert id) runs where the token lives. Arrival counters order the phases,
  // so the whole exchange is device-side and replays from a CUDA graph. Every
  // row goes through the same kernels as on one GPU: bitwise identical to the
  // replica engine. All ranks must run the same sequence of engine calls.
  bool moe_ep(const MoeW& m, const T* x, int rows, float* h, T* post, const float* post_gain) {
    const orx_config& c = cfg_;
    const int d = c.d_model, E = c.n_experts, k = c.experts_active;
    launch_ep_counts(E, counts_, ep_, st_);
    launch_ep_wait(ep_, EP_COUNTS, st_);
    launch_ep_plan(E, ep_, kMoeTile, max_tiles_, cursor_, ep_tiles_, ep_ntiles_, ep_seg_, m.ep_owner, m.ep_slot,
                   m.ep_list, El_, m.ep_load, st_);
    launch_ep_dispatch<T>(rows, k, d, x, d, sel_, wts_, cursor_, slot_, m.ep_owner, ep_, st_);
    launch_ep_signal(ep_, EP_DISPATCH, st_);
    launch_ep_wait(ep_, EP_DISPATCH, st_);
    // grouped GEMMs of the local experts over the received rows (in place)
    T* saved_xg = xg_;
    float* saved_rs = row_scale_;
    int32_t* saved_te = tile_expert_;
    int32_t* saved_nm = n_mtiles_;
    xg_ = static_cast<T*>(ep_.xr[ep_rank_]);
    row_scale_ = ep_.wr[ep_rank_];
    tile_expert_ = ep_tiles_;
    n_mtiles_ = ep_ntiles_;
    // bf16: the W2 epilogue stores each output row into its token rank's return buffer
    const bool fused_return = kBf16 && d % 128 == 0;
    expert_ffn(m, static_cast<int>(S_), static_cast<long long>(rows) * k, fused_return);  // FLOPs: average share
    xg_ = saved_xg;
    row_scale_ = saved_rs;
    tile_expert_ = saved_te;
    n_mtiles_ = saved_nm;
    if (!fused_return) launch_ep_return(El_, d, ep_seg_, yg_, ep_, st_);
    launch_ep_signal(ep_, EP_RETURN, st_);
    launch_ep_wait(ep_, EP_RETURN, st_);
    const T* yr = static_cast<const T*>(ep_.yr[ep_rank_]);
    if constexpr (kBf16) {
      if (post && launch_moe_combine_norm(rows, k, d, yr, slot_, h, d, post_gain, post, d, st_, counts_, 2 * E))
        return true;
    }
    launch_moe_combine(rows, k, d, yr, slot_, h, d, st_, counts_, 2 * E);
    return false;
  }

  // Expert-parallel exchange failures (peer timeout, capacity) surface here.
  void check_ep() {
    if (ep_world_ <= 1) return;
    int32_t e = 0;
    CUDA_CHECK(cudaMemcpyAsync(&e, ep_.err, 4, cudaMemcpyDeviceToHost, st_));
    CUDA_CHECK(cudaStreamSynchronize(st_));
    if (e == 1) throw RuntimeError("expert-parallel exchange: a peer did not arrive within 30 s");
    if (e == 2) throw RuntimeError("expert-parallel exchange: receive buffer overflow");
  }

  void prepare_decoder(int U) {
    const int d = cfg_.d_model, Tn = enc_seq_len(cfg_);
    if constexpr (kBf16)
      if (!zt_fresh_) launch_convert<T>(U * Tn, d, z_, d, zt_, d, st_);  // else the encoder's last GEMM wrote it
    if (tc_attn_) {  // cross K of every decoder layer [rows][Ld*d]; cross V transposed per layer
      const int kn = xkv_w_.N / 2;  // K of all layers | V of all layers
      gemm(zt_, d, xkv_w_, U * Tn,
           split_epi(vt_epi(vt_x_, Tpad_, Tn, nullptr, nullptr, static_cast<long long>(maxU_) * d * Tpad_), xkv_, kn,
                     kn));
    } else {
      gemm(zt_, d, xkv_w_, U * Tn, epi(xkv_, xkv_w_.N, false));
    }
  }

  // One decoder position for `rows` rows (policy.cpp:267-295). Rows of a
  // group (user) are contiguous: group g = rows [gq.start(g), +gq.len(g)),
  // cross-attending to encoder rows [gk.start(g), +Tn).
  // vt_user: encoder user of each group (NULL: group g is user g).
  void decode_step(int step, int rows, int groups, Seg gq, Seg gk, const int32_t* codes, int code_stride,
                   const int32_t* anc, int anc_stride, int max_group_rows, const int32_t* vt_user = nullptr,
                   float2* head_stats = nullptr) {
    const orx_config& c = cfg_;
    const int d = c.d_model, H = c.n_heads, dh = d / H, Ld = dec_layers(c), Tn = enc_seq_len(c);
    if (c.moe_enabled) zero_moe_counters();
    const float* emb = step == 0 ? bos_ : tokens_[step - 1];
    const int32_t* emb_code = step == 0 ? nullptr : codes + (step - 1);
    bool have_x = false;  // xn_ already holds the next op's input (fused into the MoE combine / embedding)
    if constexpr (kBf16)
      have_x = launch_dec_embed_norm(rows, d, emb, emb_code, code_stride, h_, dec_[0].n1, xn_, st_);
    if (!have_x) launch_dec_embed(rows, d, emb, emb_code, code_stride, h_, st_);
    for (int l = 0; l < Ld; ++l) {
      const DecL& w = dec_[l];
      if (!have_x) launch_rmsnorm<T>(rows, d, h_, d, w.n1, xn_, d, st_);
      have_x = false;
      T* qkv_now = kvpos_[static_cast<size_t>(step) * Ld + l];  // this position's QKV = its K/V cache entry
      gemm(xn_, d, w.sqkv, rows, epi(qkv_now, 3 * d, false));
      launch_dec_self_attn<T>(rows, d, H, step, l, Ld, qkv_now, kvpos_ptrs_, anc, anc_stride, att_, st_);
      Epi e = epi(h_, d, true);
      e.resid = h_;
      e.ld_resid = d;
      // folded n2 (cq carries its gain): beyond 128 rows the so GEMM writes bf16(h) and its sums of
      // squares and cq scales rows; at step 0 (1-CTA GEMMs) an explicit gain-free RMSNorm
      const bool nf2 = fold_norm_ && rows > 128;
      Epi es = e;
      if (nf2) norm_out(es);
      gemm(att_, d, w.so, rows, es);
      if (!nf2) launch_rmsnorm<T>(rows, d, h_, d, fold_norm_ ? ones_ : w.n2, xn_, d, st_);
      Epi ecq = epi(qkv_, d, false);
      if (nf2) norm_in(ecq);
      gemm(xn_, d, w.cq, rows, ecq);
      if (tc_attn_) {  // beam rows of a user over its cached encoder K / V^T (computed once, prepare_decoder)
        FmhaArgs f = fmha(groups, max_group_rows, qkv_, rows, d, xkv_, static_cast<long long>(maxU_) * Tn, Ld * d,
                          l * d, vt_x_ + static_cast<size_t>(l) * maxU_ * d * Tpad_, maxU_, Tpad_, vt_user, gq, gk,
                          gq, 4.0 * rows * Tn * d);
        f.prof_cat = PROF_XATTN;  // one pass over every user's cached K and V^T, plus the beam rows' Q and O
        f.bytes = static_cast<double>(groups) * Tn * d * 2.0 * sizeof(T) + 2.0 * rows * d * sizeof(T);
        launch_fmha_tc(f, st_);
      } else {
        const int ldkv = 2 * d * Ld;
        launch_attention<T>(groups, max_group_rows, H, dh, qkv_, d, xkv_ + (size_t)l * 2 * d, ldkv,
                            xkv_ + (size_t)l * 2 * d + d, ldkv, att_, d, gq, gk, gq, st_, 4.0 * rows * Tn * d);
      }
      // folded n3 (FFN fc1 / MoE W1|W3 carry its gain): co writes bf16(h) and its sums of
      // squares; fc1 scales rows, the MoE scatter hands each grouped row its scale to the
      // SwiGLU epilogue (expert-parallel: an explicit gain-free norm before the dispatch)
      static const bool no_n3 = getenv("ORX_NO_N3_FOLD") != nullptr;  // A/B
      const bool nf3 = fold_norm_ && rows > 128 && (!c.moe_enabled || ep_world_ == 1) && !no_n3;
      Epi e3 = e;
      if (nf3) norm_out(e3);
      gemm(att_, d, w.co, rows, e3);
      if (!nf3) launch_rmsnorm<T>(rows, d, h_, d, fold_norm_ ? ones_ : w.n3, xn_, d, st_);
      if (c.moe_enabled)  // next layer's n1 norm (or the head's bf16 copy) fused into the combine
        have_x = moe(w.moe, xn_, rows, h_, w.n3, xn_, l + 1 < Ld ? dec_[l + 1].n1 : nullptr, nf3);
      else
        ffn(w.fc1, w.fc2, xn_, rows, h_, nf3);
    }
    (void)Tn;
    // position_logits: no final norm (policy.cpp:290-295)
    if (!have_x) launch_convert<T>(rows, d, h_, d, xn_, d, st_);
    Epi he = epi(logits_, c.codebook_size, true);
    if (head_stats) {  // + per-chunk log-sum-exp statistics for launch_beam_select
      he.stats = head_stats;
      he.stats_ld = Rd_;
    }
    gemm(xn_, d, heads_[step], rows, he);
  }

  // ------------------------------------------------------------------------
  // public flows
  // ------------------------------------------------------------------------
  void encode(float* z_out) override {
    CUDA_CHECK(cudaSetDevice(dev_));
    run_encode();
    if (z_out) {
      size_t n = static_cast<size_t>(sg_.U) * enc_seq_len(cfg_) * cfg_.d_model;
      CUDA_CHECK(cudaMemcpyAsync(z_out, z_, n * 4, cudaMemcpyDeviceToHost, st_));
      d2h_bytes += static_cast<int64_t>(n * 4);
    }
    CUDA_CHECK(cudaStreamSynchronize(st_));
    CUDA_CHECK(cudaGetLastError());
    check_ep();
    if (z_out) require_finite(z_out, static_cast<size_t>(sg_.U) * enc_seq_len(cfg_) * cfg_.d_model);
  }

  void beam_search(int width, orx_beam_out* out) override { run_beam(width, out, false); }
  void beam_search_constrained(int width, orx_beam_out* out) override {
    require(has_trie_, "constrained beam search over an empty trie");  // generation.cpp:44-45
    run_beam(width, out, true);
  }

  void set_trie(int n_nodes, const int32_t* child_off, int64_t n_edges, const int32_t* child_code,
                const int32_t* child_node) override {
    CUDA_CHECK(cudaSetDevice(dev_));
    require(n_nodes >= 1 && n_edges >= 0 && child_off && (n_edges == 0 || (child_code && child_node)),
            "trie: bad CSR arrays");
    require(child_off[0] == 0 && child_off[n_nodes] == n_edges, "trie: child offsets must span the edges");
    for (int64_t i = 0; i < n_edges; ++i) {
      require(child_code[i] >= 0 && child_code[i] < cfg_.codebook_size, "trie: code outside the codebook");
      require(child_node[i] > 0 && child_node[i] < n_nodes, "trie: child node out of range");
    }
    for (int n = 0; n < n_nodes; ++n)
      for (int32_t i = child_off[n] + 1; i < child_off[n + 1]; ++i)
        require(child_code[i - 1] < child_code[i], "trie: children must have ascending, distinct codes");
    CUDA_CHECK(cudaStreamSynchronize(st_));
    trie_ar_.reset();
    int32_t* off = trie_ar_.alloc<int32_t>(n_nodes + 1);
    int32_t* code = trie_ar_.alloc<int32_t>(std::max<int64_t>(n_edges, 1));
    int32_t* nd = trie_ar_.alloc<int32_t>(std::max<int64_t>(n_edges, 1));
    CUDA_CHECK(cudaMemcpy(off, child_off, (n_nodes + 1) * 4, cudaMemcpyHostToDevice));
    if (n_edges) {
      CUDA_CHECK(cudaMemcpy(code, child_code, n_edges * 4, cudaMemcpyHostToDevice));
      CUDA_CHECK(cudaMemcpy(nd, child_node, n_edges * 4, cudaMemcpyHostToDevice));
    }
    trie_.child_off = off;
    trie_.child_code = code;
    trie_.child_node = nd;
    has_trie_ = n_edges > 0;
    // captured constrained searches hold the old trie's device pointers in
    // their kernel parameters: drop them
    for (size_t i = graphs_.size(); i-- > 0;)
      if (graphs_[i].key.constrained) {
        cudaGraphExecDestroy(graphs_[i].exec);
        graphs_.erase(graphs_.begin() + static_cast<std::ptrdiff_t>(i));
      }
  }

  struct GraphKey {
    int U, W;
    bool constrained;
    int n_rec[3];
    int n_keys, n_pad;
    const void* stage;
    bool operator==(const GraphKey& o) const {
      return U == o.U && W == o.W && constrained == o.constrained && n_rec[0] == o.n_rec[0] &&
             n_rec[1] == o.n_rec[1] && n_rec[2] == o.n_rec[2] && n_keys == o.n_keys && n_pad == o.n_pad &&
             stage == o.stage;
    }
  };

  // encode + decode + prune for the staged batch (only stream work: capturable)
  void beam_body(int width, bool constrained) {
    const orx_config& c = cfg_;
    const int U = sg_.U, V = c.codebook_size, L = c.n_code_layers, Tn = enc_seq_len(c);
    run_encode();
    prepare_decoder(U);
    int cur = 0;
    bs_[0].node = constrained ? node_[0] : nullptr;
    bs_[1].node = constrained ? node_[1] : nullptr;
    launch_beam_init(U, bs_[cur], st_);
    int n_live = 1;
    for (int step = 0; step < L; ++step) {
      const int rows = U * n_live;
      Seg gq;
      gq.stride = n_live;
      gq.fixed_len = n_live;
      Seg gk;
      gk.stride = Tn;
      gk.fixed_len = Tn;
      const int n_new = static_cast<int>(std::min<int64_t>(width, static_cast<int64_t>(n_live) * V));
      // fused selection: unconstrained (the head GEMM then runs on the CTA-pair kernel, any M)
      static const bool step0_topk = getenv("ORX_STEP0_TOPK") != nullptr;  // A/B: materialised path at M <= 128
      const bool fused = fused_select_ && !constrained && (rows > 128 || !step0_topk);
      decode_step(step, rows, U, gq, gk, bs_[cur].codes, L, bs_[cur].anc, L, n_live, nullptr,
                  fused ? head_stats_ : nullptr);
      if (fused) {
        launch_beam_select(U, n_live, n_new, V, L, step, logits_, head_stats_, Rd_, lse_, sel_scratch_, bs_[cur],
                           bs_[cur ^ 1], st_);
        cur ^= 1;
        n_live = n_new;
        continue;
      }
      const int ksel = std::min(width, V);
      if (constrained)
        launch_row_topk_trie(rows, V, ksel, logits_, bs_[cur].score, bs_[cur].lexrank, bs_[cur].node, trie_, lse_,
                             cand_, st_);
      else
        launch_row_topk(rows, V, ksel, logits_, bs_[cur].score, bs_[cur].lexrank, lse_, cand_, topk_fail_, st_);
      launch_beam_merge(U, n_live, ksel, n_new, V, L, step, cand_, logits_, lse_, bs_[cur], bs_[cur ^ 1], st_,
                        constrained ? &trie_ : nullptr);
      cur ^= 1;
      n_live = n_new;
    }
  }

  // Launch the staged request's beam search (CUDA graph replay when shapes
  // repeat) and enqueue the D2H of its result into the slot's pinned bounce
  // buffer; the result is read by collect().
  void launch_beam(int width, bool constrained, bool want_out) {
    CUDA_CHECK(cudaSetDevice(dev_));
    const orx_config& c = cfg_;
    require(width >= 1, "generation width must be >= 1");  // validate_request, generation.cpp:35
    require(width <= maxW_, "beam width above the engine capacity");
    require(staged_, "no user batch staged");
    const int U = sg_.U, V = c.codebook_size, L = c.n_code_layers;
    // The whole encode + decode + prune sequence is replayed from a CUDA graph
    // when the request has the same shapes as a captured one (no host work
    // or launch gaps between its ~250 kernels; the expert-parallel exchange is
    // device-side too); profiling runs launch directly.
    const bool graphs = !prof_enabled() && !getenv("ORX_NO_GRAPH") && !route_stats_;
    int n_live = 1;
    for (int step = 0; step < L; ++step) n_live = static_cast<int>(std::min<int64_t>(width, (int64_t)n_live * V));
    int cur = L % 2;
    if (graphs) {
      const GraphKey key{U, width, constrained, {sg_.n_rec[0], sg_.n_rec[1], sg_.n_rec[2]}, sg_.n_keys,
                         sg_.n_pad_keys, dev_stage_[stage_slot_]};
      CachedGraph* hit = nullptr;
      for (auto& g : graphs_)
        if (g.key == key) hit = &g;
      if (!hit) {
        if (graphs_.size() >= 4) {  // small LRU: one graph per staging slot and shape
          cudaGraphExecDestroy(graphs_.front().exec);
          graphs_.erase(graphs_.begin());
        }
        cudaGraph_t g = nullptr;
        CUDA_CHECK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
        try {
          beam_body(width, constrained);
        } catch (...) {
          cudaStreamEndCapture(st_, &g);
          if (g) cudaGraphDestroy(g);
          throw;
        }
        CUDA_CHECK(cudaStreamEndCapture(st_, &g));
        // the replay launches these kernel nodes every call: count them like
        // direct launches (memset nodes are not kernels)
        size_t n_nodes = 0;
        CUDA_CHECK(cudaGraphGetNodes(g, nullptr, &n_nodes));
        std::vector<cudaGraphNode_t> nodes(n_nodes);
        if (n_nodes) CUDA_CHECK(cudaGraphGetNodes(g, nodes.data(), &n_nodes));
        long long kernels = 0;
        for (cudaGraphNode_t nd : nodes) {
          cudaGraphNodeType t;
          CUDA_CHECK(cudaGraphNodeGetType(nd, &t));
          if (t == cudaGraphNodeTypeKernel) ++kernels;
        }
        CachedGraph cg;
        cg.key = key;
        cg.kernels = kernels;
        CUDA_CHECK(cudaGraphInstantiate(&cg.exec, g, 0));
        cudaGraphDestroy(g);
        graphs_.push_back(cg);
        hit = &graphs_.back();
        launch_counter() -= kernels;  // capture itself launched nothing
      } else if (hit != &graphs_.back()) {  // keep LRU order
        CachedGraph keep = *hit;
        graphs_.erase(graphs_.begin() + (hit - graphs_.data()));
        graphs_.push_back(keep);
        hit = &graphs_.back();
      }
      CUDA_CHECK(cudaGraphLaunch(hit->exec, st_));
      launch_counter() += hit->kernels;
    } else {
      beam_body(width, constrained);
    }
    CUDA_CHECK(cudaEventRecord(dev_free_[stage_slot_], st_));  // the staged inputs of this slot are consumed
    last_n_live_ = n_live;
    last_state_ = cur;
    Pending pd;
    pd.slot = stage_slot_;
    pd.U = U;
    pd.n_live = n_live;
    pd.width = width;
    pd.has_out = want_out;
    if (want_out) {
      const size_t nc = static_cast<size_t>(U) * n_live * L, nl = static_cast<size_t>(U) * n_live;
      const size_t need = nc * 4 + nl * 8 + 4;  // codes, log-probs, non-finite flag
      const int k = stage_slot_;
      if (need > host_out_cap_[k]) {
        CUDA_CHECK(cudaEventSynchronize(out_ready_[k]));
        if (host_out_[k]) cudaFreeHost(host_out_[k]);
        CUDA_CHECK(cudaMallocHost(&host_out_[k], need));
        host_out_cap_[k] = need;
      }
      uint8_t* ho = static_cast<uint8_t*>(host_out_[k]);
      CUDA_CHECK(cudaMemcpyAsync(ho, bs_[cur].codes, nc * 4, cudaMemcpyDeviceToHost, st_));
      CUDA_CHECK(cudaMemcpyAsync(ho + nc * 4, bs_[cur].score64, nl * 8, cudaMemcpyDeviceToHost, st_));
      CUDA_CHECK(cudaMemcpyAsync(ho + nc * 4 + nl * 8, nonfinite_, 4, cudaMemcpyDeviceToHost, st_));
      CUDA_CHECK(cudaEventRecord(out_ready_[k], st_));
      d2h_bytes += static_cast<int64_t>(need);
    }
    pending_.push_back(pd);
  }

  // Wait for the oldest launched request and scatter its beams (rows of width) into `out`.
  void collect_beam(orx_beam_out* out) {
    require(!pending_.empty(), "no beam search in flight");
    const Pending pd = pending_.front();
    pending_.erase(pending_.begin());
    const int L = cfg_.n_code_layers;
    if (!pd.has_out || !out) {
      CUDA_CHECK(cudaEventSynchronize(dev_free_[pd.slot]));
      CUDA_CHECK(cudaGetLastError());
    check_ep();
      return;
    }
    CUDA_CHECK(cudaEventSynchronize(out_ready_[pd.slot]));
    CUDA_CHECK(cudaGetLastError());
    check_ep();
    const int U = pd.U, n_live = pd.n_live, width = pd.width;
    const size_t nc = static_cast<size_t>(U) * n_live * L;
    const uint8_t* ho = static_cast<const uint8_t*>(host_out_[pd.slot]);
    const int32_t* hc = reinterpret_cast<const int32_t*>(ho);
    const double* hl = reinterpret_cast<const double*>(ho + nc * 4);
    int32_t bad = 0;
    memcpy(&bad, ho + nc * 4 + static_cast<size_t>(U) * n_live * 8, 4);
    if (bad) throw RuntimeError("non-finite value produced on tape");  // tape.cpp:29
    for (int u = 0; u < U; ++u) {
      int n_u = n_live;  // constrained search: empty slots (log-prob -inf) sort last
      while (n_u > 0 && std::isinf(hl[(size_t)u * n_live + n_u - 1])) --n_u;
      if (out->n_items) out->n_items[u] = n_u;
      for (int b = 0; b < width; ++b) {
        for (int j = 0; j < L; ++j)
          out->codes[((size_t)u * width + b) * L + j] = b < n_u ? hc[((size_t)u * n_live + b) * L + j] : -1;
        out->log_prob[(size_t)u * width + b] = b < n_u ? hl[(size_t)u * n_live + b] : 0.0;
      }
    }
  }

  void run_beam(int width, orx_beam_out* out, bool constrained) {
    while (!pending_.empty()) collect_beam(nullptr);  // synchronous call: nothing else in flight
    launch_beam(width, constrained, out != nullptr);
    collect_beam(out);
    CUDA_CHECK(cudaStreamSynchronize(st_));
    CUDA_CHECK(cudaGetLastError());
    check_ep();
  }

  // Pipelined serving: stage + launch request i+1 while request i runs; at
  // most two in flight (one per staging slot).
  void submit_beam(const orx_user_batch& b, int width) override {
    require(pending_.size() < 2, "two beam searches already in flight: collect one first");
    for (const Pending& p : pending_) require(p.has_out, "a staged-only search is in flight");
    stage_batch(b);
    launch_beam(width, false, true);
  }
  void collect(orx_beam_out* out) override {
    require(out && out->codes && out->log_prob, "collect needs output arrays");
    collect_beam(out);
  }

  // Teacher-forced logits. Queries are grouped by encoder row block; every
  // query is its own row at every position (anc[r][p] = r).
  void teacher_forced(int n_groups_users, int n, const int32_t* z_index, const int32_t* prefixes,
                      const int32_t* prefix_len, float* logits) {
    const orx_config& c = cfg_;
    const int V = c.codebook_size, L = c.n_code_layers, Tn = enc_seq_len(c);
    require(n >= 0 && n <= Rd_, "too many prefix queries for the engine capacity");
    if (n == 0) return;
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return z_index[a] < z_index[b]; });
    std::vector<int32_t> codes(static_cast<size_t>(n) * L, 0), anc(static_cast<size_t>(n) * L), gs, gl, gk;
    int max_len = 0, max_group = 0;
    for (int r = 0; r < n; ++r) {
      const int q = order[r];
      require(z_index[q] >= 0 && z_index[q] < n_groups_users, "query user index out of range");
      require(prefix_len[q] >= 0 && prefix_len[q] < L, "no prediction head at this position");
      max_len = std::max(max_len, prefix_len[q]);
      for (int j = 0; j < L; ++j) {
        anc[(size_t)r * L + j] = r;
        if (j < prefix_len[q]) {
          int code = prefixes[(size_t)q * L + j];
          require(code >= 0 && code < V, "decoder token outside its layer vocabulary");
          codes[(size_t)r * L + j] = code;
        }
      }
      if (r == 0 || z_index[order[r - 1]] != z_index[q]) {
        gs.push_back(r);
        gl.push_back(0);
        gk.push_back(z_index[q] * Tn);
      }
      ++gl.back();
      max_group = std::max(max_group, gl.back());
    }
    const int G = static_cast<int>(gs.size());
    CUDA_CHECK(cudaMemcpyAsync(tf_codes_, codes.data(), codes.size() * 4, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemcpyAsync(tf_anc_, anc.data(), anc.size() * 4, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemcpyAsync(grp_start_, gs.data(), G * 4, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemcpyAsync(grp_len_, gl.data(), G * 4, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemcpyAsync(grp_kstart_, gk.data(), G * 4, cudaMemcpyHostToDevice, st_));
    std::vector<int32_t> gu(G);
    for (int g = 0; g < G; ++g) gu[g] = gk[g] / Tn;
    CUDA_CHECK(cudaMemcpyAsync(grp_user_, gu.data(), G * 4, cudaMemcpyHostToDevice, st_));
    Seg gq;
    gq.start = grp_start_;
    gq.len = grp_len_;
    Seg gkseg;
    gkseg.start = grp_kstart_;
    gkseg.fixed_len = Tn;
    std::vector<float> host(static_cast<size_t>(n) * V);
    if (ep_world_ > 1) max_len = L - 1;  // expert-parallel ranks run the same number of MoE layers
    for (int step = 0; step <= max_len; ++step) {
      decode_step(step, n, G, gq, gkseg, tf_codes_, L, tf_anc_, L, max_group, grp_user_);
      CUDA_CHECK(cudaMemcpyAsync(host.data(), logits_, host.size() * 4, cudaMemcpyDeviceToHost, st_));
      CUDA_CHECK(cudaStreamSynchronize(st_));
      for (int r = 0; r < n; ++r)
        if (prefix_len[order[r]] == step) {
          require_finite(host.data() + (size_t)r * V, static_cast<size_t>(V));
          memcpy(logits + (size_t)order[r] * V, host.data() + (size_t)r * V, static_cast<size_t>(V) * 4);
        }
    }
    CUDA_CHECK(cudaGetLastError());
    check_ep();
  }

  void score_prefixes(int n, const int32_t* user, const int32_t* prefixes, const int32_t* prefix_len,
                      float* logits) override {
    CUDA_CHECK(cudaSetDevice(dev_));
    run_encode();
    prepare_decoder(sg_.U);
    teacher_forced(sg_.U, n, user, prefixes, prefix_len, logits);
  }

  void sample(int width, double temperature, int top_k, double top_p, uint64_t seed, const uint64_t* streams,
              orx_beam_out* out) override {
    CUDA_CHECK(cudaSetDevice(dev_));
    const orx_config& c = cfg_;
    // validate_request, generation.cpp:34-39
    require(width >= 1, "generation width must be >= 1");
    require(top_p > 0 && top_p <= 1.0, "top_p must lie in (0,1]");
    require(top_k >= 0, "top_k must be >= 1 (or 0 for the full vocabulary)");
    require(temperature > 0, "temperature must be positive");
    require(width <= maxW_, "sample count above the engine capacity");
    const int U = sg_.U, V = c.codebook_size, L = c.n_code_layers, Tn = enc_seq_len(c);
    const int rows = U * width;
    run_encode();
    prepare_decoder(U);
    // the reference draws one uniform per (sample, step), sample-major, from the user's Rng
    std::vector<double> uni(static_cast<size_t>(rows) * L);
    for (int u = 0; u < U; ++u) {
      Rng r = Rng(seed).split(streams ? streams[u] : static_cast<uint64_t>(u));
      for (int s = 0; s < width; ++s)
        for (int j = 0; j < L; ++j) uni[((size_t)u * width + s) * L + j] = r.uniform();
    }
    if (!uni_) uni_ = ar_.alloc<double>(static_cast<size_t>(Rd_) * L);
    std::vector<int32_t> anc(static_cast<size_t>(rows) * L);
    for (int r = 0; r < rows; ++r)
      for (int j = 0; j < L; ++j) anc[(size_t)r * L + j] = r;
    CUDA_CHECK(cudaMemcpyAsync(uni_, uni.data(), uni.size() * 8, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemcpyAsync(tf_anc_, anc.data(), anc.size() * 4, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemsetAsync(tf_codes_, 0, static_cast<size_t>(rows) * L * 4, st_));
    CUDA_CHECK(cudaMemsetAsync(seq_acc_, 0, static_cast<size_t>(rows) * 8, st_));
    Seg gq;
    gq.stride = width;
    gq.fixed_len = width;
    Seg gk;
    gk.stride = Tn;
    gk.fixed_len = Tn;
    for (int step = 0; step < L; ++step) {
      decode_step(step, rows, U, gq, gk, tf_codes_, L, tf_anc_, L, width);
      launch_sample(rows, V, L, step, static_cast<float>(temperature), top_k, top_p, logits_, uni_, tf_codes_,
                    seq_acc_, st_);
    }
    std::vector<int32_t> hc(static_cast<size_t>(rows) * L);
    std::vector<double> hl(rows);
    CUDA_CHECK(cudaMemcpyAsync(hc.data(), tf_codes_, hc.size() * 4, cudaMemcpyDeviceToHost, st_));
    CUDA_CHECK(cudaMemcpyAsync(hl.data(), seq_acc_, hl.size() * 8, cudaMemcpyDeviceToHost, st_));
    CUDA_CHECK(cudaStreamSynchronize(st_));
    CUDA_CHECK(cudaGetLastError());
    check_ep();
    d2h_bytes += static_cast<int64_t>(hc.size() * 4 + hl.size() * 8);
    require_finite(hl.data(), hl.size());
    for (int u = 0; u < U; ++u) {
      if (out->n_items) out->n_items[u] = width;
      for (int s = 0; s < width; ++s) {
        for (int j = 0; j < L; ++j)
          out->codes[((size_t)u * width + s) * L + j] = hc[((size_t)u * width + s) * L + j];
        out->log_prob[(size_t)u * width + s] = hl[(size_t)u * width + s];
      }
    }
  }

  // PolicyModel::sequence_log_prob (policy.cpp:297-310) for n queries: decode
  // [BOS, c1 .. c_{L-1}] teacher-forced and sum log_softmax(logits_j)[c_j] (f64).
  void sequence_log_prob(int n, const int32_t* user, const int32_t* codes, double* out) override {
    CUDA_CHECK(cudaSetDevice(dev_));
    const orx_config& c = cfg_;
    const int L = c.n_code_layers, V = c.codebook_size, Tn = enc_seq_len(c);
    require(n >= 0 && n <= Rd_, "too many sequences for the engine capacity");
    for (int q = 0; q < n; ++q) {
      require(user[q] >= 0 && user[q] < sg_.U, "query user index out of range");
      for (int j = 0; j < L; ++j)
        require(codes[(size_t)q * L + j] >= 0 && codes[(size_t)q * L + j] < V, "target must be a full semantic id");
    }
    run_encode();
    prepare_decoder(sg_.U);
    if (n == 0) return;
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return user[a] < user[b]; });
    std::vector<int32_t> cs(static_cast<size_t>(n) * L), anc(static_cast<size_t>(n) * L), gs, gl, gk, gu;
    int max_group = 0;
    for (int r = 0; r < n; ++r) {
      const int q = order[r];
      for (int j = 0; j < L; ++j) {
        cs[(size_t)r * L + j] = codes[(size_t)q * L + j];
        anc[(size_t)r * L + j] = r;
      }
      if (r == 0 || user[order[r - 1]] != user[q]) {
        gs.push_back(r);
        gl.push_back(0);
        gk.push_back(user[q] * Tn);
        gu.push_back(user[q]);
      }
      ++gl.back();
      max_group = std::max(max_group, gl.back());
    }
    const int G = static_cast<int>(gs.size());
    CUDA_CHECK(cudaMemcpyAsync(tf_codes_, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemcpyAsync(tf_anc_, anc.data(), anc.size() * 4, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemcpyAsync(grp_start_, gs.data(), G * 4, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemcpyAsync(grp_len_, gl.data(), G * 4, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemcpyAsync(grp_kstart_, gk.data(), G * 4, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemcpyAsync(grp_user_, gu.data(), G * 4, cudaMemcpyHostToDevice, st_));
    CUDA_CHECK(cudaMemsetAsync(seq_acc_, 0, static_cast<size_t>(n) * 8, st_));
    Seg gq;
    gq.start = grp_start_;
    gq.len = grp_len_;
    Seg gkseg;
    gkseg.start = grp_kstart_;
    gkseg.fixed_len = Tn;
    for (int step = 0; step < L; ++step) {  // position j predicts code j from [BOS, c1 .. c_j]
      decode_step(step, n, G, gq, gkseg, tf_codes_, L, tf_anc_, L, max_group, grp_user_);
      launch_pick_logprob(n, V, logits_, tf_codes_, L, step, seq_acc_, st_);
    }
    std::vector<double> host(n);
    CUDA_CHECK(cudaMemcpyAsync(host.data(), seq_acc_, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, st_));
    CUDA_CHECK(cudaStreamSynchronize(st_));
    CUDA_CHECK(cudaGetLastError());
    check_ep();
    require_finite(host.data(), host.size());
    for (int r = 0; r < n; ++r) out[order[r]] = host[r];
  }

  void next_logits(const float* z, int n_z, int n, const int32_t* z_index, const int32_t* prefixes,
                   const int32_t* prefix_len, float* logits) override {
    CUDA_CHECK(cudaSetDevice(dev_));
    require(n_z >= 1 && n_z <= maxU_, "encoding count outside the engine capacity");
    const size_t nz = static_cast<size_t>(n_z) * enc_seq_len(cfg_) * cfg_.d_model;
    require_finite(z, nz);
    CUDA_CHECK(cudaMemcpyAsync(z_, z, nz * 4, cudaMemcpyHostToDevice, st_));
    zt_fresh_ = false;  // caller-supplied encodings: convert
    prepare_decoder(n_z);
    teacher_forced(n_z, n, z_index, prefixes, prefix_len, logits);
  }

 private:
  orx_config cfg_;
  int dev_, maxU_, maxW_;
  cudaStream_t st_ = nullptr;
  Arena ar_;
  // weights
  const float *t_uid_, *t_gender_, *t_age_, *t_vid_, *t_aid_, *t_label_, *t_tag_, *t_ts_, *t_play_, *t_dur_;
  const float *pad_s_, *pad_p_, *pad_l_, *pos_, *bos_;
  const __nv_bfloat16 *t_vid16_ = nullptr, *t_aid16_ = nullptr;
  std::vector<const float*> tokens_;
  std::vector<Lin<T>> heads_;
  Mlp p_static_, p_short_, p_pos_, p_life_;
  // short / positive / lifelong fc1 folded through the feature tables (bf16)
  FoldTables fold_[3];
  bool fold_on_ = false;
  const T* queries_ = nullptr;
  std::vector<QBlock> qblocks_;
  std::vector<EncL> enc_;
  std::vector<DecL> dec_;
  Lin<T> xkv_w_, qkv_all_;
  Lin<T> kvf_;                    // lifelong fc2 folded into the QFormer K|V weights (build_kv_fold)
  const float* kv_pad_ = nullptr;  // pad.lifelong . Wkv
  bool kv_fold_ = false;
  bool fold_norm_ = false;        // RMSNorm folded into the GEMMs around it (bf16, d % 256 == 0)
  const float* ones_ = nullptr;   // unit gain for the explicit gain-free norms of the folded path
  float* ssq_ = nullptr;
  long long ssq_ld_ = 0;
  bool tc_attn_ = false;
  int Tpad_ = 0, Lpad_ = 0;
  T *vt_enc_ = nullptr, *vt_q_ = nullptr, *vt_x_ = nullptr;
  int32_t* grp_user_ = nullptr;
  // activations
  int Fp_ = 0, Sp_ = 0;
  int64_t Rd_ = 0, S_ = 0;
  int max_tiles_ = 0;
  T *feat_, *hid_, *keys_, *kvl_, *xn_, *qkv_, *att_, *ffh_, *qproj_, *qcur_, *zt_, *xkv_;
  float *z_, *qo_, *h_, *logits_, *lse_;
  bool zt_fresh_ = false;  // zt_ = bf16(z_) was written by the encoder's last GEMM / combine
  std::vector<T*> kvpos_;       // [position * dec_layers + layer] -> [Rd_][3d] QKV output (self-attention cache)
  T** kvpos_ptrs_ = nullptr;
  uint64_t* cand_ = nullptr;
  int32_t* topk_fail_ = nullptr;
  BeamState bs_[2];
  int32_t* nonfinite_ = nullptr;
  bool fused_select_ = false;
  float2* head_stats_ = nullptr;     // [V/32][Rd_] head GEMM chunk statistics
  uint32_t* sel_scratch_ = nullptr;  // beam_select chunk keys that do not fit on chip
  int32_t* node_[2] = {nullptr, nullptr};
  // device trie (constrained search)
  Arena trie_ar_;
  TrieDev trie_;
  bool has_trie_ = false;
  double* seq_acc_ = nullptr;
  double* uni_ = nullptr;
  WorkerPool pool_{static_cast<int>(std::clamp(std::thread::hardware_concurrency(), 1u, 16u))};
  int32_t *tf_anc_, *tf_codes_, *grp_start_, *grp_len_, *grp_kstart_;
  int32_t *sel_ = nullptr, *slot_ = nullptr, *counts_ = nullptr, *cursor_ = nullptr, *tile_expert_ = nullptr,
          *n_mtiles_ = nullptr;
  float *wts_ = nullptr, *row_scale_ = nullptr, *ga_ = nullptr, *gb_ = nullptr;
  T* yg_ = nullptr;  // weighted expert outputs (bf16 in the bf16 engine)
  float* row_rsq_ = nullptr;  // folded pre-MoE RMSNorm: scale of every grouped row
  float* route_part_ = nullptr;      // tensor-pipe router: K-half partial scores
  int32_t* route_ticket_ = nullptr;  // tensor-pipe router: per-tile arrival tickets (after counts_)
  int n_route_tickets_ = 0;
  T *xg_ = nullptr, *hg_ = nullptr;
  // expert parallelism
  int ep_rank_ = 0, ep_world_ = 1, El_ = 0;  // El_: local expert slots per MoE layer
  EpPlacement place_;                  // expert parallelism: who computes which expert (ep_plan.hpp)
  int n_moe_ = 0;                      // MoE layers packed so far (MoeW::li)
  std::vector<long long*> ep_loads_;   // per MoE layer: accumulated global rows per expert
  const bool route_stats_ = getenv("ORX_ROUTE_STATS") != nullptr;
  std::vector<std::vector<int32_t>> route_hist_;
  ncclComm_t comm_ = nullptr;
  EpPeers ep_{};                      // peer views of the symmetric exchange regions
  void* ep_region_ = nullptr;          // this rank's region
  std::vector<void*> ep_peer_base_;    // every rank's region mapped here
  int32_t *ep_seg_ = nullptr, *ep_tiles_ = nullptr, *ep_ntiles_ = nullptr;
  // staging
  void* host_stage_[2] = {nullptr, nullptr};
  uint8_t* dev_stage_[2] = {nullptr, nullptr};
  size_t stage_cap_[2] = {0, 0};
  int stage_slot_ = 1;  // slot of the most recently staged batch (the first batch goes to slot 0)
  cudaStream_t cs_ = nullptr;  // H2D copy stream
  cudaEvent_t h2d_done_[2] = {}, dev_free_[2] = {}, out_ready_[2] = {};
  bool staged_ = false;
  void* host_out_[2] = {nullptr, nullptr};
  size_t host_out_cap_[2] = {0, 0};
  struct Pending {
    int slot, U, n_live, width;
    bool has_out;
  };
  std::vector<Pending> pending_;
  struct CachedGraph {
    GraphKey key;
    cudaGraphExec_t exec = nullptr;
    long long kernels = 0;
  };
  std::vector<CachedGraph> graphs_;
  int last_n_live_ = 0, last_state_ = 0;
};

void nccl_unique_id(uint8_t out[128]) {
  ncclUniqueId id;
  NCCL_CHECK(nccl().GetUniqueId(&id));
  memcpy(out, id.internal, 128);
}

std::unique_ptr<Engine> Engine::create(const HostWeights& w, int device, int precision, int max_users,
                                       int max_width, const EpConfig* ep) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    throw RuntimeError("no CUDA device available (the engine has no CPU fallback)");
  }
  require(device >= 0 && device < n, "device index out of range");
  if (precision == ORX_PRECISION_FP32) return std::make_unique<EngineT<float>>(w, device, max_users, max_width, ep);
  if (precision == ORX_PRECISION_BF16)
    return std::make_unique<EngineT<__nv_bfloat16>>(w, device, max_users, max_width, ep);
  throw InvalidArgument("unknown precision");
}

}  // namespace orx
