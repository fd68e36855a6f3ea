// extern "C" boundary (include/orx.h). Exceptions never cross it: they are
// mapped to ORX_EINVAL / ORX_ERUNTIME / ORX_ECUDA plus a thread-local message.
#include <cuda_bf16.h>

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/orx.h"
#include "engine.hpp"
#include "ep_plan.hpp"
#include "attention.cuh"
#include "beam.cuh"
#include "kernels.cuh"
#include "compress.cuh"
#include "gemm.cuh"
#include "model.hpp"
#include "synth_users.hpp"

struct orx_weights {
  orx::HostWeights w;
};
struct orx_engine {
  std::unique_ptr<orx::Engine> e;
  const orx::HostWeights* w = nullptr;
  orx_config cfg{};
  int staged_users = 0;
};
struct orx_synth_batch {
  std::vector<int32_t> uid, gender, age;
  struct P {
    std::vector<int64_t> offsets, vid;
    std::vector<int32_t> aid;
    std::vector<double> tag, ts, play, dur;
    std::vector<uint32_t> labels;
  } p[3];
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return ORX_OK;
  } catch (const orx::InvalidArgument& e) {
    g_err = e.what();
    return ORX_EINVAL;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return ORX_EINVAL;
  } catch (const orx::RuntimeError& e) {
    g_err = e.what();
    return std::string(e.what()).rfind("CUDA", 0) == 0 || strstr(e.what(), "CUDA") ? ORX_ECUDA : ORX_ERUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ORX_ERUNTIME;
  } catch (...) {
    g_err = "unknown error";
    return ORX_ERUNTIME;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw orx::InvalidArgument(std::string(what) + " must not be NULL");
}

}  // namespace

extern "C" {

const char* orx_last_error(void) { return g_err.c_str(); }
const char* orx_version(void) { return "orx 0.1 (sm_100a)"; }

int orx_config_default(orx_config* cfg) {
  return guarded([&] {
    need(cfg, "cfg");
    *cfg = orx::config_default();
  });
}

int orx_config_preset(const char* name, orx_config* cfg) {
  return guarded([&] {
    need(cfg, "cfg");
    need(name, "name");
    *cfg = orx::config_preset(name);
  });
}

int64_t orx_config_enc_seq_len(const orx_config* cfg) { return cfg ? orx::enc_seq_len(*cfg) : -1; }
int64_t orx_config_expert_hidden(const orx_config* cfg) {
  int64_t v = -1;
  guarded([&] {
    need(cfg, "cfg");
    v = orx::expert_hidden(*cfg);
  });
  return v;
}

int orx_weights_create_random(const orx_config* cfg, orx_weights** out) {
  return guarded([&] {
    need(cfg, "cfg");
    need(out, "out");
    auto w = std::make_unique<orx_weights>();
    w->w = orx::HostWeights::random(*cfg);
    *out = w.release();
  });
}

int orx_weights_create_random_ep(const orx_config* cfg, int32_t ep_rank, int32_t ep_world, orx_weights** out) {
  return orx_weights_create_random_ep_placed(cfg, ep_rank, ep_world, nullptr, out);
}

namespace {
// a caller's placement table, validated (shape, owners, slot capacity)
orx::EpPlacement placement_of(const orx_config& cfg, int32_t world, const int32_t* owner) {
  orx::EpPlacement p;
  p.layers = orx::moe_layers(cfg);
  p.E = cfg.n_experts;
  p.W = world;
  p.owner.assign(owner, owner + static_cast<size_t>(p.layers) * p.E);
  p.validate();
  return p;
}
}  // namespace

int orx_weights_create_random_ep_placed(const orx_config* cfg, int32_t ep_rank, int32_t ep_world,
                                        const int32_t* owner, orx_weights** out) {
  return guarded([&] {
    need(cfg, "cfg");
    need(out, "out");
    if (owner) {
      if (!cfg->moe_enabled) throw orx::InvalidArgument("expert placement needs a MoE config");
      placement_of(*cfg, ep_world, owner);
    }
    auto w = std::make_unique<orx_weights>();
    w->w = orx::HostWeights::random(*cfg, ep_rank, ep_world, owner);
    *out = w.release();
  });
}

int32_t orx_config_moe_layers(const orx_config* cfg) { return cfg ? orx::moe_layers(*cfg) : 0; }

int orx_ep_place(const int64_t* load, int32_t layers, int32_t n_experts, int32_t world, int32_t min_replicas,
                 int32_t max_replicas, int32_t* owner_out, double* predicted_imbalance) {
  return guarded([&] {
    need(load, "load");
    need(owner_out, "owner_out");
    std::vector<double> pred;
    const orx::EpPlacement p =
        orx::ep_place_balanced(load, layers, n_experts, world, max_replicas, 1.05, &pred, min_replicas);
    p.validate();
    std::copy(p.owner.begin(), p.owner.end(), owner_out);
    if (predicted_imbalance) std::copy(pred.begin(), pred.end(), predicted_imbalance);
  });
}

int orx_weights_load_grcp(const char* path, orx_weights** out) {
  return guarded([&] {
    need(path, "path");
    need(out, "out");
    auto w = std::make_unique<orx_weights>();
    w->w = orx::HostWeights::load_grcp(path);
    *out = w.release();
  });
}

int orx_weights_save_grcp(const orx_weights* w, const char* path) {
  return guarded([&] {
    need(w, "weights");
    need(path, "path");
    w->w.save_grcp(path);
  });
}

int orx_weights_config(const orx_weights* w, orx_config* cfg) {
  return guarded([&] {
    need(w, "weights");
    need(cfg, "cfg");
    *cfg = w->w.cfg;
  });
}

int64_t orx_weights_count(const orx_weights* w) { return w ? static_cast<int64_t>(w->w.tensors.size()) : -1; }

int orx_weights_entry(const orx_weights* w, int64_t i, const char** name, int32_t* ndim, int32_t dims[2],
                      const float** data) {
  return guarded([&] {
    need(w, "weights");
    if (i < 0 || i >= static_cast<int64_t>(w->w.tensors.size())) throw orx::InvalidArgument("entry index out of range");
    const orx::Tensor& t = w->w.tensors[static_cast<size_t>(i)];
    if (name) *name = t.name.c_str();
    if (ndim) *ndim = 2;
    if (dims) {
      dims[0] = t.rows;
      dims[1] = t.cols;
    }
    if (data) *data = t.data.data();
  });
}

int orx_weights_find(const orx_weights* w, const char* name, int64_t* index) {
  return guarded([&] {
    need(w, "weights");
    need(name, "name");
    auto it = w->w.index.find(name);
    if (it == w->w.index.end()) throw orx::InvalidArgument(std::string("unknown parameter: ") + name);
    if (index) *index = it->second;
  });
}

int orx_weights_set(orx_weights* w, const char* name, const float* data, int64_t n) {
  return guarded([&] {
    need(w, "weights");
    need(name, "name");
    need(data, "data");
    auto it = w->w.index.find(name);
    if (it == w->w.index.end()) throw orx::InvalidArgument(std::string("unknown parameter: ") + name);
    orx::Tensor& t = w->w.tensors[static_cast<size_t>(it->second)];
    if (n != static_cast<int64_t>(t.data.size())) throw orx::InvalidArgument(std::string("size mismatch for ") + name);
    std::copy(data, data + n, t.data.begin());
  });
}

void orx_weights_destroy(orx_weights* w) { delete w; }

int orx_validate_batch(const orx_config* cfg, const orx_user_batch* batch) {
  return guarded([&] {
    need(cfg, "cfg");
    need(batch, "batch");
    orx::validate_batch(*cfg, *batch);
  });
}

int orx_engine_create(const orx_weights* w, int device, int precision, int32_t max_users, int32_t max_width,
                      orx_engine** out) {
  return guarded([&] {
    need(w, "weights");
    need(out, "out");
    auto e = std::make_unique<orx_engine>();
    e->e = orx::Engine::create(w->w, device, precision, max_users, max_width);
    e->w = &w->w;
    e->cfg = w->w.cfg;
    *out = e.release();
  });
}

int orx_ep_unique_id(uint8_t id_out[ORX_EP_ID_BYTES]) {
  return guarded([&] {
    need(id_out, "id_out");
    orx::nccl_unique_id(id_out);
  });
}

int orx_engine_create_ep(const orx_weights* w, int device, int precision, int32_t max_users, int32_t max_width,
                         const uint8_t id[ORX_EP_ID_BYTES], int32_t ep_rank, int32_t ep_world, orx_engine** out) {
  return orx_engine_create_ep_placed(w, device, precision, max_users, max_width, id, ep_rank, ep_world, nullptr, out);
}

int orx_engine_create_ep_placed(const orx_weights* w, int device, int precision, int32_t max_users,
                                int32_t max_width, const uint8_t id[ORX_EP_ID_BYTES], int32_t ep_rank,
                                int32_t ep_world, const int32_t* owner, orx_engine** out) {
  return guarded([&] {
    need(w, "weights");
    need(out, "out");
    need(id, "id");
    orx::EpConfig ep;
    ep.rank = ep_rank;
    ep.world = ep_world;
    memcpy(ep.unique_id, id, ORX_EP_ID_BYTES);
    if (owner) {
      if (!w->w.cfg.moe_enabled) throw orx::InvalidArgument("expert placement needs a MoE config");
      ep.owner = placement_of(w->w.cfg, ep_world, owner).owner;
    }
    auto e = std::make_unique<orx_engine>();
    e->e = orx::Engine::create(w->w, device, precision, max_users, max_width, &ep);
    e->w = &w->w;
    e->cfg = w->w.cfg;
    *out = e.release();
  });
}

void orx_engine_destroy(orx_engine* e) { delete e; }

int orx_engine_expert_load(orx_engine* e, int64_t* load_out, int32_t reset) {
  return guarded([&] {
    need(e, "engine");
    need(load_out, "load_out");
    e->e->expert_load(load_out, reset != 0);
  });
}

int orx_encode(orx_engine* e, const orx_user_batch* batch, float* z_out) {
  return guarded([&] {
    need(e, "engine");
    need(batch, "batch");
    e->e->require_idle();
    e->e->stage_batch(*batch);
    e->e->encode(z_out);
  });
}

int orx_next_logits(orx_engine* e, const float* z_enc, int32_t n_z, int32_t n, const int32_t* z_index,
                    const int32_t* prefixes, const int32_t* prefix_len, float* logits_out) {
  return guarded([&] {
    need(e, "engine");
    need(z_enc, "z_enc");
    need(z_index, "z_index");
    need(prefixes, "prefixes");
    need(prefix_len, "prefix_len");
    need(logits_out, "logits_out");
    e->e->next_logits(z_enc, n_z, n, z_index, prefixes, prefix_len, logits_out);
  });
}

int orx_score_prefixes(orx_engine* e, const orx_user_batch* batch, int32_t n, const int32_t* user,
                       const int32_t* prefixes, const int32_t* prefix_len, float* logits_out) {
  return guarded([&] {
    need(e, "engine");
    need(batch, "batch");
    need(user, "user");
    need(prefixes, "prefixes");
    need(prefix_len, "prefix_len");
    need(logits_out, "logits_out");
    e->e->require_idle();
    e->e->stage_batch(*batch);
    e->e->score_prefixes(n, user, prefixes, prefix_len, logits_out);
  });
}

int orx_beam_search(orx_engine* e, const orx_user_batch* batch, int32_t width, orx_beam_out* out) {
  return guarded([&] {
    need(e, "engine");
    need(batch, "batch");
    need(out, "out");
    need(out->codes, "out->codes");
    need(out->log_prob, "out->log_prob");
    e->e->require_idle();
    e->e->stage_batch(*batch);
    e->e->beam_search(width, out);
  });
}

int orx_beam_search_submit(orx_engine* e, const orx_user_batch* batch, int32_t width) {
  return guarded([&] {
    need(e, "engine");
    need(batch, "batch");
    e->e->submit_beam(*batch, width);
  });
}

int orx_beam_search_collect(orx_engine* e, orx_beam_out* out) {
  return guarded([&] {
    need(e, "engine");
    need(out, "out");
    e->e->collect(out);
  });
}

int orx_engine_set_trie(orx_engine* e, const orx_trie* t) {
  return guarded([&] {
    need(e, "engine");
    need(t, "trie");
    e->e->require_idle();
    e->e->set_trie(t->n_nodes, t->child_off, t->n_edges, t->child_code, t->child_node);
  });
}

int orx_beam_search_constrained(orx_engine* e, const orx_user_batch* batch, int32_t width, orx_beam_out* out) {
  return guarded([&] {
    need(e, "engine");
    need(batch, "batch");
    need(out, "out");
    need(out->codes, "out->codes");
    need(out->log_prob, "out->log_prob");
    e->e->require_idle();
    e->e->stage_batch(*batch);
    e->e->beam_search_constrained(width, out);
  });
}

int orx_sequence_log_prob(orx_engine* e, const orx_user_batch* batch, int32_t n, const int32_t* user,
                          const int32_t* codes, double* log_prob_out) {
  return guarded([&] {
    need(e, "engine");
    need(batch, "batch");
    if (n > 0) {
      need(user, "user");
      need(codes, "codes");
      need(log_prob_out, "log_prob_out");
    }
    e->e->require_idle();
    e->e->stage_batch(*batch);
    e->e->sequence_log_prob(n, user, codes, log_prob_out);
  });
}

int orx_sample(orx_engine* e, const orx_user_batch* batch, int32_t width, double temperature, int32_t top_k,
               double top_p, uint64_t seed, const uint64_t* user_stream, orx_beam_out* out) {
  return guarded([&] {
    need(e, "engine");
    need(batch, "batch");
    need(out, "out");
    need(out->codes, "out->codes");
    need(out->log_prob, "out->log_prob");
    e->e->require_idle();
    e->e->stage_batch(*batch);
    e->e->sample(width, temperature, top_k, top_p, seed, user_stream, out);
  });
}

int orx_engine_stage_batch(orx_engine* e, const orx_user_batch* batch) {
  return guarded([&] {
    need(e, "engine");
    need(batch, "batch");
    e->e->require_idle();
    e->e->stage_batch(*batch);
  });
}

int orx_beam_search_staged(orx_engine* e, int32_t width, orx_beam_out* out) {
  return guarded([&] {
    need(e, "engine");
    e->e->require_idle();
    e->e->beam_search(width, out);
  });
}

int orx_engine_stats(const orx_engine* e, int64_t* launches, int64_t* h2d, int64_t* d2h) {
  return guarded([&] {
    need(e, "engine");
    if (launches) *launches = orx::launch_counter_value();
    if (h2d) *h2d = e->e->h2d_bytes;
    if (d2h) *d2h = e->e->d2h_bytes;
  });
}

void* orx_engine_stream(orx_engine* e) { return e ? e->e->stream() : nullptr; }

int orx_profile_enable(int on) {
  return guarded([&] { orx::prof_enable(on != 0); });
}

int orx_profile_read(int32_t n, int64_t* launches, double* ms, double* flops, double* bytes) {
  return guarded([&] {
    long long c[orx::PROF_N];
    double t[orx::PROF_N], f[orx::PROF_N], b[orx::PROF_N];
    orx::prof_collect(c, t, f, b);
    for (int i = 0; i < n && i < orx::PROF_N; ++i) {
      if (launches) launches[i] = c[i];
      if (ms) ms[i] = t[i];
      if (flops) flops[i] = f[i];
      if (bytes) bytes[i] = b[i];
    }
  });
}

int orx_debug_gemm(const orx_gemm_args* a, void* stream) {
  return guarded([&] {
    need(a, "args");
    orx::Epi e;
    e.bias = a->bias;
    e.row_scale = a->row_scale;
    e.resid = a->resid;
    e.ld_resid = a->ld_resid;
    e.out = a->out;
    e.row_map = a->row_map;
    e.ldo = a->ldo;
    e.out_bf16 = a->out_bf16;
    e.act = a->act;
    e.swiglu = a->swiglu;
    e.n_out = a->n_out ? a->n_out : (a->swiglu ? a->N / 2 : a->N);
    e.m_valid = a->m_valid ? a->m_valid : a->M;
    e.col_off = a->col_off;
    orx::Grouped g;
    g.tile_expert = a->tile_expert;
    g.n_mtiles = a->n_mtiles;
    g.b_rows_per_expert = a->b_rows_per_expert;
    g.n_groups = a->n_groups;
    g.tile_rows = a->tile_rows ? a->tile_rows : 128;
    g.algo_rows = a->M;
    auto st = static_cast<cudaStream_t>(stream);
    const bool saved = orx::force_single_cta();
    orx::force_single_cta() = a->force_single_cta != 0;
    try {
      if (a->precision == ORX_PRECISION_BF16)
        orx::gemm_bf16(a->A, a->lda, a->B, a->ldb, a->M, a->N, a->K, e, a->tile_expert ? &g : nullptr, st);
      else
        orx::gemm_f32(static_cast<const float*>(a->A), a->lda, static_cast<const float*>(a->B), a->ldb, a->M, a->N,
                      a->K, e, a->tile_expert ? &g : nullptr, st);
    } catch (...) {
      orx::force_single_cta() = saved;
      throw;
    }
    orx::force_single_cta() = saved;
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) throw orx::RuntimeError(std::string("CUDA: ") + cudaGetErrorString(err));
  });
}

int orx_debug_row_topk(int32_t rows, int32_t V, int32_t k, const float* logits, const float* pscore,
                       const int32_t* plex, float* lse, uint64_t* cand, void* stream) {
  return guarded([&] {
    if (rows < 0 || V < 1 || k < 1 || k > V) throw orx::InvalidArgument("row_topk: bad sizes");
    int32_t* fail = nullptr;
    if (cudaMalloc(&fail, (static_cast<size_t>(rows) + 1) * sizeof(int32_t)) != cudaSuccess)
      throw orx::RuntimeError("CUDA: workspace allocation failed");
    orx::launch_row_topk(rows, V, k, logits, pscore, plex, lse, cand, fail, static_cast<cudaStream_t>(stream));
    cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
    cudaFree(fail);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) throw orx::RuntimeError(std::string("CUDA: ") + cudaGetErrorString(err));
  });
}

int orx_debug_attention(const orx_attn_args* a, void* stream) {
  return guarded([&] {
    need(a, "args");
    orx::Seg q, k, o;
    q.start = a->q_start, q.len = a->q_len, q.stride = a->q_stride, q.fixed_len = a->q_fixed;
    k.start = a->k_start, k.len = a->k_len, k.stride = a->k_stride, k.fixed_len = a->k_fixed;
    o.start = a->o_start, o.stride = a->o_stride;
    auto st = static_cast<cudaStream_t>(stream);
    if (a->kernel == 1) {
      orx::FmhaArgs f;
      f.B = a->B, f.max_q = a->max_q, f.heads = a->heads, f.dh = a->dh;
      f.Q = a->Q, f.q_rows = a->q_rows, f.ldq = a->ldq, f.q_col0 = a->q_col0;
      f.K = a->K, f.k_rows = a->k_rows, f.ldk = a->ldk, f.k_col0 = a->k_col0;
      f.Vt = a->Vt, f.vt_rows = a->vt_rows, f.vt_cols = a->vt_cols, f.vt_ld = a->vt_ld, f.vt_user = a->vt_user;
      f.O = a->O, f.ldo = a->ldo;
      f.q = q, f.k = k, f.o = o;
      orx::launch_fmha_tc(f, st);
    } else {
      using B16 = __nv_bfloat16;
      orx::launch_attention<B16>(a->B, a->max_q, a->heads, a->dh, static_cast<const B16*>(a->Q) + a->q_col0, a->ldq,
                                 static_cast<const B16*>(a->K) + a->k_col0, a->ldk,
                                 static_cast<const B16*>(a->V) + a->v_col0, a->ldv, static_cast<B16*>(a->O), a->ldo,
                                 q, k, o, st);
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) throw orx::RuntimeError(std::string("CUDA: ") + cudaGetErrorString(err));
  });
}

int orx_debug_moe_route(int32_t rows, int32_t d, int32_t n_experts, int32_t k, const float* x, const float* gate,
                        const float* bias, int32_t variant, int32_t* sel_out, float* wts_out) {
  return guarded([&] {
    need(x, "x");
    need(gate, "gate");
    need(bias, "bias");
    need(sel_out, "sel_out");
    need(wts_out, "wts_out");
    if (rows < 0 || d <= 0 || n_experts < 1 || n_experts > 32 || k < 1 || k > n_experts || k > 8)
      throw orx::InvalidArgument("debug_moe_route: bad shape");
    orx::debug_moe_route(rows, d, n_experts, k, x, gate, bias, variant, sel_out, wts_out);
  });
}

int64_t orx_debug_topk_fallback_rows(void) {
  return static_cast<int64_t>(orx::topk_fallback_rows(true));
}

int orx_debug_ep_plan(int32_t world, int32_t rank, int32_t n_experts, const int32_t* counts, const int32_t* owner,
                      int32_t tile, int32_t max_tiles, int32_t slots, int32_t* cursor, int32_t* seg, int32_t* tiles,
                      int32_t* n_tiles, int64_t* rows_needed) {
  return guarded([&] {
    need(counts, "counts");
    need(owner, "owner");
    need(cursor, "cursor");
    need(seg, "seg");
    need(tiles, "tiles");
    need(n_tiles, "n_tiles");
    const int64_t r = orx::ep_plan_placed(world, rank, n_experts, counts, owner, tile, max_tiles, cursor, seg, slots,
                                          tiles, n_tiles);
    if (rows_needed) *rows_needed = r;
  });
}

int orx_compress_lifelong(int device, int32_t n_users, const orx_records* history, const double* content,
                          int32_t content_dim, int32_t threshold, int32_t max_out, int32_t n_code_layers,
                          const uint64_t* rng_seeds, orx_records_out* out) {
  return guarded([&] {
    need(history, "history");
    need(out, "out");
    if (n_users < 0) throw orx::InvalidArgument("negative user count");
    need(history->offsets, "history->offsets");
    need(out->offsets, "out->offsets");
    if (history->offsets[0] != 0) throw orx::InvalidArgument("offsets must start at 0");
    const int64_t n = history->offsets[n_users];
    if (n > 0) {
      need(content, "content");
      need(rng_seeds, "rng_seeds");
      need(history->vid, "history->vid");
      need(history->aid, "history->aid");
      need(history->tag, "history->tag");
      need(history->ts, "history->ts");
      need(history->playtime, "history->playtime");
      need(history->duration, "history->duration");
      need(history->labels, "history->labels");
    }
    orx::CompressHost h{};
    h.n_users = n_users, h.D = content_dim, h.threshold = threshold, h.max_out = max_out;
    h.n_code_layers = n_code_layers;
    h.offsets = history->offsets, h.vid = history->vid, h.aid = history->aid, h.labels = history->labels;
    h.tag = history->tag, h.ts = history->ts, h.playtime = history->playtime, h.duration = history->duration;
    h.sid = history->sid, h.content = content, h.rng_seeds = rng_seeds;
    h.out_offsets = out->offsets, h.out_vid = out->vid, h.out_aid = out->aid, h.out_labels = out->labels;
    h.out_tag = out->tag, h.out_ts = out->ts, h.out_playtime = out->playtime, h.out_duration = out->duration;
    h.out_sid = out->sid;
    orx::compress_lifelong_gpu(h, device);
  });
}

int orx_synth_batch_create(uint64_t seed, int64_t user_begin, int32_t n_users, int32_t n_short, int32_t n_positive,
                           int32_t n_lifelong, orx_synth_batch** out) {
  return guarded([&] {
    need(out, "out");
    if (n_users < 0 || n_short < 0 || n_positive < 0 || n_lifelong < 0)
      throw orx::InvalidArgument("synthetic batch sizes must be non-negative");
    auto b = std::make_unique<orx_synth_batch>();
    orx_synth::Lengths len{n_short, n_positive, n_lifelong};
    for (auto& p : b->p) p.offsets.push_back(0);
    for (int32_t i = 0; i < n_users; ++i) {
      orx_synth::synth_user<orx::Rng>(
          seed, static_cast<uint64_t>(user_begin + i), len,
          [&](int uid, int gender, int age) {
            b->uid.push_back(uid);
            b->gender.push_back(gender);
            b->age.push_back(age);
          },
          [&](int pathway, int64_t vid, int aid, double tag, double ts, double play, double dur, uint32_t labels) {
            auto& p = b->p[pathway];
            p.vid.push_back(vid);
            p.aid.push_back(aid);
            p.tag.push_back(tag);
            p.ts.push_back(ts);
            p.play.push_back(play);
            p.dur.push_back(dur);
            p.labels.push_back(labels);
          });
      for (auto& p : b->p) p.offsets.push_back(static_cast<int64_t>(p.vid.size()));
    }
    *out = b.release();
  });
}

int orx_synth_batch_view(const orx_synth_batch* b, orx_user_batch* v) {
  return guarded([&] {
    need(b, "batch");
    need(v, "view");
    v->n_users = static_cast<int32_t>(b->uid.size());
    v->uid = b->uid.data();
    v->gender = b->gender.data();
    v->age_bucket = b->age.data();
    orx_records* dst[3] = {&v->short_seq, &v->positive_seq, &v->lifelong_seq};
    for (int i = 0; i < 3; ++i) {
      const auto& p = b->p[i];
      dst[i]->offsets = p.offsets.data();
      dst[i]->vid = p.vid.data();
      dst[i]->aid = p.aid.data();
      dst[i]->tag = p.tag.data();
      dst[i]->ts = p.ts.data();
      dst[i]->playtime = p.play.data();
      dst[i]->duration = p.dur.data();
      dst[i]->labels = p.labels.data();
      dst[i]->sid = nullptr;
    }
  });
}

void orx_synth_batch_destroy(orx_synth_batch* b) { delete b; }

}  // extern "C"
