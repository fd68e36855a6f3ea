/*
 * orx.h — C-ABI of the B200-native OneRec inference hot path.
 *
 * Drop-in boundary for the reference's encode / generate entry points
 * (reference: /root/reference/proj/core). Plain pointers and sizes only;
 * every function returns ORX_OK (0) or a negative error code, with the
 * message available from orx_last_error() (thread-local). No exceptions
 * cross the ABI. One engine per GPU; an engine is not thread-safe.
 *
 * Reference interface each entry point replaces:
 *   orx_config / orx_config_preset ........ PolicyConfig, policy.hpp:36-85
 *   orx_weights_create_random ............. PolicyModel::PolicyModel(cfg), policy.cpp:59-137
 *   orx_weights_load_grcp / save_grcp ..... PolicyModel::load / save, policy.cpp:411-443
 *   orx_user_batch ........................ UserContext / InteractionFeature, policy.hpp:15-32
 *   orx_validate_batch .................... validate_context, policy.cpp:23-38
 *   orx_encode ............................ PolicyModel::encode_eval, policy.cpp:317-321
 *   orx_next_logits ....................... PolicyModel::next_logits_eval, policy.cpp:323-329
 *   orx_score_prefixes .................... encode_eval + next_logits_eval per (user, prefix)
 *   orx_beam_search ....................... generate(req{beam}) = beam_search(req, policy_scorer(m, z), ...),
 *                                           generation.cpp:41-88,150-167, batched over users
 */
#ifndef ORX_H_
#define ORX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORX_OK 0
#define ORX_EINVAL -1  /* std::invalid_argument in the reference (GENREC_REQUIRE) */
#define ORX_ERUNTIME -2 /* std::runtime_error in the reference (I/O, non-finite)   */
#define ORX_ECUDA -3    /* CUDA error or missing device                           */

#define ORX_PRECISION_FP32 0 /* parity mode: fp32 SIMT GEMMs, fp32 activations   */
#define ORX_PRECISION_BF16 1 /* throughput mode: tcgen05 bf16 GEMMs, fp32 accum  */

/* Mirror of genrec::PolicyConfig (policy.hpp:36-85), same field meanings. */
typedef struct orx_config {
  int32_t n_layers;
  int32_t d_model;
  int32_t ffn_hidden;
  int32_t n_heads;
  int32_t moe_enabled;
  int32_t n_experts;
  int32_t experts_active;
  int32_t moe_location; /* 0 = decoder, 1 = enc_and_dec */
  int32_t expert_round_multiple;
  int32_t n_code_layers;
  int32_t codebook_size;
  int32_t short_len;
  int32_t positive_len;
  int32_t lifelong_len;
  int32_t n_queries;
  int32_t lifelong_blocks;
  int32_t vid_vocab;
  int32_t aid_vocab;
  int32_t uid_vocab;
  int32_t gender_vocab;
  int32_t age_vocab;
  int32_t n_label_flags;
  int32_t use_sid_history;
  int32_t vid_only_features;
  int32_t compress_threshold;
  double moe_bias_update;
  uint64_t seed;
} orx_config;

/* One pathway's records for all users, concatenated user after user
 * (each user's records time-ascending). offsets has n_users+1 entries. */
typedef struct orx_records {
  const int64_t* offsets;
  const int64_t* vid;
  const int32_t* aid;
  const double* tag;
  const double* ts;
  const double* playtime;
  const double* duration;
  const uint32_t* labels;
  const int32_t* sid; /* [n_records * n_code_layers]; required iff use_sid_history */
} orx_records;

typedef struct orx_user_batch {
  int32_t n_users;
  const int32_t* uid;
  const int32_t* gender;
  const int32_t* age_bucket;
  orx_records short_seq;
  orx_records positive_seq;
  orx_records lifelong_seq;
} orx_user_batch;

/* Beam-search results: per user `width` items sorted by (log_prob desc,
 * codes asc); n_items[u] < width only when fewer candidates exist. */
typedef struct orx_beam_out {
  int32_t* codes;    /* [n_users * width * n_code_layers] */
  double* log_prob;  /* [n_users * width] */
  int32_t* n_items;  /* [n_users] */
} orx_beam_out;

typedef struct orx_weights orx_weights;
typedef struct orx_engine orx_engine;
typedef struct orx_synth_batch orx_synth_batch;

const char* orx_last_error(void);
const char* orx_version(void);

/* Config: reference defaults (PolicyConfig{}) or a named paper preset:
 * "tiny", "0.015B", "0.121B", "0.935B", "2.633B". */
int orx_config_default(orx_config* cfg);
int orx_config_preset(const char* name, orx_config* cfg);
int64_t orx_config_enc_seq_len(const orx_config* cfg);
int64_t orx_config_expert_hidden(const orx_config* cfg);

/* Host weights (fp32 copies of the reference's f64 parameters). */
int orx_weights_create_random(const orx_config* cfg, orx_weights** out);
/* Same stream, but only the experts of expert-parallel rank ep_rank of
 * ep_world are materialised (for orx_engine_create_ep; cannot be saved). */
int orx_weights_create_random_ep(const orx_config* cfg, int32_t ep_rank, int32_t ep_world, orx_weights** out);
int orx_weights_load_grcp(const char* path, orx_weights** out);
int orx_weights_save_grcp(const orx_weights* w, const char* path);
int orx_weights_config(const orx_weights* w, orx_config* cfg);
int64_t orx_weights_count(const orx_weights* w);
/* Name / shape / data of entry i in reference insertion order. */
int orx_weights_entry(const orx_weights* w, int64_t i, const char** name, int32_t* ndim, int32_t dims[2],
                      const float** data);
int orx_weights_find(const orx_weights* w, const char* name, int64_t* index);
/* Overwrite the n = rows * cols values of a named parameter (e.g. from the
 * caller's own f64 ParamStore, converted; ORX_EINVAL on an unknown name or a
 * size mismatch). Engines created afterwards see the new values. */
int orx_weights_set(orx_weights* w, const char* name, const float* data, int64_t n);
void orx_weights_destroy(orx_weights* w);

int orx_validate_batch(const orx_config* cfg, const orx_user_batch* batch);

/* Engine on one GPU. max_users / max_width size the device arena. */
int orx_engine_create(const orx_weights* w, int device, int precision, int32_t max_users, int32_t max_width,
                      orx_engine** out);
void orx_engine_destroy(orx_engine* e);

/* Expert parallelism over NVLink peer memory, SURVEY.md §8(e) / BASELINE
 * config 4: ep_world engines (one process per GPU) each compute n_experts /
 * ep_world experts of every MoE layer; MoE layers exchange (token, expert)
 * rows by device-side stores into the peers' buffers (CUDA IPC regions, set
 * up once over an NCCL communicator). Rank 0 creates a fresh id per engine
 * (orx_ep_unique_id; an id bootstraps one communicator only) and every rank
 * receives it out of band (e.g. torch.distributed broadcast). All ranks must
 * then call the same sequence of orx_encode / orx_beam_search /
 * orx_score_prefixes / orx_next_logits (each with its own users; widths
 * equal). Results are bitwise identical to a replica engine's. */
#define ORX_EP_ID_BYTES 128
int orx_ep_unique_id(uint8_t id_out[ORX_EP_ID_BYTES]);
int orx_engine_create_ep(const orx_weights* w, int device, int precision, int32_t max_users, int32_t max_width,
                         const uint8_t id[ORX_EP_ID_BYTES], int32_t ep_rank, int32_t ep_world, orx_engine** out);
/* Expert placement (load balancing): owner [moe_layers * n_experts] gives,
 * per MoE layer (encoder layers first when they are MoE, then decoder
 * layers; orx_config_moe_layers), the rank that computes each expert, or -1
 * = replicated on every rank (computed where the token lives, never sent).
 * Every rank must pass the same table (checked at creation); the weights must
 * hold the experts the rank computes (orx_weights_create_random_ep_placed, or
 * full weights). NULL = contiguous blocks (orx_engine_create_ep). */
int32_t orx_config_moe_layers(const orx_config* cfg);
int orx_engine_create_ep_placed(const orx_weights* w, int device, int precision, int32_t max_users,
                                int32_t max_width, const uint8_t id[ORX_EP_ID_BYTES], int32_t ep_rank,
                                int32_t ep_world, const int32_t* owner, orx_engine** out);
int orx_weights_create_random_ep_placed(const orx_config* cfg, int32_t ep_rank, int32_t ep_world,
                                        const int32_t* owner, orx_weights** out);
/* Rows routed to each expert of each MoE layer, summed over every rank and
 * every MoE call since creation / the last reset: load_out [moe_layers *
 * n_experts]; identical on every expert-parallel rank (zeros otherwise). */
int orx_engine_expert_load(orx_engine* e, int64_t* load_out, int32_t reset);
/* Load-balanced placement from such loads (csrc/ep_plan.hpp
 * ep_place_balanced): per layer the fewest heaviest experts (between
 * min_replicas and max_replicas) are replicated such that the rest, packed
 * heaviest-first onto the least-loaded rank and refined by moves / swaps, leave
 * the busiest rank within 5% of the mean (else the best found); replicated
 * experts' rows stay on their token's rank, so min_replicas > 0 trades expert
 * memory for NVLink traffic. predicted_imbalance [moe_layers] (optional) =
 * busiest / mean rank load under that placement. Deterministic. */
int orx_ep_place(const int64_t* load, int32_t layers, int32_t n_experts, int32_t world, int32_t min_replicas,
                 int32_t max_replicas, int32_t* owner_out, double* predicted_imbalance);

/* z_out (host, optional): [n_users * enc_seq_len * d_model] fp32. */
int orx_encode(orx_engine* e, const orx_user_batch* batch, float* z_out);
/* Teacher-forced logits for n queries over caller-supplied encodings:
 * z_enc [n_z * T * d] fp32, query q uses z_index[q] and prefix
 * prefixes[q * n_code_layers ...] of length prefix_len[q] (< n_code_layers).
 * logits_out: [n * codebook_size] fp32. */
int orx_next_logits(orx_engine* e, const float* z_enc, int32_t n_z, int32_t n, const int32_t* z_index,
                    const int32_t* prefixes, const int32_t* prefix_len, float* logits_out);
/* encode + teacher-forced logits for (user, prefix) queries of a batch. */
int orx_score_prefixes(orx_engine* e, const orx_user_batch* batch, int32_t n, const int32_t* user,
                       const int32_t* prefixes, const int32_t* prefix_len, float* logits_out);
/* encode + unconstrained beam search of depth n_code_layers, batched. */
int orx_beam_search(orx_engine* e, const orx_user_batch* batch, int32_t width, orx_beam_out* out);

/* Pipelined serving form of orx_beam_search (same results): submit stages the
 * batch (host packing + H2D on a copy stream) and launches its search without
 * waiting; collect blocks for the OLDEST submitted request and writes its
 * beams into `out` (layout of orx_beam_search). At most two requests are in
 * flight (one per staging slot), so request i+1's host packing and H2D overlap
 * request i's device work. A third submit before a collect fails (EINVAL). */
int orx_beam_search_submit(orx_engine* e, const orx_user_batch* batch, int32_t width);
int orx_beam_search_collect(orx_engine* e, orx_beam_out* out);

/* Semantic-ID trie (SemanticTrie, trie.hpp:27-62) as CSR over prefix nodes:
 * node 0 is the root, node n's children are entries [child_off[n],
 * child_off[n+1]) of child_code (strictly ascending) / child_node. Uploaded
 * to the device for orx_beam_search_constrained (generation.cpp:58-64). */
typedef struct orx_trie {
  int32_t n_nodes;
  const int32_t* child_off; /* [n_nodes + 1] */
  int64_t n_edges;
  const int32_t* child_code; /* [n_edges] */
  const int32_t* child_node; /* [n_edges] */
} orx_trie;
int orx_engine_set_trie(orx_engine* e, const orx_trie* trie);
/* Beam search expanding only trie children (GenerationRequest::constrain_to_trie);
 * n_items[u] < width when the trie offers fewer candidates. */
int orx_beam_search_constrained(orx_engine* e, const orx_user_batch* batch, int32_t width, orx_beam_out* out);
/* PolicyModel::sequence_log_prob (policy.cpp:297-310): log-prob (f64) of the
 * full semantic id codes[q * n_code_layers ...] for user user[q] of the batch. */
int orx_sequence_log_prob(orx_engine* e, const orx_user_batch* batch, int32_t n, const int32_t* user,
                          const int32_t* codes, double* log_prob_out);

/* sample_topk_topp (generation.cpp:90-148): `width` independent samples per
 * user (tempered by temperature, cut to top_k (0 = all) and top_p), user u
 * drawing uniforms from Rng(seed).split(user_stream[u]) (NULL: u) exactly as
 * the reference's Rng; log_prob is the untempered model log-prob (f64). */
int orx_sample(orx_engine* e, const orx_user_batch* batch, int32_t width, double temperature, int32_t top_k,
               double top_p, uint64_t seed, const uint64_t* user_stream, orx_beam_out* out);

/* Same as orx_beam_search, but inputs are already resident on the device
 * (uploaded by orx_engine_stage_batch); results stay on the device unless
 * out is non-NULL. Used to time the kernel path without host copies. */
int orx_engine_stage_batch(orx_engine* e, const orx_user_batch* batch);
int orx_beam_search_staged(orx_engine* e, int32_t width, orx_beam_out* out);
/* Counters: kernel launches issued by the engine so far, bytes H2D / D2H. */
int orx_engine_stats(const orx_engine* e, int64_t* launches, int64_t* h2d_bytes, int64_t* d2h_bytes);
/* Stream the engine launches on (cudaStream_t as void*). */
void* orx_engine_stream(orx_engine* e);
/* Per-kernel-class CUDA-event timing (process-wide; off by default).
 * Classes: 0 dense GEMM, 1 MoE grouped GEMM, 2 encoder / QFormer attention,
 * 3 decoder self-attention, 4 MoE routing/scatter/combine, 5 beam selection,
 * 6 other, 7 decoder cross attention over the K/V cache, 8 record features,
 * 9 RMSNorm. flops / bytes are algorithmic (bytes: HBM traffic the kernel must
 * do, for the HBM-bound classes). orx_profile_read fills n (<= 10) entries and
 * resets the log. */
#define ORX_PROF_CLASSES 10
int orx_profile_enable(int on);
int orx_profile_read(int32_t n, int64_t* launches, double* ms, double* flops, double* bytes);

/* Kernel-level test hook: one GEMM C = A . B^T with the engine's fused
 * epilogue, on DEVICE pointers (e.g. torch tensors' data_ptr), on the given
 * stream (cudaStream_t as void*, NULL = default). Used by the kernel tests
 * against a PyTorch fp32 reference; not part of the reference surface. */
typedef struct orx_gemm_args {
  const void* A; int32_t lda;        /* [M][K] bf16 (or fp32 if precision == FP32) */
  const void* B; int32_t ldb;        /* [N][K] (grouped: [n_groups * b_rows_per_expert][K]) */
  int32_t M, N, K;
  int32_t precision;                 /* ORX_PRECISION_BF16 (tcgen05) or ORX_PRECISION_FP32 (SIMT) */
  const float* bias;                 /* [N] or NULL */
  const float* row_scale;            /* [M] or NULL */
  const float* resid; int32_t ld_resid; /* fp32, indexed by output row, or NULL */
  const int32_t* row_map;            /* output row of A row r (< 0 dropped), or NULL */
  void* out; int32_t ldo; int32_t out_bf16;
  int32_t act;                       /* 0 none, 1 LeakyReLU(0.01), 2 SiLU */
  int32_t swiglu;                    /* B rows interleaved per 128 as [W1 | W3]; out = silu(a)*b, N/2 cols */
  int32_t n_out, m_valid, col_off;
  const int32_t* tile_expert;        /* grouped: expert per tile_rows-row M tile (-1 skip), or NULL */
  const int32_t* n_mtiles;           /* grouped: device scalar */
  int32_t b_rows_per_expert, n_groups, tile_rows;
  int32_t force_single_cta;          /* 1: use the 1-CTA tcgen05 kernel even for M > 128 */
} orx_gemm_args;
int orx_debug_gemm(const orx_gemm_args* args, void* stream);
/* Kernel-level test hook for the per-row beam pruning step (device pointers):
 * lse[r] = logsumexp(logits[r]); cand[r][0..k) = the k largest keys
 * (ordered fp32 score pscore[r] + logits[r][i] - lse[r]) << 32 |
 * (0xFFFFFFFF - (plex[r] * V + i)), in unspecified order. */
int orx_debug_row_topk(int32_t rows, int32_t V, int32_t k, const float* logits, const float* pscore,
                       const int32_t* plex, float* lse, uint64_t* cand, void* stream);
/* Kernel-level test hook for segmented bf16 attention (device pointers):
 * segment b's query rows [qs(b), +ql(b)) attend to key rows [ks(b), +kl(b)),
 * output rows start at os(b); a NULL array means start = b * stride /
 * len = fixed. kernel 0: mma.sync kernel (row-major V); kernel 1: tcgen05
 * kernel (V transposed per (vt_user[b] or b, head): Vt rows (u*heads+h)*dh+c,
 * columns = key position in the segment). Q/K/V are buffer bases with head 0
 * at column q_col0 / k_col0 / v_col0. */
typedef struct orx_attn_args {
  int32_t B, max_q, heads, dh;
  const void* Q; int64_t q_rows; int32_t ldq, q_col0;
  const void* K; int64_t k_rows; int32_t ldk, k_col0;
  const void* V; int32_t ldv, v_col0;
  const void* Vt; int64_t vt_rows, vt_cols; int32_t vt_ld; const int32_t* vt_user;
  void* O; int32_t ldo;
  const int32_t *q_start, *q_len, *k_start, *k_len, *o_start;
  int32_t q_stride, q_fixed, k_stride, k_fixed, o_stride;
  int32_t kernel;
} orx_attn_args;
int orx_debug_attention(const orx_attn_args* args, void* stream);
/* MoE gate routing through one router kernel, for the GPU tests (host
 * buffers): x [rows * d] (the fp32 residual rows), gate [n_experts * d] (the
 * pre-MoE RMSNorm gain folded in), bias [n_experts]; variant 0 = SIMT
 * moe_route2, 1 = SIMT moe_route4 (swizzled gate), 2 = 3xTF32 tensor-pipe
 * moe_route_tc. Outputs sel / wts [rows * k]: selected experts ascending and
 * their softmax weights (moe_forward, nn.cpp:117-147). */
int orx_debug_moe_route(int32_t rows, int32_t d, int32_t n_experts, int32_t k, const float* x, const float* gate,
                        const float* bias, int32_t variant, int32_t* sel_out, float* wts_out);
/* Rows of the beam-pruning fast path that took its exact radix-select
 * fallback since the last call (process-wide counter, reset on read). */
int64_t orx_debug_topk_fallback_rows(void);

/* Host restatement of the device plan of one expert-parallel exchange
 * (csrc/ep_plan.hpp ep_plan_placed), for the CPU tests: counts [world *
 * n_experts] (all-gathered histograms), owner [n_experts] (one layer's
 * placement), slots = local expert slots per rank. Outputs for `rank`:
 * cursor [n_experts] (first row of its expert-e rows in the computing rank's
 * buffer), seg [2 * slots] (start, rows of each local slot), tiles
 * [max_tiles] (local slot per grouped-GEMM tile, -1 past the end), n_tiles,
 * rows_needed (its buffer rows, padded). */
int orx_debug_ep_plan(int32_t world, int32_t rank, int32_t n_experts, const int32_t* counts, const int32_t* owner,
                      int32_t tile, int32_t max_tiles, int32_t slots, int32_t* cursor, int32_t* seg, int32_t* tiles,
                      int32_t* n_tiles, int64_t* rows_needed);

/* Lifelong-history compression on the GPU (the step before the encoder;
 * compress_lifelong, policy.cpp:447-510, over hierarchical K-means,
 * kmeans.cpp:22-183): per user u, records [offsets[u], offsets[u+1]) of
 * `history` with content rows content[i * content_dim ...] (f64) are
 * clustered (threshold records per leaf) with the reference Rng seeded by
 * rng_seeds[u] (build_user_context uses cfg.seed ^ (0x9e3779b97f4a7c15 *
 * (user + 1))), and replaced by their leaf's representative (categorical
 * fields) with leaf-mean tag / playtime / duration and their own ts; the last
 * min(n_u, max_out) records are written to `out` (out->offsets [n_users+1]). */
typedef struct orx_records_out {
  int64_t* offsets;
  int64_t* vid;
  int32_t* aid;
  double* tag;
  double* ts;
  double* playtime;
  double* duration;
  uint32_t* labels;
  int32_t* sid; /* [n * n_code_layers] or NULL */
} orx_records_out;
int orx_compress_lifelong(int device, int32_t n_users, const orx_records* history, const double* content,
                          int32_t content_dim, int32_t threshold, int32_t max_out, int32_t n_code_layers,
                          const uint64_t* rng_seeds, orx_records_out* out);

/* Seeded synthetic users (synth_users.hpp). */
int orx_synth_batch_create(uint64_t seed, int64_t user_begin, int32_t n_users, int32_t n_short, int32_t n_positive,
                           int32_t n_lifelong, orx_synth_batch** out);
int orx_synth_batch_view(const orx_synth_batch* b, orx_user_batch* view);
void orx_synth_batch_destroy(orx_synth_batch* b);

#ifdef __cplusplus
}
#endif

#endif /* ORX_H_ */
