// Non-GEMM kernels of the hot path (host launchers). All launches go on the
// caller's stream and bump launch_counter().
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace orx {

struct RecordsDev {  // one pathway, all users, packed (device pointers)
  int n = 0;
  const int32_t* vid = nullptr;  // hashed vid row index (host-side, policy.cpp:14-17)
  const int32_t* aid = nullptr;  // hashed aid row index
  const float* tag = nullptr;
  const float* ts = nullptr;
  const float* play = nullptr;
  const float* dur = nullptr;
  const uint32_t* labels = nullptr;
  const int32_t* sid = nullptr;  // [n * n_code_layers] or null
};

struct FeatureTables {  // fp32 embedding tables (policy.cpp:139-198)
  const float* vid;       // [vid_vocab][d]
  const float* aid;       // [aid_vocab][aid_dim]
  const float* tag;       // [2][minor]
  const float* ts;
  const float* play;
  const float* dur;
  const float* label;     // [n_flags][minor]
  const float* tokens[8]; // sid history: per code layer [V][d]
  int d, aid_dim, minor, vid_vocab, aid_vocab, n_flags, n_code_layers, use_sid, vid_only;
  // bf16 copies of the vid / aid tables (bf16 engine): a single-row gather
  // rounded once gives the same bf16 output as the fp32 row
  const __nv_bfloat16* vid16 = nullptr;
  const __nv_bfloat16* aid16 = nullptr;
};

template <class T>
void launch_features(const RecordsDev& r, const FeatureTables& t, T* out, int ldo, cudaStream_t s);
// Pathway first layer folded through the feature tables (bf16 engine, no sid
// history): fc1(features(r)) = Pv[vid] + Pa[aid] + Pl[labels] + tag*u0 + ts*u1 +
// play*u2 + dur*u3, LeakyReLU'd (policy.cpp:175-216).
struct FoldTables {
  const float* pv = nullptr;  // [vid_vocab][d] = emb.vid . W1[0:d]
  const float* pa = nullptr;  // [aid_vocab][d] = emb.aid . W1[d:d+ad]
  const float* pl = nullptr;  // [2^n_flags][d]: label multi-hot . W1[lab] + scalar-section b rows + fc1 bias
  const float* u = nullptr;   // [4][d]: tag / ts / playtime / duration w rows through W1
  // optional [aid_vocab << n_flags][d] = pa[aid] + pl[labels]: one gather less per
  // record (the kernel is bound by L2 reads of these rows)
  const float* pal = nullptr;
  int d = 0, n_flags = 0;
};
// pal[(a << n_flags) | m][j] = pa[a][j] + pl[m][j]
void launch_fold_pal(int naid, int n_flags, int d, const float* pa, const float* pl, float* pal, cudaStream_t s);
bool fold_features_supported(int d, int n_flags);
void launch_fold_features(const RecordsDev& r, const FoldTables& f, __nv_bfloat16* out, int ldo, cudaStream_t s);
template <class T>
void launch_static_features(int U, const int32_t* uid, const int32_t* gender, const int32_t* age,
                            const float* uid_emb, const float* gender_emb, const float* age_emb, int sdim,
                            int uid_vocab, int gender_vocab, int age_vocab, T* out, int ldo, cudaStream_t s);
// z[u*T + t] = pos[t] + pad row at the left-padding rows of the short / positive
// pathways only (every other row is a GEMM output over the position table).
void launch_z_init(int U, int T, int d, const float* pos, const float* pad_short, const float* pad_pos,
                   const int32_t* n_short, const int32_t* n_pos, int Ls, int Lp, float* z, cudaStream_t s);
template <class T>
void launch_rmsnorm(int rows, int d, const float* x, int ldx, const float* gain, T* out, int ldo, cudaStream_t s);
template <class T>
void launch_convert(int rows, int cols, const float* x, int ldx, T* out, int ldo, cudaStream_t s);
// Copy rows (src_row = map ? map[r] : r) of a fp32 matrix, e.g. pad.lifelong keys.
template <class T>
void launch_fill_rows(int rows, int cols, const float* src_row, T* out, int ldo, const int32_t* row_idx,
                      cudaStream_t s);

// Decoder: h[r] = step == 0 ? bos : tokens[code[r]]
void launch_dec_embed(int rows, int d, const float* table, const int32_t* code, int code_stride, float* h,
                      cudaStream_t s);
// bf16: dec_embed and the first decoder layer's RMSNorm (gain) into out in one
// pass; false if the shape is unsupported (then launch_dec_embed + rmsnorm)
bool launch_dec_embed_norm(int rows, int d, const float* table, const int32_t* code, int code_stride, float* h,
                           const float* gain, __nv_bfloat16* out, cudaStream_t s);
// Decoder causal self-attention over cached positions (policy.cpp:282-283).
// qkv: [rows][3d] this position's QKV output; kv[p * n_layers + layer]: position p's
// QKV output [rows_p][3d] (its K|V columns are the cache, nothing is copied);
// anc: [rows][anc_stride] row index of position p < step.
template <class T>
void launch_dec_self_attn(int rows, int d, int heads, int step, int layer, int n_layers, const T* qkv,
                          T* const* kv, const int32_t* anc, int anc_stride, T* out, cudaStream_t s);

// MoE (nn.cpp:117-172)
// Routing reads the fp32 residual x and the pre-MoE RMSNorm gain (norm recomputed in fp32).
// gate_gain [E][d] = gain[c] * W_g[c][e] selects the fast path (d % 4 == 0);
// gate_sw (E <= 24, d % 128 == 0) is the same in moe_route4's swizzled layout.
void launch_moe_route(int rows, int d, int E, int k, const float* x, int ldx, const float* gain, const float* gate_t,
                      const float* gate_gain, const float* bias, int32_t* sel, float* wts, int32_t* counts,
                      cudaStream_t s, const float* gate_sw = nullptr);
// bf16 engine: the MoE combine fused with the next op's input (RMSNorm with
// `gain`, or a plain bf16 copy when gain is null); false if the shape is not
// supported (then run launch_moe_combine + the norm / convert).
template <class YT>
// zero / nzero (<= 256): counters zeroed by the combine for the next MoE layer
bool launch_moe_combine_norm(int rows, int k, int d, const YT* yg, const int32_t* slot, float* h, int ldh,
                             const float* gain, __nv_bfloat16* out, int ldo, cudaStream_t s, int32_t* zero = nullptr,
                             int nzero = 0);
// K|V of the empty-history pad key rows when the lifelong fc2 is folded into the
// QFormer K|V weights (engine build_kv_fold): kv = pad . Wkv [2 nkv] (K then V).
template <class T>
void launch_fill_kv_pad(int n_pad, const int32_t* rows, const int32_t* row_user, const int32_t* row_pos,
                        const float* kv, int nkv, T* kvl, int ldk, T* vt, int vt_ld, long long vt_user_stride,
                        long long vt_layer_stride, int d, cudaStream_t s);
// Gate scores on the tensor pipe (3xTF32, route_tc.cu) for the bf16 engine:
// gate_hi / gate_lo [32][d] = the gain-folded gate split into tf32 hi and
// residual lo (expert rows >= E zero). Same outputs as launch_moe_route.
bool moe_route_tc_supported(int d, int E, int k, int ldx);
// host-side gate layouts (pack_moe and orx_debug_moe_route): gate [E][d] ->
// moe_route4's swizzled [d / 4][96] (E <= 24, d % 128 == 0), and the tf32
// hi / residual lo split padded to 32 expert rows [32][d]
void gate_route4_layout(const float* gate, int E, int d, float* sw);
void gate_tf32_split(const float* gate, int E, int d, float* hi, float* lo);
// Debug / test entry (orx_debug_moe_route): host x [rows][d], gate [E][d]
// (gain folded), bias [E] -> host sel / wts [rows][k] through one router:
// variant 0 = moe_route2 (SIMT), 1 = moe_route4 (SIMT, swizzled gate),
// 2 = moe_route_tc (3xTF32 tensor pipe).
void debug_moe_route(int rows, int d, int E, int k, const float* x, const float* gate, const float* bias,
                     int variant, int32_t* sel, float* wts);
// part: moe_route_tc_scratch_floats(max rows) floats; ticket: one int per 128-row
// tile, zero before the first call (the kernel leaves it zero)
size_t moe_route_tc_scratch_floats(int max_rows);
void launch_moe_route_tc(int rows, int d, int E, int k, const float* x, int ldx, const float* gate_hi,
                         const float* gate_lo, const float* bias, int32_t* sel, float* wts, int32_t* counts,
                         float* part, int32_t* ticket, cudaStream_t s);
// The grouped-GEMM plan, computed by the scatter itself from the final routing
// histogram: expert segments padded to tile_rows, tile_expert / n_mtiles for
// the grouped GEMMs; fill [E] must be zero (it is zeroed with counts).
struct MoePlan {
  const int32_t* counts = nullptr;
  int32_t* fill = nullptr;
  int32_t* tile_expert = nullptr;
  int32_t* n_mtiles = nullptr;
  int max_tiles = 0, tile_rows = 0, E = 0;
  // optional folded pre-MoE RMSNorm: the token rows are un-normalised; every
  // grouped row gets rsqrt(sum_i ssq[i][token] / d + 1e-6) in row_rsq
  const float* ssq = nullptr;
  long long ssq_ld = 0;
  int ssq_n = 0;
  float inv_d = 0.f;
  float* row_rsq = nullptr;
};
template <class T>
void launch_moe_scatter(int rows, int k, int d, const T* x, int ldx, const int32_t* sel, const float* wts,
                        const MoePlan& plan, int32_t* slot, T* xg, float* row_scale, cudaStream_t s);
// yg: fp32 (fp32 engine) or bf16 (bf16 engine) weighted expert outputs
template <class YT>
void launch_moe_combine(int rows, int k, int d, const YT* yg, const int32_t* slot, float* h, int ldh,
                        cudaStream_t s, int32_t* zero = nullptr, int nzero = 0);

// ---- expert-parallel exchange over NVLink peer memory (graph-capturable) ----
// Every rank maps every peer's symmetric exchange region (CUDA IPC); the
// dispatch / return are device-side stores into the peers' buffers at offsets
// computed on the device from the all-gathered routing histograms, ordered by
// per-(phase, source) monotonic arrival counters. No host synchronisation.
constexpr int kEpMaxWorld = 8;
struct EpPeers {
  void* xr[kEpMaxWorld];       // [recv_cap][d] T: expert-grouped received rows (256-row padded segments)
  float* wr[kEpMaxWorld];      // [recv_cap] gate weight of each received row
  int32_t* src[kEpMaxWorld];   // [recv_cap] (source rank << 24) | source (token, slot) index
  void* yr[kEpMaxWorld];       // [send_cap][d] T: weighted expert outputs returned to the token's rank
  int32_t* cnt[kEpMaxWorld];   // [W][E] routing histograms of every rank
  uint32_t* flag[kEpMaxWorld];  // [3 phases][W sources] arrival counters
  uint32_t* epoch = nullptr;   // local [3] exchanges completed per phase
  int32_t* err = nullptr;      // local: 1 = wait timeout, 2 = receive capacity overflow
  int me = 0, world = 1;
  int recv_cap = 0;
};
enum EpPhase { EP_COUNTS = 0, EP_DISPATCH = 1, EP_RETURN = 2 };
// counts[E] -> every rank's cnt[me][:], then signal EP_COUNTS
void launch_ep_counts(int E, const int32_t* counts, const EpPeers& P, cudaStream_t s);
// wait until every rank signalled `phase` for the current exchange
void launch_ep_wait(const EpPeers& P, int phase, cudaStream_t s);
void launch_ep_signal(const EpPeers& P, int phase, cudaStream_t s);
// From the local copy of every rank's histogram: cursor[e] = where this rank's
// rows for global expert e start in the owner's grouped buffer; this rank's
// grouped-GEMM tile table, n_mtiles and segment (start, count) per local expert.
// owner / slot [E], list [W][C]: the MoE layer's placement tables (ep_plan.hpp);
// load [E] (optional) accumulates the layer's global rows per expert
void launch_ep_plan(int E, const EpPeers& P, int tile, int max_tiles, int32_t* cursor, int32_t* tile_expert,
                    int32_t* n_mtiles, int32_t* seg, const int32_t* owner, const int32_t* slot, const int32_t* list,
                    int C, long long* load, cudaStream_t s);
// (token, slot) rows -> the experts' ranks' grouped buffers (+ gate weight, source id); slot[i] = i
template <class T>
void launch_ep_dispatch(int rows, int k, int d, const T* x, int ldx, const int32_t* sel, const float* wts,
                        int32_t* cursor, int32_t* slot, const int32_t* owner, const EpPeers& P, cudaStream_t s);
// this rank's received rows' outputs (yg, grouped order) -> the tokens' ranks' yr[slot]
template <class T>
void launch_ep_return(int El, int d, const int32_t* seg, const T* yg, const EpPeers& P, cudaStream_t s);
void launch_swiglu_mul(long long n, const float* a, const float* b, float* out, cudaStream_t s);

}  // namespace orx
