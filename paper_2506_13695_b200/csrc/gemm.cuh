// GEMM interface shared by the tcgen05 (bf16) and SIMT (fp32 parity) kernels.
//
// C[M, N] = A[M, K] . B[N, K]^T, i.e. y = x . W with the reference's (in, out)
// Linear weight W (nn.cpp:8-22) stored transposed as B = W^T [out][in]
// ("K-major" for both operands, the native UMMA layout). Every linear of the
// hot path goes through here with a fused epilogue:
//   bias add (linear, nn.cpp:18-22), LeakyReLU / SiLU (mlp_leaky / ffn,
//   nn.cpp:32-34,71-73), SwiGLU pairing (swiglu, nn.cpp:84-86), MoE combine
//   weight (nn.cpp:167-168), residual add (policy.cpp:261-262,283-285).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace orx {

enum Act { ACT_NONE = 0, ACT_LEAKY = 1, ACT_SILU = 2 };
// Epilogue mode bits (Epi::mode, set by the launcher): specialised code paths.
enum EpiMode {
  EPI_BIAS = 1, EPI_LEAKY = 2, EPI_SILU = 4, EPI_RS = 8, EPI_RESID = 16, EPI_BF16 = 32,
  EPI_SWIGLU = 64,  // silu(a) * b over the interleaved W1|W3 accumulator (bf16 out, nothing else)
  EPI_SPLITVT = 128,  // bf16 out below Epi::vt_col0, transposed V store from it on (nothing else)
  EPI_STATS = 256,    // fp32 out + per-(row, 32-column chunk) log-sum-exp statistics (the head GEMM)
  EPI_XSSQ = 512,     // residual producers: also a bf16 copy of the output and per-row sum-of-squares partials
  EPI_RSQ = 1024,     // consumers: accumulator pre-scaled by rsqrt(mean(x^2) + eps) from those partials
  EPI_PEER = 2048,    // rows scattered to peer memory: row r -> peer_out[code >> 24] + (code & 0xFFFFFF) * ldo
  EPI_RMOD = 4096     // residual row = output row % resid_mod (a per-position residual table)
};
constexpr int kEpiMaxPeers = 8;

struct Epi {
  const float* bias = nullptr;       // [N] (or [N/2] for swiglu: not used)
  const float* row_scale = nullptr;  // [M] per-row multiplier
  // SwiGLU only (the grouped W1|W3 GEMM): per-row pre-scale of both halves,
  // rsqrt(mean(x^2) + eps) of the un-normalised token row (folded pre-MoE RMSNorm)
  const float* row_rsq = nullptr;
  const float* resid = nullptr;      // fp32 [rows, ld_resid], indexed by output row
  void* out = nullptr;               // [rows, ldo]
  const int* row_map = nullptr;      // output row = row_map[r] (< 0: dropped)
  int ld_resid = 0;
  int resid_mod = 0;  // > 0: the residual row of output row r is r % resid_mod (a per-position table)
  int ldo = 0;
  int out_bf16 = 0;
  int act = 0;      // Act
  int swiglu = 0;   // B rows interleaved per 128: [W1 block | W3 block] -> silu(a)*b
  int n_out = 0;    // number of valid output columns
  int m_valid = 0;  // rows >= m_valid are not stored
  int col_off = 0;  // added to output column index
  // Transposed store (bf16 only; the attention V operand, K-major for P.V):
  // element (row r, col n) goes to vt[u * vt_user_stride + t + (n % vt_cols) * vt_ld
  //                                  + (n / vt_cols) * vt_layer_stride]
  // with (u, t) = (vt_row_user[r], vt_row_pos[r]) or (r / vt_T, r % vt_T).
  void* vt = nullptr;
  int vt_ld = 0, vt_T = 0, vt_cols = 0;
  long long vt_user_stride = 0, vt_layer_stride = 0;
  const int32_t* vt_row_user = nullptr;
  const int32_t* vt_row_pos = nullptr;
  // columns >= vt_col0 take the transposed store (as column n - vt_col0);
  // columns below it are regular bf16 stores to out / ldo (one GEMM for K|V)
  int vt_col0 = 0;
  // Head GEMM statistics (EPI_STATS, plain fp32 out only): for every output
  // row r and 32-column chunk c, stats[c * stats_ld + r] = (max, sum exp(x - max))
  // over columns [32c, 32c + 32) -- the inputs of the fused log-softmax +
  // beam selection (beam_select, beam.cuh). Chunk-major so a warp's 32 rows
  // store 256 contiguous bytes.
  float2* stats = nullptr;
  long long stats_ld = 0;
  // RMSNorm folded into the GEMMs either side of it (bf16 engine): the GEMM
  // that writes the fp32 residual row also writes bf16(row) to out2 and, per
  // row and 128-column half tile, the partial sum of squares ssq[slot][row]
  // (slot = 2 * n_tile + half). The next GEMM reads out2 as its A operand (the
  // RMSNorm gain is folded into its weights) and scales each accumulator row
  // by rsqrt(sum_{i < rsq_n} rsq[i][row] / d + 1e-6) before anything else.
  void* out2 = nullptr;
  int ldo2 = 0;
  float* ssq = nullptr;
  long long ssq_ld = 0;
  const float* rsq = nullptr;
  long long rsq_ld = 0;
  int rsq_n = 0;
  float rsq_inv_d = 0.f;
  // Expert-parallel return fused into the grouped W2 GEMM (EPI_PEER, bf16 out):
  // output row r goes to peer_out[code >> 24] + (code & 0xFFFFFF) * ldo with
  // code = peer_code[r] (< 0: padding row, not stored) -- the token's rank's
  // return buffer, mapped into this process over NVLink.
  const int32_t* peer_code = nullptr;
  void* peer_out[kEpiMaxPeers] = {};
  int mode = -1;  // EpiMode bits of a specialised path, -1 = generic (set by gemm_bf16)
};

// Grouped (MoE) addressing: M tile i uses B rows [tile_expert[i]*b_rows_per_expert, ...).
struct Grouped {
  const int* tile_expert = nullptr;  // [max m tiles], -1 = skip
  const int* n_mtiles = nullptr;     // device scalar: number of valid M tiles
  int b_rows_per_expert = 0;
  int n_groups = 0;  // number of experts stacked in B
  int tile_rows = 128;  // rows per tile_expert entry (expert segments padded to it); 256 = CTA-pair kernel
  long long algo_rows = 0;  // real (token, expert) rows, for FLOP accounting
};

// bf16 A [M x K] (row stride lda elements), bf16 B [N x K] (row stride ldb).
// K must be a multiple of 8 (16-byte TMA strides); rows beyond M/N and the K
// tail are zero-filled by TMA.
void gemm_bf16(const void* A, int lda, const void* B, int ldb, int M, int N, int K, const Epi& epi,
               const Grouped* grp, cudaStream_t stream);

// fp32 A [M x K], fp32 B [N x K]; same epilogue. Parity mode only.
void gemm_f32(const float* A, int lda, const float* B, int ldb, int M, int N, int K, const Epi& epi,
              const Grouped* grp, cudaStream_t stream);

int num_sms();
// ORX_GEMM_SINGLE_CTA=1 disables the CTA-pair kernel for dense GEMMs (A/B comparison).
bool& force_single_cta();
int epi_mode(const Epi& e);
long long& launch_counter();

// Optional per-kernel-class timing with CUDA events on the launching stream
// (bench.py's roofline). Disabled by default; zero cost when off.
// PROF_ATTN: encoder / QFormer attention (tensor-bound); PROF_XATTN: decoder
// cross attention over the cached encoder K / V (HBM-bound); PROF_FEAT: record
// feature gathers / the folded pathway fc1; PROF_NORM: RMSNorm passes.
enum ProfCat {
  PROF_GEMM = 0, PROF_GEMM_MOE, PROF_ATTN, PROF_DEC_SELF, PROF_MOE_ROUTE, PROF_BEAM, PROF_MISC,
  PROF_XATTN, PROF_FEAT, PROF_NORM, PROF_N
};
struct ProfScope {
  ProfScope(int cat, cudaStream_t s, double flops, double bytes);
  ~ProfScope();
  int idx = -1;
  cudaStream_t s;
};
void prof_enable(bool on);
void prof_note(const std::string& note);  // label the latest record (ORX_PROF_DUMP)
void prof_note_launch(const char* expr);  // label with the launched kernel's name (profiling only)
bool prof_enabled();
// Per category: launches, total ms, algorithmic flops, algorithmic bytes.
void prof_collect(long long* count, double* ms, double* flops, double* bytes);

}  // namespace orx
