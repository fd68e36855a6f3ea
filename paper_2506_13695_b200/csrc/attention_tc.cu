// tcgen05 / TMEM flash attention for the bf16 path (head dim 32, 64 or 128).
//
// One CTA per (segment b, head h, block of 128 query rows); two CTAs per SM.
//   warp 0    TMA producer: Q once; K (row-major keys x dh) and V^T (dh x keys,
//             written transposed by the producing GEMM's epilogue) in 64-key
//             blocks, double-buffered
//   warp 1    one thread issues tcgen05.mma:
//               S_j  = Q . K_j^T   (M=128, N=64, K=dh)    -> TMEM, 2 buffers
//               O   += P_j . V_j   (M=128, N=dh, K=64)     -> TMEM, A = P from TMEM
//             S_{j+1} is issued before P_j is ready, so QK^T of the next block
//             overlaps the softmax of the current one
//   warps 2-5 softmax, one thread per query row (TMEM lane = row): row max
//             with lazy rescaling (O in TMEM is rescaled only when the running
//             max grows by more than 2^8), P = exp2 packed bf16x2 and stored
//             back into the block's own S columns (tcgen05.st) as the A operand
//             of P.V, final O / l. With P in TMEM (two S/P buffers) the softmax
//             of block j+1 never waits for P_j . V_j; MMAs run in issue order,
//             so S_{j+2} overwrites P_j only after P_j . V_j has read it.
// Semantics are mha_core's (tape.cpp:822-905): softmax(Q K^T / sqrt(dh)) V,
// max-subtracted, keys beyond the segment length masked.
#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "attention.cuh"
#include "common.cuh"
#include "gemm.cuh"

namespace orx {

namespace {

__device__ __forceinline__ int seg_start(const Seg& s, int b) { return s.start ? s.start[b] : b * s.stride; }
__device__ __forceinline__ int seg_len(const Seg& s, int b) { return s.len ? s.len[b] : s.fixed_len; }

ORX_DEV void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
ORX_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// D[tmem] (+)= A[tmem] * B[smem]^T (A: 128 lanes x K, bf16 packed two per 32-bit column)
ORX_DEV void tc_mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}

template <int DH>
struct Fmha {
  static constexpr int BQ = 128, BK = 64;
  // Q / K rows are stored as ROWB-byte swizzled rows: 128 B (SWIZZLE_128B, 64
  // elements per column block) for dh >= 64, 64 B (SWIZZLE_64B) for dh = 32
  static constexpr int ROWB = DH >= 64 ? 128 : 64;
  static constexpr int CB = DH * 2 / ROWB;            // column blocks of Q / K
  static constexpr int KPR = ROWB / 32;               // K=16 MMA steps per swizzled row
  static constexpr uint32_t Q_BYTES = BQ * DH * 2;    // CB blocks of [128 rows x 128 B]
  static constexpr uint32_t K_BYTES = BK * DH * 2;    // CB blocks of [64 rows x 128 B]
  static constexpr uint32_t V_BYTES = DH * BK * 2;    // [DH rows (head dims) x 64 keys]
  static constexpr int KST = 3, VST = 2;              // K ring deeper than V: S_j needs K_j first
  static constexpr uint32_t SMEM = Q_BYTES + KST * K_BYTES + VST * V_BYTES + 256;  // + barriers (17 x 8 B)
  static constexpr uint32_t TMEM_COLS = 2 * BK + DH <= 256 ? 256 : 512;  // S[2] + O
  static_assert(DH == 32 || DH % 64 == 0, "head dim 32 or a multiple of 64");
};
// K-major operand descriptor for ROWB-byte swizzled rows (8-row core groups)
template <int ROWB>
ORX_DEV uint64_t umma_desc_rows(uint32_t smem_addr) {
  if constexpr (ROWB == 128) {
    return umma_desc_sw128(smem_addr);
  } else {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr & 0x3FFFF) >> 4);  // start address
    d |= static_cast<uint64_t>(1) << 16;                      // LBO (ignored)
    d |= static_cast<uint64_t>(512 >> 4) << 32;               // SBO: 8 rows x 64 B
    d |= static_cast<uint64_t>(1) << 46;                      // descriptor version (sm100)
    d |= static_cast<uint64_t>(4) << 61;                      // SWIZZLE_64B
    return d;
  }
}

template <int DH>
__global__ void __launch_bounds__(192) fmha_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                                                       const __grid_constant__ CUtensorMap tmK,
                                                       const __grid_constant__ CUtensorMap tmV, int heads, int nqt,
                                                       int n_seg, __nv_bfloat16* __restrict__ O, int ldo, Seg qs,
                                                       Seg ks, Seg os, const int32_t* __restrict__ vt_user,
                                                       int q_col0, int k_col0) {
  pdl_begin();
  using F = Fmha<DH>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + F::Q_BYTES;            // [KST][K_BYTES]
  uint8_t* sV = sK + F::KST * F::K_BYTES;   // [VST][V_BYTES]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + F::VST * F::V_BYTES);
  uint64_t& q_full = bars[0];
  uint64_t* k_full = bars + 1;    // [KST]
  uint64_t* k_empty = bars + 4;   // [KST]
  uint64_t* v_full = bars + 7;    // [VST]
  uint64_t* v_empty = bars + 9;   // [VST]
  uint64_t* s_full = bars + 11;   // [2]
  uint64_t& p_full = bars[13];
  uint64_t& o_done = bars[14];
  uint64_t& q_empty = bars[15];
  uint32_t& tmem_slot = *reinterpret_cast<uint32_t*>(bars + 16);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    if ((smem_u32(smem) & 1023) != 0) __trap();  // SW128 operands need 1 KB alignment
    mbar_init(&q_full, 1);
    mbar_init(&q_empty, 1);
    for (int s = 0; s < F::KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < F::VST; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) mbar_init(&s_full[s], 1);
    mbar_init(&p_full, 4);
    mbar_init(&o_done, 1);
    fence_mbar_init();
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
  }
  if (warp == 1) tmem_alloc(&tmem_slot, F::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t t_s = tmem;             // S buffers: cols [0, 64), [64, 128)
  const uint32_t t_o = tmem + 2 * F::BK;  // O: cols [128, 128 + DH)

  // Persistent: this CTA walks tiles t = blockIdx.x, + gridDim.x, ...; tile t =
  // (segment b, head h, query block qt) with t = (b * heads + h) * nqt + qt.
  // Every role walks the same list (empty tiles skipped identically), and the
  // K / V rings, S buffers and barrier phases run on CTA-global block counters,
  // so the next tile's loads and QK^T overlap the current tile's tail.
  const int total = n_seg * heads * nqt;
  struct Tile {
    int b, h, q0, qlen, qst, kst, klen, ost, nb, vrow0;
  };
  auto tile_at = [&](int t, Tile& T) {
    T.b = t / (heads * nqt);
    const int r = t - T.b * heads * nqt;
    T.h = r / nqt;
    T.q0 = (r - T.h * nqt) * F::BQ;
    T.qlen = seg_len(qs, T.b);
    T.klen = seg_len(ks, T.b);
    if (T.q0 >= T.qlen || T.klen <= 0) return false;
    T.qst = seg_start(qs, T.b);
    T.kst = seg_start(ks, T.b);
    T.ost = seg_start(os, T.b);
    T.nb = (T.klen + F::BK - 1) / F::BK;
    T.vrow0 = ((vt_user ? vt_user[T.b] : T.b) * heads + T.h) * DH;
    return true;
  };

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_normal();
      int kc = 0, vc = 0, tc = 0;  // K blocks, V blocks, tiles loaded so far
      Tile T;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        if (!tile_at(t, T)) continue;
        if (tc > 0) mbar_wait(&q_empty, (tc - 1) & 1);  // the previous tile's last QK^T has read Q
        mbar_arrive_expect_tx(&q_full, F::Q_BYTES);
        for (int cb = 0; cb < F::CB; ++cb)
          tma_load_2d(sQ + cb * (F::BQ * F::ROWB), &tmQ, &q_full, q_col0 + T.h * DH + cb * (F::ROWB / 2),
                      T.qst + T.q0, pol);
        // K runs one block ahead of V (V_j is consumed a softmax later than K_j)
        for (int i = 0; i <= T.nb; ++i) {
          if (i < T.nb) {
            const int kslot = kc % F::KST;
            if (kc >= F::KST) mbar_wait(&k_empty[kslot], ((kc / F::KST) - 1) & 1);
            mbar_arrive_expect_tx(&k_full[kslot], F::K_BYTES);
            for (int cb = 0; cb < F::CB; ++cb)
              tma_load_2d(sK + kslot * F::K_BYTES + cb * (F::BK * F::ROWB), &tmK, &k_full[kslot],
                          k_col0 + T.h * DH + cb * (F::ROWB / 2), T.kst + i * F::BK, pol);
            ++kc;
          }
          const int j = i - 1;
          if (j >= 0) {
            const int vslot = vc % F::VST;
            if (vc >= F::VST) mbar_wait(&v_empty[vslot], ((vc / F::VST) - 1) & 1);
            mbar_arrive_expect_tx(&v_full[vslot], F::V_BYTES);
            tma_load_2d(sV + vslot * F::V_BYTES, &tmV, &v_full[vslot], j * F::BK, T.vrow0, pol);
            ++vc;
          }
        }
        ++tc;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(F::BQ, F::BK);
      constexpr uint32_t idesc_o = umma_idesc_bf16(F::BQ, DH);
      // PV of global block gp (first = first block of its tile: overwrite O)
      auto issue_pv = [&](int gp, bool first) {
        const int st = gp & 1, vslot = gp % F::VST;
        mbar_wait(&v_full[vslot], (gp / F::VST) & 1);
        mbar_wait(&p_full, gp & 1);
        tc_fence_after();
        const uint32_t b0 = smem_u32(sV + vslot * F::V_BYTES);
        // A = P: 128 lanes x 64 keys bf16 = 32 TMEM columns at the start of S buffer st, 8 per K=16 step
#pragma unroll
        for (int k = 0; k < F::BK / 16; ++k)
          tc_mma_bf16_ts(t_o, t_s + st * F::BK + k * 8, umma_desc_sw128(b0 + k * 32), idesc_o, !(first && k == 0));
        tc_commit(&o_done);
        tc_commit(&v_empty[vslot]);
      };
      int g = 0, tc = 0;
      bool prev_first = false;
      Tile T;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        if (!tile_at(t, T)) continue;
        mbar_wait(&q_full, tc & 1);
        tc_fence_after();
        for (int j = 0; j < T.nb; ++j, ++g) {
          const int st = g & 1, kslot = g % F::KST;
          mbar_wait(&k_full[kslot], (g / F::KST) & 1);
          tc_fence_after();
          const uint32_t qa = smem_u32(sQ), kb = smem_u32(sK + kslot * F::K_BYTES);
#pragma unroll
          for (int k = 0; k < DH / 16; ++k) {
            const int cb = k / F::KPR, off = (k % F::KPR) * 32;
            tc_mma_bf16(t_s + st * F::BK, umma_desc_rows<F::ROWB>(qa + cb * (F::BQ * F::ROWB) + off),
                        umma_desc_rows<F::ROWB>(kb + cb * (F::BK * F::ROWB) + off), idesc_s, k != 0);
          }
          tc_commit(&s_full[st]);
          tc_commit(&k_empty[kslot]);
          if (j == T.nb - 1) tc_commit(&q_empty);
          if (g >= 1) issue_pv(g - 1, prev_first);
          prev_first = j == 0;
        }
        ++tc;
      }
      if (g >= 1) issue_pv(g - 1, prev_first);
    }
  } else {
    const int q = warp & 3;  // TMEM lane quadrant
    const int r = q * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const float scale_log2 = rsqrtf(static_cast<float>(DH)) * 1.4426950408889634f;
    int g = 0;
    Tile T;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      if (!tile_at(t, T)) continue;
      if (T.q0 + q * 32 >= T.qlen) {
        // no query row of this warp's quadrant is real (the 21-row tail tile of
        // a 405-row encoder segment, decode step 0): its P rows only feed
        // output rows that are never stored, so skip the softmax and only keep
        // the block handshake: one p_full arrival per block, each only after the
        // previous block's phase completed (an early arrival would count
        // towards the current phase and release P . V before the real rows)
        for (int j = 0; j < T.nb; ++j, ++g) {
          if (g >= 1) mbar_wait(&p_full, (g - 1) & 1);
          if (lane == 0) mbar_arrive(&p_full);
        }
        continue;
      }
      float m = -FLT_MAX, l = 0.f;
      bool first = true;
      for (int j = 0; j < T.nb; ++j, ++g) {
        const int st = g & 1;
        mbar_wait(&s_full[st], (g >> 1) & 1);
        __syncwarp();  // tcgen05.ld/st are .sync.aligned: reconverge after the per-thread wait / branches
        tc_fence_after();
        uint32_t sa[32], sb[32];
        tmem_ld32_async(t_s + lane_off + st * F::BK, sa);
        tmem_ld32_async(t_s + lane_off + st * F::BK + 32, sb);
        tmem_wait_ld();
        const int valid = T.klen - j * F::BK;
        float x[64];  // raw scores; the 1/sqrt(dh) * log2(e) scale is folded into the exponent's FMA
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = __uint_as_float(sa[i]), x[32 + i] = __uint_as_float(sb[i]);
        if (valid < F::BK) {  // tail block only: keys beyond the segment
#pragma unroll
          for (int i = 0; i < 64; ++i)
            if (i >= valid) x[i] = -INFINITY;
        }
        float bm = fmaxf(x[0], x[1]);
#pragma unroll
        for (int i = 2; i < 64; i += 2) bm = fmaxf(bm, fmaxf(x[i], x[i + 1]));  // FMNMX3
        bm *= scale_log2;
        float corr = 1.f;
        bool resc = false;
        if (first || bm > m + 8.f) {  // lazy rescale: keep a stale max unless it grew by > 2^8
          corr = first ? 0.f : ex2_fast(m - bm);
          resc = !first;
          m = bm;
          first = false;
        }
        const float2 sc = make_float2(scale_log2, scale_log2), nm = make_float2(-m, -m);
        float2 acc2 = make_float2(0.f, 0.f);
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float2 tt = ffma2(make_float2(x[2 * i], x[2 * i + 1]), sc, nm);
          const float2 p = make_float2(ex2_fast(tt.x), ex2_fast(tt.y));
          acc2 = fadd2(acc2, p);
          pk[i] = pack_bf16(p.x, p.y);
        }
        const float sum = acc2.x + acc2.y;
        l = l * corr + sum;
        // P replaces S in TMEM (columns [0, 32) of this buffer, keys 2c / 2c+1 in column c)
        __syncwarp();
        tmem_st32(t_s + lane_off + st * F::BK, pk);
        // the previous block's P . V (same tile) is normally long done by now; waiting
        // for it keeps o_done at most one phase ahead and orders the O rescale after it
        if (j >= 1) {
          mbar_wait(&o_done, (g - 1) & 1);
          __syncwarp();
          tc_fence_after();
        }
        if (__any_sync(0xffffffffu, resc)) {
          const float c = resc ? corr : 1.f;
#pragma unroll 1
          for (int cc = 0; cc < DH / 32; ++cc) {
            uint32_t o[32];
            tmem_ld32_async(t_o + lane_off + cc * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * c);
            tmem_st32(t_o + lane_off + cc * 32, o);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full);
      }
      mbar_wait(&o_done, (g - 1) & 1);  // this tile's last P . V
      __syncwarp();
      tc_fence_after();
      const float inv = 1.f / l;
      const bool store = T.q0 + r < T.qlen;
      __nv_bfloat16* orow = O + (size_t)(T.ost + T.q0 + r) * ldo + T.h * DH;
#pragma unroll 1
      for (int cc = 0; cc < DH / 32; ++cc) {
        uint32_t o[32];
        tmem_ld32_async(t_o + lane_off + cc * 32, o);
        tmem_wait_ld();
        if (store) {
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 w;
            w.x = pack_bf16(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv);
            w.y = pack_bf16(__uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv);
            w.z = pack_bf16(__uint_as_float(o[i + 4]) * inv, __uint_as_float(o[i + 5]) * inv);
            w.w = pack_bf16(__uint_as_float(o[i + 6]) * inv, __uint_as_float(o[i + 7]) * inv);
            *reinterpret_cast<uint4*>(orow + cc * 32 + i) = w;
          }
        }
      }
      // the next tile's first P . V overwrites O: issued only after p_full of its
      // first block, which these threads arrive after this read (tcgen05.ld waited)
      tc_fence_before();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, F::TMEM_COLS);
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

CUtensorMap map2d(const void* ptr, long long rows, long long cols, long long ld, int box_cols, int box_rows,
                  CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  CUtensorMap m;
  cuuint64_t gdim[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t gstride[1] = {static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), gdim, gstride, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("attention tensor map encode failed (" + std::to_string(int(r)) + ")");
  return m;
}

template <int DH>
void launch_fmha(const FmhaArgs& a, cudaStream_t s) {
  using F = Fmha<DH>;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(fmha_tc_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(F::SMEM));
    set = true;
  }
  // Q/K maps start at the head-0 column of their buffers (column offsets are
  // added in the kernel): rows x (q_col0 + heads * DH) columns.
  constexpr CUtensorMapSwizzle qk_swz = F::ROWB == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  CUtensorMap mq = map2d(a.Q, a.q_rows, a.q_col0 + a.heads * DH, a.ldq, F::ROWB / 2, F::BQ, qk_swz);
  CUtensorMap mk = map2d(a.K, a.k_rows, a.k_col0 + a.heads * DH, a.ldk, F::ROWB / 2, F::BK, qk_swz);
  CUtensorMap mv = map2d(a.Vt, a.vt_rows, a.vt_cols, a.vt_ld, 64, DH);
  const int nqt = (a.max_q + F::BQ - 1) / F::BQ;
  const long long tiles = static_cast<long long>(nqt) * a.heads * a.B;
  const int grid = static_cast<int>(std::min<long long>(tiles, 2LL * num_sms()));  // persistent, two CTAs per SM
  launch_pdl(fmha_tc_kernel<DH>, grid, 192, F::SMEM, s, mq, mk, mv, a.heads, nqt, a.B,
             static_cast<__nv_bfloat16*>(a.O), a.ldo, a.q, a.k, a.o, a.vt_user, a.q_col0, a.k_col0);
}

}  // namespace

bool fmha_supported(int dh) { return dh == 32 || dh == 64 || dh == 128; }

void launch_fmha_tc(const FmhaArgs& a, cudaStream_t s) {
  if (a.B <= 0 || a.max_q <= 0) return;
  if (a.ldq % 8 || a.ldk % 8 || a.vt_ld % 8 || a.q_col0 % 8 || a.k_col0 % 8)
    throw std::invalid_argument("fmha: strides / column offsets must be multiples of 8 elements");
  ProfScope ps(a.prof_cat, s, a.flops, a.bytes);
  if (prof_enabled())
    prof_note("fmha B=" + std::to_string(a.B) + " heads=" + std::to_string(a.heads) + " max_q=" +
              std::to_string(a.max_q) + " k_rows=" + std::to_string(a.k_rows));
  if (a.dh == 128) launch_fmha<128>(a, s);
  else if (a.dh == 64) launch_fmha<64>(a, s);
  else if (a.dh == 32) launch_fmha<32>(a, s);
  else throw std::invalid_argument("fmha: head dim must be 32, 64 or 128");
  ++launch_counter();
}

}  // namespace orx
