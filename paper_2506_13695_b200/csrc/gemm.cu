// tcgen05/TMEM/TMA GEMM for sm_100a (bf16 in, fp32 accumulate in TMEM) and
// the fp32 SIMT GEMM used by the fp32 parity mode. See gemm.cuh.
//
// tcgen05 kernel structure (persistent, warp-specialised, 192 threads):
//   warp 0    : TMA producer, STAGES-deep smem ring (full/empty mbarriers)
//   warp 1    : TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5 : epilogue; TMEM -> registers (tcgen05.ld 32x32b) -> fused
//               bias/activation/scale/residual -> global
// Accumulators are double-buffered in TMEM (2 x BN fp32 columns) so the
// epilogue of tile i overlaps the MMAs of tile i+1.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"
#include "gemm.cuh"

namespace orx {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = 128 B = one swizzle row

// ---------------------------------------------------------------------------
// epilogue (shared by the 1-CTA and CTA-pair kernels)
//
// 8 epilogue warps per CTA: warp w may only touch TMEM lanes 32*(w%4)..+31
// (its row quadrant); the two warps of a quadrant split the tile's columns.
// Each thread owns one output row. The residual of the next 32-column chunk
// is loaded while the current chunk is finished, and the first chunk's
// residual is in flight before the accumulator is even ready.
// ---------------------------------------------------------------------------
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;  // warp 0 TMA, warp 1 MMA, 8 epilogue warps

__device__ __forceinline__ int resid_row(const Epi& e, int orow) {
  return e.resid_mod > 0 ? orow % e.resid_mod : orow;
}
__device__ __forceinline__ void epi_load_resid(const Epi& e, int orow, int col0, float (&r)[32]) {
  const float* rp = e.resid + (size_t)resid_row(e, orow) * e.ld_resid + col0;
  if (col0 + 32 <= e.n_out && ((reinterpret_cast<uintptr_t>(rp) & 15) == 0)) {
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      float4 t = __ldg(reinterpret_cast<const float4*>(rp + j));
      r[j] = t.x, r[j + 1] = t.y, r[j + 2] = t.z, r[j + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = col0 + j < e.n_out ? rp[j] : 0.f;
  }
}

// Specialised epilogue for a full, aligned 32-column chunk: MODE is the
// Epi::mode bit set (no per-element predication, vector bias loads).
template <int MODE>
__device__ __forceinline__ void epi_fast(const Epi& e, int orow, float rs, int col0, float (&v)[32],
                                         const float (&r)[32]) {
  if (MODE & EPI_BIAS) {
    const float4* b4 = reinterpret_cast<const float4*>(e.bias + col0);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 b = __ldg(b4 + q);
      v[4 * q] += b.x, v[4 * q + 1] += b.y, v[4 * q + 2] += b.z, v[4 * q + 3] += b.w;
    }
  }
  if (MODE & EPI_LEAKY) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = v[j] > 0.f ? v[j] : 0.01f * v[j];  // tape.hpp:88
  }
  if (MODE & EPI_SILU) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = silu_fast(v[j]);
  }
  if (MODE & EPI_RS) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] *= rs;
  }
  if (MODE & EPI_RESID) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] += r[j];
  }
  const int oc = col0 + e.col_off;
  if (MODE & EPI_BF16) {
    uint4* op = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(e.out) + (size_t)orow * e.ldo + oc);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      op[q] = make_uint4(pack_bf16(v[8 * q], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                         pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
  } else {
    float4* op = reinterpret_cast<float4*>(reinterpret_cast<float*>(e.out) + (size_t)orow * e.ldo + oc);
#pragma unroll
    for (int q = 0; q < 8; ++q) op[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
}

// bias -> activation -> row scale -> + residual -> store (bf16 or fp32)
__device__ __forceinline__ void epi_finish32(const Epi& e, int orow, float rs, int col0, float (&v)[32],
                                             const float (&r)[32], bool has_res) {
  if (col0 >= e.n_out) return;
  const bool full = col0 + 32 <= e.n_out;
  if (full && e.mode >= 0) {  // host verified alignment and that the flags match a specialised mode
    switch (e.mode) {
      case 0: epi_fast<0>(e, orow, rs, col0, v, r); return;
      case EPI_RS: epi_fast<EPI_RS>(e, orow, rs, col0, v, r); return;
      case EPI_RS | EPI_BF16: epi_fast<EPI_RS | EPI_BF16>(e, orow, rs, col0, v, r); return;
      case EPI_RESID: epi_fast<EPI_RESID>(e, orow, rs, col0, v, r); return;
      case EPI_BIAS | EPI_RESID: epi_fast<EPI_BIAS | EPI_RESID>(e, orow, rs, col0, v, r); return;
      case EPI_BF16: epi_fast<EPI_BF16>(e, orow, rs, col0, v, r); return;
      case EPI_BIAS | EPI_BF16: epi_fast<EPI_BIAS | EPI_BF16>(e, orow, rs, col0, v, r); return;
      case EPI_BIAS | EPI_LEAKY | EPI_BF16: epi_fast<EPI_BIAS | EPI_LEAKY | EPI_BF16>(e, orow, rs, col0, v, r); return;
      case EPI_BIAS | EPI_SILU | EPI_BF16: epi_fast<EPI_BIAS | EPI_SILU | EPI_BF16>(e, orow, rs, col0, v, r); return;
      default: break;
    }
  }
  if (e.bias) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (full || col0 + j < e.n_out) v[j] += __ldg(e.bias + col0 + j);
  }
  if (e.act == ACT_LEAKY) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = v[j] > 0.f ? v[j] : 0.01f * v[j];  // tape.hpp:88
  } else if (e.act == ACT_SILU) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = silu_fast(v[j]);
  }
  if (rs != 1.f) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] *= rs;
  }
  if (has_res) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] += r[j];
  }
  const int oc = col0 + e.col_off;
  if (e.vt && oc >= e.vt_col0) {  // transposed bf16 store: lanes (consecutive rows) write consecutive t
    const int u = e.vt_row_user ? e.vt_row_user[orow] : orow / e.vt_T;
    const int t = e.vt_row_pos ? e.vt_row_pos[orow] : orow % e.vt_T;
    const int l = (oc - e.vt_col0) / e.vt_cols, m0 = (oc - e.vt_col0) - l * e.vt_cols;  // a 32-column chunk stays in one layer (vt_cols % 32 == 0)
    __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(e.vt) + (long long)u * e.vt_user_stride + t +
                          (long long)l * e.vt_layer_stride + (long long)m0 * e.vt_ld;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (full || col0 + j < e.n_out) base[(long long)j * e.vt_ld] = __float2bfloat16_rn(v[j]);
    return;
  }
  if (e.out_bf16) {
    __nv_bfloat16* op = reinterpret_cast<__nv_bfloat16*>(e.out) + (size_t)orow * e.ldo + oc;
    if (full && ((reinterpret_cast<uintptr_t>(op) & 15) == 0)) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 w;
        w.x = pack_bf16(v[j], v[j + 1]);
        w.y = pack_bf16(v[j + 2], v[j + 3]);
        w.z = pack_bf16(v[j + 4], v[j + 5]);
        w.w = pack_bf16(v[j + 6], v[j + 7]);
        *reinterpret_cast<uint4*>(op + j) = w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < e.n_out) op[j] = __float2bfloat16_rn(v[j]);
    }
  } else {
    float* op = reinterpret_cast<float*>(e.out) + (size_t)orow * e.ldo + oc;
    if (full && ((reinterpret_cast<uintptr_t>(op) & 15) == 0)) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(op + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < e.n_out) op[j] = v[j];
    }
  }
}

// One accumulator tile, this thread's row, this warp's column half.
// tb = TMEM address of (quadrant lane 0, accumulator column 0).
template <int BN>
__device__ __forceinline__ void epilogue_tile(const Epi& e, uint32_t tb, int row, int nt, int half, uint64_t* tfull,
                                              uint32_t acc_phase) {
  int orow = -1;
  float rs = 1.f;
  if (row < e.m_valid) {
    orow = e.row_map ? e.row_map[row] : row;
    if (e.row_scale) rs = e.row_scale[row];
  }
  const bool ok = orow >= 0;
  if (e.swiglu) {
    // B rows interleaved per 128: accumulator cols [0,BN/2) = W1, [BN/2,BN) = W3 (swiglu, nn.cpp:84-86)
    constexpr int CP = BN / 64 / 2;
    mbar_wait(tfull, acc_phase);
    __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after the per-thread wait
    tc_fence_after();
#pragma unroll
    for (int i = 0; i < CP; ++i) {
      const int c = half * CP + i;
      uint32_t ra[32], rb[32];
      tmem_ld32_async(tb + c * 32, ra);
      tmem_ld32_async(tb + BN / 2 + c * 32, rb);
      tmem_wait_ld();
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = silu_fast(__uint_as_float(ra[j])) * __uint_as_float(rb[j]);
      float r[32];
      const bool hr = ok && e.resid;
      if (hr) epi_load_resid(e, orow, nt * (BN / 2) + c * 32, r);
      if (ok) epi_finish32(e, orow, rs, nt * (BN / 2) + c * 32, v, r, hr);
    }
  } else {
    constexpr int CH = BN / 32 / 2;
    const bool hr = ok && e.resid != nullptr;
    float rc[32];
    if (hr) {
      // pull this thread's residual row segment (CH * 128 B) into L2 while the MMAs run;
      // the chunk loads below then hit L2 instead of waiting on HBM one chunk at a time
      const float* rp = e.resid + (size_t)resid_row(e, orow) * e.ld_resid + nt * BN + half * CH * 32;
      if (nt * BN + (half + 1) * CH * 32 <= e.n_out && (reinterpret_cast<uintptr_t>(rp) & 15) == 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rp), "r"(CH * 128) : "memory");
      epi_load_resid(e, orow, nt * BN + half * CH * 32, rc);  // in flight while the MMAs finish
    }
    mbar_wait(tfull, acc_phase);
    __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after the per-thread wait
    tc_fence_after();
#pragma unroll 1
    for (int i = 0; i < CH; ++i) {
      const int c = half * CH + i;
      uint32_t ra[32];
      tmem_ld32_async(tb + c * 32, ra);
      if (hr && i > 0) epi_load_resid(e, orow, nt * BN + c * 32, rc);  // overlaps the TMEM load
      tmem_wait_ld();
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(ra[j]);
      if (ok) epi_finish32(e, orow, rs, nt * BN + c * 32, v, rc, hr);
    }
  }
}

// Staged epilogue for full, aligned tiles (CTA-pair kernel). TMEM hands each
// thread one ROW of 32 columns; storing that directly makes every warp access
// touch 32 rows (32 L1 wavefronts per instruction, 2-3 TB/s on the fp32
// residual GEMMs). Instead each warp transposes its 32x32 chunk through a
// 4 KB XOR-swizzled SMEM tile and then reads / writes global memory row-wise:
// 8 lanes cover one row's 128 B, one instruction covers 4 rows. The residual
// chunk is loaded in that coalesced layout while tcgen05.ld runs.
template <int BN, int MODE>
__device__ __forceinline__ void epilogue_tile_staged(const Epi& e, float* stg, uint32_t tb, int row, int nt,
                                                     int half, uint64_t* tfull, uint32_t acc_phase) {
  constexpr int CH = BN / 32 / 2;
  const int lane = threadIdx.x & 31, sub = lane >> 3, q = lane & 7;
  int orow = -1;
  float rs = 1.f, rsq = 1.f;
  unsigned long long pbase = 0;  // EPI_PEER: this row's destination buffer
  if (row < e.m_valid) {
    if (MODE & EPI_PEER) {
      const int code = e.peer_code[row];
      orow = code < 0 ? -1 : (code & 0xFFFFFF);
      pbase = reinterpret_cast<unsigned long long>(e.peer_out[code < 0 ? 0 : (code >> 24)]);
    } else {
      orow = e.row_map ? e.row_map[row] : row;
    }
    if (MODE & EPI_RS) rs = e.row_scale[row];
    if (MODE & EPI_RSQ) {  // folded RMSNorm: this row's scale from the producer's partial sums of squares
      float ss = 0.f;
      for (int i = 0; i < e.rsq_n; ++i) ss += e.rsq[(long long)i * e.rsq_ld + row];
      rsq = rsqrtf(ss * e.rsq_inv_d + 1e-6f);
    }
  }
  float ssp[8];  // producer: partial sums of squares of rows 4k + sub over this warp's columns
#pragma unroll
  for (int k = 0; k < 8; ++k) ssp[k] = 0.f;
  int orr[8];  // output rows this lane stores: r = 4 * k + sub
#pragma unroll
  for (int k = 0; k < 8; ++k) orr[k] = __shfl_sync(0xffffffffu, orow, 4 * k + sub);
  // EPI_PEER stores 16 B per lane (4 lanes per row, rows 8k + lane / 4): half
  // the store instructions of the 8-B layout, 64 B contiguous per row and chunk
  unsigned long long pb[(MODE & EPI_PEER) ? 4 : 1];
  int prow[(MODE & EPI_PEER) ? 4 : 1];
  if constexpr ((MODE & EPI_PEER) != 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      pb[k] = __shfl_sync(0xffffffffu, pbase, 8 * k + (lane >> 2));
      prow[k] = __shfl_sync(0xffffffffu, orow, 8 * k + (lane >> 2));
    }
  }
  if (MODE & EPI_RESID) {
    if (orow >= 0)  // this row's residual segment into L2 while the MMAs run
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(e.resid + (size_t)((MODE & EPI_RMOD) ? orow % e.resid_mod : orow) * e.ld_resid +
                                                                       nt * BN + half * CH * 32),
                   "r"(CH * 128)
                   : "memory");
  }
  float4* s4 = reinterpret_cast<float4*>(stg);
  // residual chunks in the coalesced layout, one chunk ahead: chunk 0 is in
  // flight while the MMAs finish, chunk i+1 while chunk i is finished
  float4 rr[2][8];
  auto load_resid = [&](int i, float4 (&dst)[8]) {
    const int col0 = nt * BN + (half * CH + i) * 32;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      dst[k] = orr[k] >= 0 ? __ldg(reinterpret_cast<const float4*>(e.resid + (size_t)((MODE & EPI_RMOD) ? orr[k] % e.resid_mod : orr[k]) * e.ld_resid + col0) + q)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  if (MODE & EPI_RESID) load_resid(0, rr[0]);
  mbar_wait(tfull, acc_phase);
  __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after the per-thread wait
  tc_fence_after();
  auto do_chunk = [&](int i, const float4 (&cur)[8], float4 (&nxt)[8]) {
    const int col0 = nt * BN + (half * CH + i) * 32;
    uint32_t ra[32];
    tmem_ld32_async(tb + (half * CH + i) * 32, ra);
    if ((MODE & EPI_RESID) && i + 1 < CH) load_resid(i + 1, nxt);
    tmem_wait_ld();
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(ra[j]);
    if (MODE & EPI_RSQ) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] *= rsq;
    }
    if (MODE & EPI_BIAS) {
      const float4* b4 = reinterpret_cast<const float4*>(e.bias + col0);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float4 b = __ldg(b4 + k);
        v[4 * k] += b.x, v[4 * k + 1] += b.y, v[4 * k + 2] += b.z, v[4 * k + 3] += b.w;
      }
    }
    if (MODE & EPI_LEAKY) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = v[j] > 0.f ? v[j] : 0.01f * v[j];  // tape.hpp:88
    }
    if (MODE & EPI_SILU) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = silu_fast(v[j]);
    }
    if (MODE & EPI_RS) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] *= rs;
    }
    if (MODE & EPI_STATS) {  // this row's 32-column chunk: max and sum exp(x - max) (log-softmax inputs)
      float m = fmaxf(v[0], v[1]);
#pragma unroll
      for (int j = 2; j < 32; ++j) m = fmaxf(m, v[j]);
      const float2 l2 = make_float2(1.4426950408889634f, 1.4426950408889634f);
      const float2 nm = make_float2(-m * 1.4426950408889634f, -m * 1.4426950408889634f);
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float2 t = ffma2(make_float2(v[j], v[j + 1]), l2, nm);
        acc = fadd2(acc, make_float2(ex2_fast(t.x), ex2_fast(t.y)));
      }
      if (row < e.m_valid) e.stats[(long long)(col0 >> 5) * e.stats_ld + row] = make_float2(m, acc.x + acc.y);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
      s4[lane * 8 + (k ^ (lane & 7))] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
    __syncwarp();
    if constexpr ((MODE & EPI_PEER) != 0) {  // rows 8k + lane / 4, columns 8 (lane % 4) .. + 8
      const int c8 = lane & 3, pc = col0 + e.col_off + 8 * c8;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int r = 8 * k + (lane >> 2);
        const float4 a = s4[r * 8 + ((2 * c8) ^ (r & 7))], b = s4[r * 8 + ((2 * c8 + 1) ^ (r & 7))];
        if (prow[k] >= 0)
          *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(pb[k]) + (size_t)prow[k] * e.ldo + pc) =
              make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y), pack_bf16(b.z, b.w));
      }
      __syncwarp();
      return;
    }
    const int oc = col0 + e.col_off + 4 * q;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = 4 * k + sub;
      float4 x = s4[r * 8 + (q ^ (r & 7))];
      if (orr[k] < 0) continue;
      if (MODE & EPI_RESID) {
        const float4 y = cur[k];
        x.x += y.x, x.y += y.y, x.z += y.z, x.w += y.w;
      }
      if (MODE & EPI_BF16) {
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(e.out) + (size_t)orr[k] * e.ldo + oc) =
            make_uint2(pack_bf16(x.x, x.y), pack_bf16(x.z, x.w));
      } else {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(e.out) + (size_t)orr[k] * e.ldo + oc) = x;
      }
      if (MODE & EPI_XSSQ) {  // the next GEMM's A operand and its RMSNorm statistics
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(e.out2) + (size_t)orr[k] * e.ldo2 + oc) =
            make_uint2(pack_bf16(x.x, x.y), pack_bf16(x.z, x.w));
        ssp[k] += x.x * x.x + x.y * x.y + x.z * x.z + x.w * x.w;
      }
    }
    __syncwarp();  // the next chunk reuses stg
  };
  static_assert(CH % 2 == 0, "chunks are processed in pairs");
#pragma unroll 1
  for (int i = 0; i < CH; i += 2) {
    do_chunk(i, rr[0], rr[1]);
    do_chunk(i + 1, rr[1], rr[0]);
  }
  if (MODE & EPI_XSSQ) {  // rows 4k + sub: reduce over the 8 lanes of the row group, one store per row
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float t = ssp[k];
      t += __shfl_xor_sync(0xffffffffu, t, 1);
      t += __shfl_xor_sync(0xffffffffu, t, 2);
      t += __shfl_xor_sync(0xffffffffu, t, 4);
      if (q == 0 && orr[k] >= 0) e.ssq[(long long)(nt * 2 + half) * e.ssq_ld + orr[k]] = t;
    }
  }
}

// Staged SwiGLU epilogue (MoE W1|W3 GEMM): silu(a) * b per 32-column chunk,
// then the same SMEM transpose and coalesced bf16 row stores as above.
template <int BN>
__device__ __forceinline__ void epilogue_tile_swiglu_staged(const Epi& e, float* stg, uint32_t tb, int row, int nt,
                                                            int half, uint64_t* tfull, uint32_t acc_phase) {
  constexpr int CP = BN / 64 / 2;  // 32-column output chunks per warp
  const int lane = threadIdx.x & 31, sub = lane >> 3, q = lane & 7;
  const int orow = row < e.m_valid ? (e.row_map ? e.row_map[row] : row) : -1;
  const float rr = e.row_rsq && row < e.m_valid ? e.row_rsq[row] : 1.f;  // folded RMSNorm scale of this row
  int orr[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) orr[k] = __shfl_sync(0xffffffffu, orow, 4 * k + sub);
  float4* s4 = reinterpret_cast<float4*>(stg);
  mbar_wait(tfull, acc_phase);
  __syncwarp();
  tc_fence_after();
#pragma unroll 1
  for (int i = 0; i < CP; ++i) {
    const int c = half * CP + i;
    uint32_t ra[32], rb[32];
    tmem_ld32_async(tb + c * 32, ra);
    tmem_ld32_async(tb + BN / 2 + c * 32, rb);
    tmem_wait_ld();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        v[j] = silu_fast(__uint_as_float(ra[4 * k + j]) * rr) * (__uint_as_float(rb[4 * k + j]) * rr);
      s4[lane * 8 + (k ^ (lane & 7))] = make_float4(v[0], v[1], v[2], v[3]);
    }
    __syncwarp();
    const int oc = nt * (BN / 2) + c * 32 + e.col_off + 4 * q;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = 4 * k + sub;
      const float4 x = s4[r * 8 + (q ^ (r & 7))];
      if (orr[k] >= 0)
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(e.out) + (size_t)orr[k] * e.ldo + oc) =
            make_uint2(pack_bf16(x.x, x.y), pack_bf16(x.z, x.w));
    }
    __syncwarp();
  }
}

// Transposed-V tile of a split K|V GEMM (columns >= vt_col0): per 32-column
// chunk, lanes (consecutive rows = consecutive key positions) store column j's
// 64-byte run of positions, one column per instruction.
template <int BN>
__device__ __forceinline__ void epilogue_tile_vt(const Epi& e, uint32_t tb, int row, int nt, int half, uint64_t* tfull,
                                                 uint32_t acc_phase) {
  constexpr int CH = BN / 32 / 2;
  const int orow = row < e.m_valid ? (e.row_map ? e.row_map[row] : row) : -1;
  const bool valid = orow >= 0;
  float rsq = 1.f;
  if (e.rsq && row < e.m_valid) {  // folded RMSNorm (EPI_RSQ), as in epilogue_tile_staged
    float ss = 0.f;
    for (int i = 0; i < e.rsq_n; ++i) ss += e.rsq[(long long)i * e.rsq_ld + row];
    rsq = rsqrtf(ss * e.rsq_inv_d + 1e-6f);
  }
  int u = 0, t = 0;
  if (valid) {
    u = e.vt_row_user ? e.vt_row_user[orow] : orow / e.vt_T;
    t = e.vt_row_pos ? e.vt_row_pos[orow] : orow % e.vt_T;
  }
  const int lane = threadIdx.x & 31;
  // 32 consecutive positions of one user starting at an even t0: lane pairs
  // swap values so each lane stores two positions of one column (4 bytes),
  // two columns per instruction, 16 stores per chunk instead of 32
  const int u0 = __shfl_sync(0xffffffffu, u, 0), t0 = __shfl_sync(0xffffffffu, t, 0);
  const bool pairs = __all_sync(0xffffffffu, valid && u == u0 && t == t0 + lane) && (t0 & 1) == 0;
  const bool odd = lane & 1;
  mbar_wait(tfull, acc_phase);
  __syncwarp();
  tc_fence_after();
#pragma unroll 1
  for (int i = 0; i < CH; ++i) {
    const int c = half * CH + i;
    uint32_t ra[32];
    tmem_ld32_async(tb + c * 32, ra);
    tmem_wait_ld();
    if (e.rsq) {
#pragma unroll
      for (int j = 0; j < 32; ++j) ra[j] = __float_as_uint(__uint_as_float(ra[j]) * rsq);
    }
    if (e.bias) {  // bias of the GEMM output column (the folded lifelong fc2 bias through Wk|Wv)
      const float* bp = e.bias + nt * BN + c * 32;
#pragma unroll
      for (int j = 0; j < 32; ++j) ra[j] = __float_as_uint(__uint_as_float(ra[j]) + __ldg(bp + j));
    }
    if (pairs) {
      const int oc = nt * BN + c * 32 + e.col_off - e.vt_col0;
      const int l = oc / e.vt_cols, m0 = oc - l * e.vt_cols;
      __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(e.vt) + (long long)u0 * e.vt_user_stride + t0 +
                            (lane & ~1) + (long long)l * e.vt_layer_stride + (long long)(m0 + odd) * e.vt_ld;
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float vj = __uint_as_float(ra[j]), vj1 = __uint_as_float(ra[j + 1]);
        const float recv = __shfl_xor_sync(0xffffffffu, odd ? vj : vj1, 1);
        *reinterpret_cast<uint32_t*>(base + (long long)j * e.vt_ld) = odd ? pack_bf16(recv, vj1) : pack_bf16(vj, recv);
      }
      continue;
    }
    if (!valid) continue;
    const int oc = nt * BN + c * 32 + e.col_off - e.vt_col0;
    const int l = oc / e.vt_cols, m0 = oc - l * e.vt_cols;
    __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(e.vt) + (long long)u * e.vt_user_stride + t +
                          (long long)l * e.vt_layer_stride + (long long)m0 * e.vt_ld;
#pragma unroll
    for (int j = 0; j < 32; ++j) base[(long long)j * e.vt_ld] = __float2bfloat16_rn(__uint_as_float(ra[j]));
  }
}

// ---------------------------------------------------------------------------
// tcgen05 persistent GEMM, one CTA per tile (128 x BN): small M
// ---------------------------------------------------------------------------
template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                   int N, int K, Epi epi, Grouped grp) {
  constexpr uint32_t A_BYTES = kBM * kBK * 2;
  constexpr uint32_t B_BYTES = BN * kBK * 2;
  constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN;  // double-buffered accumulator
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps);
    }
    fence_mbar_init();
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // setup above touches only parameters, SMEM and TMEM: overlap it with the
  // previous kernel's tail, then wait for that kernel's outputs
  pdl_begin();
  const int tile_rows = grp.tile_rows ? grp.tile_rows : kBM;
  const int m_tiles = grp.n_mtiles ? *grp.n_mtiles * (tile_rows / kBM) : (M + kBM - 1) / kBM;
  const int n_tiles = (N + BN - 1) / BN;
  const int total = m_tiles * n_tiles;
  const int kblocks = (K + kBK - 1) / kBK;
  auto expert_of = [&](int mt) { return grp.tile_expert[mt / (tile_rows / kBM)]; };

  if (warp == 0) {
    if (lane == 0) {
      // A is re-read by every N tile of its row block: keep it in L2 unless it is read once.
      const uint64_t pol_a = n_tiles > 1 ? l2_policy_evict_normal() : l2_policy_evict_first();
      const uint64_t pol_b = l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int mt = t / n_tiles, nt = t % n_tiles;
        int brow = nt * BN;
        if (grp.tile_expert) {
          int e = expert_of(mt);
          if (e < 0) continue;
          brow += e * grp.b_rows_per_expert;
        }
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_2d(sA + stage * A_BYTES, &tmA, &full[stage], kb * kBK, mt * kBM, pol_a);
          tma_load_2d(sB + stage * B_BYTES, &tmB, &full[stage], kb * kBK, brow, pol_b);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        if (grp.tile_expert && expert_of(t / n_tiles) < 0) continue;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            tc_mma_bf16(d_tmem, umma_desc_sw128(a_base + k * 32), umma_desc_sw128(b_base + k * 32), idesc,
                        (kb | k) != 0);
          }
          tc_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    const int q = warp & 3;            // TMEM lane quadrant this warp may access
    const int half = (warp - 2) >> 2;  // column half
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const int mt = t / n_tiles, nt = t % n_tiles;
      if (grp.tile_expert && expert_of(mt) < 0) continue;
      const int row = mt * kBM + q * 32 + lane;
      const uint32_t tb = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
      epilogue_tile<BN>(epi, tb, row, nt, half, &tfull[acc], acc_phase);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// tcgen05 persistent GEMM over a CTA pair (cluster of 2, cta_group::2):
// tile 256 x BN per pair; each CTA stages its 128 rows of A and BN/2 rows of
// B (half the per-SM operand traffic of the 1-CTA kernel at the same MMA
// rate), the leader CTA issues M=256 MMAs, each CTA drains its own 128-row
// half of the accumulator from its TMEM.
// ---------------------------------------------------------------------------
template <int BN, int STAGES, int EPI>  // EPI: specialised EpiMode (staged epilogue) or -1 (generic)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    tc2_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                    int N, int K, Epi epi, Grouped grp) {
  constexpr int PM = 2 * kBM;                    // pair tile rows
  constexpr uint32_t A_BYTES = kBM * kBK * 2;    // this CTA's 128 rows
  constexpr uint32_t B_BYTES = (BN / 2) * kBK * 2;  // this CTA's BN/2 rows
  constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);   // leader: its own expect_tx arrive; bytes from both CTAs
      mbar_init(&empty[s], 1);  // one multicast commit per use
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kEpiWarps);  // leader: epilogue warps of both CTAs
    }
    fence_mbar_init();
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_begin();  // as in tc_gemm_kernel: setup overlaps the previous kernel
  const int m_tiles = grp.n_mtiles ? *grp.n_mtiles : (M + PM - 1) / PM;  // grouped: tile_rows == 256
  const int n_tiles = (N + BN - 1) / BN;
  const int total = m_tiles * n_tiles;
  const int kblocks = (K + kBK - 1) / kBK;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_a = n_tiles > 1 ? l2_policy_evict_normal() : l2_policy_evict_first();
      const uint64_t pol_b = l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < total; t += npairs) {
        const int mt = t / n_tiles, nt = t % n_tiles;
        int brow = nt * BN;
        if (grp.tile_expert) {
          int e = grp.tile_expert[mt];
          if (e < 0) continue;
          brow += e * grp.b_rows_per_expert;
        }
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t fb = mapa_shared(&full[stage], 0);
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * STAGE_BYTES);
          tma_load_2d_pair(sA + stage * A_BYTES, &tmA, fb, kb * kBK, mt * PM + static_cast<int>(rank) * kBM, pol_a);
          tma_load_2d_pair(sB + stage * B_BYTES, &tmB, fb, kb * kBK, brow + static_cast<int>(rank) * (BN / 2), pol_b);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(PM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = pair; t < total; t += npairs) {
        if (grp.tile_expert && grp.tile_expert[t / n_tiles] < 0) continue;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            tc_mma_bf16_pair(d_tmem, umma_desc_sw128(a_base + k * 32), umma_desc_sw128(b_base + k * 32), idesc,
                             (kb | k) != 0);
          }
          tc_commit_pair(&empty[stage], 3);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit_pair(&tfull[acc], 3);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const uint32_t tempty_leader0 = mapa_shared(&tempty[0], 0), tempty_leader1 = mapa_shared(&tempty[1], 0);
    // 4 KB transpose tile per epilogue warp, after the barrier block
    float* stg = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256) + (warp - 2) * 1024;
    (void)stg;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = pair; t < total; t += npairs) {
      const int mt = t / n_tiles, nt = t % n_tiles;
      if (grp.tile_expert && grp.tile_expert[mt] < 0) continue;
      const int row = mt * PM + static_cast<int>(rank) * kBM + q * 32 + lane;
      const uint32_t tb = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
      if constexpr (EPI >= 0 && (EPI & EPI_SPLITVT) != 0) {
        if (nt * BN >= epi.vt_col0)
          epilogue_tile_vt<BN>(epi, tb, row, nt, half, &tfull[acc], acc_phase);
        else
          epilogue_tile_staged<BN, EPI & ~EPI_SPLITVT>(epi, stg, tb, row, nt, half, &tfull[acc], acc_phase);
      } else if constexpr (EPI == (EPI_SWIGLU | EPI_BF16))
        epilogue_tile_swiglu_staged<BN>(epi, stg, tb, row, nt, half, &tfull[acc], acc_phase);
      else if constexpr (EPI >= 0)
        epilogue_tile_staged<BN, EPI>(epi, stg, tb, row, nt, half, &tfull[acc], acc_phase);
      else
        epilogue_tile<BN>(epi, tb, row, nt, half, &tfull[acc], acc_phase);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// fp32 SIMT GEMM (parity mode): 64x64 tile, BK 16, 256 threads, 4x4 per thread
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) simt_gemm_kernel(const float* __restrict__ A, int lda,
                                                         const float* __restrict__ B, int ldb, int M, int N,
                                                         int K, Epi epi, Grouped grp) {
  pdl_begin();
  __shared__ float sA[16][64 + 4];
  __shared__ float sB[16][64 + 4];
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int tile_rows = grp.tile_rows ? grp.tile_rows : kBM;
  if (grp.n_mtiles && m0 >= *grp.n_mtiles * tile_rows) return;
  int boff = 0;
  if (grp.tile_expert) {
    int e = grp.tile_expert[m0 / tile_rows];
    if (e < 0) return;
    boff = e * grp.b_rows_per_expert;
  }
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 64 * 16; i += 256) {
      int r = i / 16, c = i % 16;
      int gm = m0 + r, gk = k0 + c;
      sA[c][r] = (gm < M && gk < K) ? A[(size_t)gm * lda + gk] : 0.f;
      int gn = n0 + r;
      sB[c][r] = (gn < N && gk < K) ? B[(size_t)(boff + gn) * ldb + gk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sA[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sB[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  // Generic scalar epilogue (swiglu handled via paired columns).
  for (int i = 0; i < 4; ++i) {
    int row = m0 + ty * 4 + i;
    if (row >= epi.m_valid || row >= M) continue;
    int orow = epi.row_map ? epi.row_map[row] : row;
    if (orow < 0) continue;
    float rs = epi.row_scale ? epi.row_scale[row] : 1.f;
    for (int j = 0; j < 4; ++j) {
      int col = n0 + tx * 4 + j;
      if (col >= N) continue;
      float x = acc[i][j];
      int oc;
      if (epi.swiglu) {
        continue;  // swiglu in fp32 mode uses gemm_f32 twice + swiglu_mul kernel (see engine)
      } else {
        oc = col;
        if (oc >= epi.n_out) continue;
        if (epi.bias) x += epi.bias[oc];
        x = act_apply(x, epi.act);
        x *= rs;
      }
      if (epi.resid) x += epi.resid[(size_t)(epi.resid_mod > 0 ? orow % epi.resid_mod : orow) * epi.ld_resid + oc];
      oc += epi.col_off;
      if (epi.out_bf16)
        reinterpret_cast<__nv_bfloat16*>(epi.out)[(size_t)orow * epi.ldo + oc] = __float2bfloat16_rn(x);
      else
        reinterpret_cast<float*>(epi.out)[(size_t)orow * epi.ldo + oc] = x;
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

CUtensorMap make_map_bf16(const void* ptr, int rows, int cols, int ld, int box_rows) {
  CUtensorMap m;
  cuuint64_t gdim[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t gstride[1] = {static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estride[2] = {1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), gdim, gstride, box,
                            estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ") rows=" +
                             std::to_string(rows) + " cols=" + std::to_string(cols) + " ld=" + std::to_string(ld));
  return m;
}

template <int BN, int STAGES>
void launch_tc(const void* A, int lda, const void* B, int ldb, int M, int N, int K, const Epi& epi,
               const Grouped* grp, cudaStream_t stream) {
  constexpr size_t smem = STAGES * (kBM * kBK * 2 + BN * kBK * 2) + 1024 + 256;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(tc_gemm_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    attr_set = true;
  }
  Grouped g = grp ? *grp : Grouped{};
  CUtensorMap ma = make_map_bf16(A, M, K, lda, kBM);
  const int b_rows = g.tile_expert ? g.n_groups * g.b_rows_per_expert : N;
  CUtensorMap mb = make_map_bf16(B, b_rows, K, ldb, BN);
  int tiles;
  if (g.n_mtiles) {
    tiles = num_sms();
  } else {
    tiles = ((M + kBM - 1) / kBM) * ((N + BN - 1) / BN);
    if (tiles > num_sms()) tiles = num_sms();
  }
  launch_pdl(tc_gemm_kernel<BN, STAGES>, tiles, kThreads, smem, stream, ma, mb, M, N, K, epi, g);
  ++launch_counter();
}

template <int BN, int STAGES, int EPI>
void launch_tc2(const void* A, int lda, const void* B, int ldb, int M, int N, int K, const Epi& epi,
                const Grouped* grp, cudaStream_t stream) {
  constexpr size_t smem = STAGES * (kBM * kBK * 2 + (BN / 2) * kBK * 2) + 1024 + 256 + (EPI >= 0 ? kEpiWarps * 4096 : 0);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(tc2_gemm_kernel<BN, STAGES, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    attr_set = true;
  }
  Grouped g = grp ? *grp : Grouped{};
  if (g.tile_expert && g.tile_rows != 2 * kBM)
    throw std::invalid_argument("gemm_bf16: grouped CTA-pair GEMM needs 256-row expert tiles");
  CUtensorMap ma = make_map_bf16(A, M, K, lda, kBM);
  const int b_rows = g.tile_expert ? g.n_groups * g.b_rows_per_expert : N;
  CUtensorMap mb = make_map_bf16(B, b_rows, K, ldb, BN / 2);
  const int max_pairs = num_sms() / 2;
  int pairs;
  if (g.n_mtiles) {
    pairs = max_pairs;
  } else {
    pairs = ((M + 2 * kBM - 1) / (2 * kBM)) * ((N + BN - 1) / BN);
    if (pairs > max_pairs) pairs = max_pairs;
  }
  launch_pdl(tc2_gemm_kernel<BN, STAGES, EPI>, 2 * pairs, kThreads, smem, stream, ma, mb, M, N, K, epi, g);
  ++launch_counter();
}

// BN=256 keeps 5 stages (6 without the 32 KB transpose tiles), BN=128 7 (8).
template <int BN>
void launch_tc2_mode(int staged, const void* A, int lda, const void* B, int ldb, int M, int N, int K,
                     const Epi& epi, const Grouped* grp, cudaStream_t stream) {
  constexpr int S = BN == 256 ? 5 : 7, SG = S + 1;
  switch (staged) {
    case 0: launch_tc2<BN, S, 0>(A, lda, B, ldb, M, N, K, epi, grp, stream); return;
    case EPI_RS: launch_tc2<BN, S, EPI_RS>(A, lda, B, ldb, M, N, K, epi, grp, stream); return;
    case EPI_RS | EPI_BF16: launch_tc2<BN, S, EPI_RS | EPI_BF16>(A, lda, B, ldb, M, N, K, epi, grp, stream); return;
    case EPI_RS | EPI_BF16 | EPI_PEER:
      launch_tc2<BN, S, EPI_RS | EPI_BF16 | EPI_PEER>(A, lda, B, ldb, M, N, K, epi, grp, stream);
      return;
    case EPI_RESID: launch_tc2<BN, S, EPI_RESID>(A, lda, B, ldb, M, N, K, epi, grp, stream); return;
    case EPI_BIAS | EPI_RESID: launch_tc2<BN, S, EPI_BIAS | EPI_RESID>(A, lda, B, ldb, M, N, K, epi, grp, stream); return;
    case EPI_BIAS | EPI_RESID | EPI_RMOD:
      launch_tc2<BN, S, EPI_BIAS | EPI_RESID | EPI_RMOD>(A, lda, B, ldb, M, N, K, epi, grp, stream);
      return;
    case EPI_BF16: launch_tc2<BN, S, EPI_BF16>(A, lda, B, ldb, M, N, K, epi, grp, stream); return;
    case EPI_BIAS | EPI_BF16: launch_tc2<BN, S, EPI_BIAS | EPI_BF16>(A, lda, B, ldb, M, N, K, epi, grp, stream); return;
    case EPI_BIAS | EPI_LEAKY | EPI_BF16:
      launch_tc2<BN, S, EPI_BIAS | EPI_LEAKY | EPI_BF16>(A, lda, B, ldb, M, N, K, epi, grp, stream);
      return;
    case EPI_BIAS | EPI_SILU | EPI_BF16:
      launch_tc2<BN, S, EPI_BIAS | EPI_SILU | EPI_BF16>(A, lda, B, ldb, M, N, K, epi, grp, stream);
      return;
    case EPI_RESID | EPI_XSSQ:
      if constexpr (BN == 256) {
        launch_tc2<BN, S, EPI_RESID | EPI_XSSQ>(A, lda, B, ldb, M, N, K, epi, grp, stream);
        return;
      }
      break;
    case EPI_XSSQ:
      if constexpr (BN == 256) {
        launch_tc2<BN, S, EPI_XSSQ>(A, lda, B, ldb, M, N, K, epi, grp, stream);
        return;
      }
      break;
    case EPI_BIAS | EPI_RESID | EPI_XSSQ:
      if constexpr (BN == 256) {
        launch_tc2<BN, S, EPI_BIAS | EPI_RESID | EPI_XSSQ>(A, lda, B, ldb, M, N, K, epi, grp, stream);
        return;
      }
      break;
    case EPI_BF16 | EPI_RSQ:
      if constexpr (BN == 256) {
        launch_tc2<BN, S, EPI_BF16 | EPI_RSQ>(A, lda, B, ldb, M, N, K, epi, grp, stream);
        return;
      }
      break;
    case EPI_BIAS | EPI_SILU | EPI_BF16 | EPI_RSQ:
      if constexpr (BN == 256) {
        launch_tc2<BN, S, EPI_BIAS | EPI_SILU | EPI_BF16 | EPI_RSQ>(A, lda, B, ldb, M, N, K, epi, grp, stream);
        return;
      }
      break;
    case EPI_SPLITVT | EPI_BF16 | EPI_RSQ:
      if constexpr (BN == 256) {
        launch_tc2<BN, S, EPI_SPLITVT | EPI_BF16 | EPI_RSQ>(A, lda, B, ldb, M, N, K, epi, grp, stream);
        return;
      }
      break;
    case EPI_STATS:
      if constexpr (BN == 256) {
        launch_tc2<BN, S, EPI_STATS>(A, lda, B, ldb, M, N, K, epi, grp, stream);
        return;
      }
      throw std::invalid_argument("gemm_bf16: head statistics need 256-wide tiles");
    case EPI_SPLITVT | EPI_BF16:
      if constexpr (BN == 256) {
        launch_tc2<BN, S, EPI_SPLITVT | EPI_BF16>(A, lda, B, ldb, M, N, K, epi, grp, stream);
        return;
      }
      launch_tc2<BN, SG, -1>(A, lda, B, ldb, M, N, K, epi, grp, stream);
      return;
    case EPI_SPLITVT | EPI_BF16 | EPI_BIAS:
      if constexpr (BN == 256) {
        launch_tc2<BN, S, EPI_SPLITVT | EPI_BF16 | EPI_BIAS>(A, lda, B, ldb, M, N, K, epi, grp, stream);
        return;
      }
      launch_tc2<BN, SG, -1>(A, lda, B, ldb, M, N, K, epi, grp, stream);
      return;
    case EPI_SWIGLU | EPI_BF16:
      if constexpr (BN == 256) {
        launch_tc2<BN, S, EPI_SWIGLU | EPI_BF16>(A, lda, B, ldb, M, N, K, epi, grp, stream);
        return;
      }
      [[fallthrough]];
    default: launch_tc2<BN, SG, -1>(A, lda, B, ldb, M, N, K, epi, grp, stream); return;
  }
  throw std::invalid_argument("gemm_bf16: epilogue mode needs 256-wide tiles");
}

}  // namespace

// Specialised epilogue mode of a launch (-1: generic path). Requires the
// output rows / bias to be 16-byte aligned per 32-column chunk.
int epi_mode(const Epi& e) {
  const bool plain = !e.bias && !e.act && !e.row_scale && !e.resid;
  // transposed V store: generic path (its per-column stores are already coalesced
  // across lanes; a SMEM-transposed variant measured slower)
  if (e.vt)  // split K|V GEMM: staged bf16 tiles below vt_col0, transposed tiles above (+ bias, row map)
    return !e.act && !e.row_scale && !e.resid && !e.swiglu && e.out_bf16 && e.vt_col0 > 0 && e.out &&
                   reinterpret_cast<uintptr_t>(e.out) % 16 == 0 && e.ldo % 8 == 0 && e.col_off == 0 &&
                   (!e.bias || reinterpret_cast<uintptr_t>(e.bias) % 16 == 0)
               ? EPI_SPLITVT | EPI_BF16 | (e.bias ? EPI_BIAS : 0) | (e.rsq ? EPI_RSQ : 0)
               : -1;
  if (e.stats)  // head GEMM: fp32 logits + chunk statistics, nothing else
    return plain && !e.swiglu && !e.row_map && !e.out_bf16 && e.col_off == 0 && e.out &&
                   reinterpret_cast<uintptr_t>(e.out) % 16 == 0 && e.ldo % 4 == 0
               ? EPI_STATS
               : -1;
  const int esz = e.out_bf16 ? 2 : 4;
  if ((reinterpret_cast<uintptr_t>(e.out) % 16) || ((long long)e.ldo * esz) % 16 || (e.col_off * esz) % 16) return -1;
  if (e.resid && ((reinterpret_cast<uintptr_t>(e.resid) % 16) || (e.ld_resid % 4))) return -1;
  if (e.bias && reinterpret_cast<uintptr_t>(e.bias) % 16) return -1;
  if (e.swiglu) return plain && e.out_bf16 ? EPI_SWIGLU | EPI_BF16 : -1;
  int m = 0;
  if (e.bias) m |= EPI_BIAS;
  if (e.act == ACT_LEAKY) m |= EPI_LEAKY;
  if (e.act == ACT_SILU) m |= EPI_SILU;
  if (e.row_scale) m |= EPI_RS;
  if (e.resid) m |= EPI_RESID;
  if (e.out_bf16) m |= EPI_BF16;
  if (e.out2) {
    if (!e.ssq || (reinterpret_cast<uintptr_t>(e.out2) % 16) || e.ldo2 % 8) return -1;
    m |= EPI_XSSQ;
  }
  if (e.rsq) m |= EPI_RSQ;
  if (e.peer_code) m |= EPI_PEER;
  if (e.resid && e.resid_mod > 0) m |= EPI_RMOD;
  switch (m) {
    case EPI_RS | EPI_BF16: case EPI_RS | EPI_BF16 | EPI_PEER: case EPI_BIAS | EPI_RESID | EPI_RMOD:
    case 0: case EPI_RS: case EPI_RESID: case EPI_BIAS | EPI_RESID: case EPI_BF16: case EPI_BIAS | EPI_BF16:
    case EPI_BIAS | EPI_LEAKY | EPI_BF16: case EPI_BIAS | EPI_SILU | EPI_BF16:
    case EPI_XSSQ: case EPI_RESID | EPI_XSSQ: case EPI_BIAS | EPI_RESID | EPI_XSSQ: case EPI_BF16 | EPI_RSQ:
    case EPI_BIAS | EPI_SILU | EPI_BF16 | EPI_RSQ:
      return m;
    default:
      return -1;
  }
}

bool& force_single_cta() {
  static bool f = getenv("ORX_GEMM_SINGLE_CTA") != nullptr;
  return f;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

long long& launch_counter() {
  static long long c = 0;
  return c;
}

long long launch_counter_value() { return launch_counter(); }

namespace {
struct ProfRec {
  int cat;
  cudaEvent_t a, b;
  double flops, bytes;
  std::string note;
};
struct Prof {
  bool on = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};
Prof& prof() {
  static Prof p;
  return p;
}
}  // namespace

ProfScope::ProfScope(int cat, cudaStream_t st, double flops, double bytes) : s(st) {
  Prof& p = prof();
  if (!p.on) return;
  ProfRec r{cat, p.get(), p.get(), flops, bytes, {}};
  cudaEventRecord(r.a, s);
  idx = static_cast<int>(p.recs.size());
  p.recs.push_back(r);
}
ProfScope::~ProfScope() {
  if (idx >= 0) cudaEventRecord(prof().recs[static_cast<size_t>(idx)].b, s);
}
void prof_enable(bool on) { prof().on = on; }
void prof_note(const std::string& note) {
  Prof& p = prof();
  if (p.on && !p.recs.empty()) p.recs.back().note = note;
}
void prof_note_launch(const char* expr) {
  Prof& p = prof();
  if (!p.on || p.recs.empty()) return;
  std::string e(expr);  // "launch_pdl(kernel<...>, grid, ..." -> "kernel<...>"
  size_t a = e.find('(');
  a = a == std::string::npos ? 0 : a + 1;
  size_t b = e.find(',', a);
  p.recs.back().note = e.substr(a, std::min<size_t>(b == std::string::npos ? e.size() : b, a + 60) - a);
}
bool prof_enabled() { return prof().on; }
void prof_collect(long long* count, double* ms, double* flops, double* bytes) {
  Prof& p = prof();
  for (int c = 0; c < PROF_N; ++c) count[c] = 0, ms[c] = flops[c] = bytes[c] = 0;
  for (auto& r : p.recs) {
    cudaEventSynchronize(r.b);
    float t = 0;
    cudaEventElapsedTime(&t, r.a, r.b);
    count[r.cat] += 1;
    ms[r.cat] += t;
    static const bool dump = getenv("ORX_PROF_DUMP") != nullptr;  // per-launch lines on stderr
    if (dump)
      fprintf(stderr, "prof cat=%d %s us=%.1f tflops=%.0f\n", r.cat, r.note.c_str(), t * 1e3,
              r.flops > 0 ? r.flops / (t * 1e-3) / 1e12 : 0.0);
    flops[r.cat] += r.flops;
    bytes[r.cat] += r.bytes;
    p.pool.push_back(r.a);
    p.pool.push_back(r.b);
  }
  p.recs.clear();
}

void gemm_bf16(const void* A, int lda, const void* B, int ldb, int M, int N, int K, const Epi& epi,
               const Grouped* grp, cudaStream_t stream) {
  if (M <= 0 || N <= 0) return;
  if (K % 8 != 0 || lda % 8 != 0 || ldb % 8 != 0)
    throw std::invalid_argument("gemm_bf16: K and row strides must be multiples of 8");
  if (epi.swiglu && N % 256 != 0) throw std::invalid_argument("gemm_bf16: swiglu needs N % 256 == 0");
  if (epi.vt && (epi.vt_cols % 32 != 0 || epi.col_off % 32 != 0 || epi.vt_col0 % 32 != 0))
    throw std::invalid_argument("gemm_bf16: transposed store needs 32-column aligned layers");
  ProfScope ps(grp && grp->tile_expert ? PROF_GEMM_MOE : PROF_GEMM, stream,
               2.0 * (grp && grp->tile_expert ? double(grp->algo_rows) : double(M)) * N * K, 0.0);
  Epi ep = epi;
  ep.mode = epi_mode(ep);
  if (prof_enabled())
    prof_note("gemm M=" + std::to_string(M) + " N=" + std::to_string(N) + " K=" + std::to_string(K) +
              " mode=" + std::to_string(ep.mode) + (grp && grp->tile_expert ? " grouped" : "") +
              (ep.swiglu ? " swiglu" : "") + (ep.vt ? " vt" : "") + (ep.row_map ? " row_map" : ""));
  const bool grouped = grp && grp->tile_expert;
  // head statistics (EPI_STATS) come from the CTA-pair kernel's staged epilogue only: any M
  const bool pair = grouped ? grp->tile_rows == 2 * kBM : ((M > kBM || epi.stats) && !force_single_cta());
  if (pair) {
    // BN=128 for small N, and where 256-wide tiles would leave a badly
    // filled last wave (e.g. M=16384, N=1024: 256 tiles on 74 pairs = 3.46
    // waves; 512 narrow tiles fill 6.92)
    bool small_n = N <= 128 && !epi.swiglu;
    if (!small_n && !epi.swiglu && !grouped && N % 128 == 0 && getenv("ORX_GEMM_BN_PICK")) {
      const int pairs = num_sms() / 2;
      const long long mt = (M + 2 * kBM - 1) / (2 * kBM);
      const long long t256 = mt * ((N + 255) / 256), t128 = mt * (N / 128);
      const double f256 = double(t256) / (double((t256 + pairs - 1) / pairs) * pairs);
      const double f128 = double(t128) / (double((t128 + pairs - 1) / pairs) * pairs);
      small_n = f128 > f256 + 0.08;
    }
    if (ep.stats) small_n = false;  // statistics are produced by the 256-wide staged epilogue only
    const int bn = small_n ? 128 : 256;
    // staged (coalesced) epilogue: specialised mode and every tile full
    const int staged = (ep.mode >= 0 && ep.n_out >= (ep.swiglu ? N / 2 : N) && N % bn == 0 &&
                        (!ep.vt || ep.vt_col0 % bn == 0))
                           ? ep.mode
                           : -1;
    if (ep.stats && staged != EPI_STATS)
      throw std::invalid_argument("gemm_bf16: head statistics need full, aligned 256-column tiles");
    if ((ep.out2 || ep.rsq) && (staged < 0 || small_n))
      throw std::invalid_argument("gemm_bf16: the folded RMSNorm needs the staged 256-wide epilogue");
    if (ep.row_rsq && staged != (EPI_SWIGLU | EPI_BF16))
      throw std::invalid_argument("gemm_bf16: per-row RMSNorm scales need the staged SwiGLU epilogue");
    if (ep.peer_code && staged < 0)
      throw std::invalid_argument("gemm_bf16: peer-scattered rows need the staged epilogue (full 128-column tiles)");
    if (small_n)
      launch_tc2_mode<128>(staged, A, lda, B, ldb, M, N, K, ep, grp, stream);
    else
      launch_tc2_mode<256>(staged, A, lda, B, ldb, M, N, K, ep, grp, stream);
  } else {
    if (ep.stats) throw std::invalid_argument("gemm_bf16: head statistics need the CTA-pair kernel (M > 128)");
    if (ep.out2 || ep.rsq) throw std::invalid_argument("gemm_bf16: the folded RMSNorm needs the CTA-pair kernel");
    if (ep.peer_code) throw std::invalid_argument("gemm_bf16: peer-scattered rows need the CTA-pair kernel");
    if (ep.row_rsq) throw std::invalid_argument("gemm_bf16: per-row RMSNorm scales need the CTA-pair kernel");
    // M <= 128 (decoder step 0): the GEMM is a weight stream; 64-wide tiles put
    // 4x more SMs on it than 256-wide ones (N=1024: 16 CTAs instead of 4)
    const bool narrow = !epi.swiglu && !grouped && N >= 512 && M <= kBM && !getenv("ORX_GEMM_NO_NARROW");
    if (narrow)
      launch_tc<64, 8>(A, lda, B, ldb, M, N, K, ep, grp, stream);
    else if (N <= 128 && !epi.swiglu)
      launch_tc<128, 6>(A, lda, B, ldb, M, N, K, ep, grp, stream);
    else
      launch_tc<256, 4>(A, lda, B, ldb, M, N, K, ep, grp, stream);
  }
}

void gemm_f32(const float* A, int lda, const float* B, int ldb, int M, int N, int K, const Epi& epi,
              const Grouped* grp, cudaStream_t stream) {
  if (M <= 0 || N <= 0) return;
  if (epi.swiglu) throw std::invalid_argument("gemm_f32: swiglu epilogue not supported");
  Grouped g = grp ? *grp : Grouped{};
  ProfScope ps(g.tile_expert ? PROF_GEMM_MOE : PROF_GEMM, stream,
               2.0 * (g.tile_expert ? double(g.algo_rows) : double(M)) * N * K, 0.0);
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  launch_pdl(simt_gemm_kernel, grid, 256, 0, stream, A, lda, B, ldb, M, N, K, epi, g);
  ++launch_counter();
}

}  // namespace orx
