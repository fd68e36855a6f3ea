// Flash attention kernels for attention.cuh.
//   fp32: SIMT, 32 query rows x 32-key tiles per CTA (parity mode).
//   bf16: mma.sync m16n8k16 (bf16 -> fp32), 64 query rows per CTA (4 warps x
//         16 rows), 64-key tiles double-buffered with cp.async, online
//         softmax in registers, P reused as the A operand of P.V.
#include <cfloat>
#include <stdexcept>

#include "attention.cuh"
#include "common.cuh"
#include "gemm.cuh"

namespace orx {

namespace {

__device__ __forceinline__ int seg_start(const Seg& s, int b) { return s.start ? s.start[b] : b * s.stride; }
__device__ __forceinline__ int seg_len(const Seg& s, int b) { return s.len ? s.len[b] : s.fixed_len; }

// ---------------------------------------------------------------------------
// fp32 SIMT flash attention
// ---------------------------------------------------------------------------
template <int DH>
__global__ void __launch_bounds__(128) attn_f32_kernel(int heads, const float* __restrict__ Q, int ldq,
                                                        const float* __restrict__ K, int ldk,
                                                        const float* __restrict__ V, int ldv, float* __restrict__ O,
                                                        int ldo, Seg qs, Seg ks, Seg os) {
  pdl_begin();
  constexpr int BQ = 32, BKV = 32, PER = (DH + 31) / 32;
  extern __shared__ float smf[];
  float (*sQ)[DH] = reinterpret_cast<float (*)[DH]>(smf);
  float (*sK)[DH + 1] = reinterpret_cast<float (*)[DH + 1]>(smf + BQ * DH);
  float (*sV)[DH] = reinterpret_cast<float (*)[DH]>(smf + BQ * DH + BKV * (DH + 1));
  float (*sP)[BKV + 1] = reinterpret_cast<float (*)[BKV + 1]>(smf + BQ * DH + BKV * (DH + 1) + BKV * DH);
  const int b = blockIdx.z, h = blockIdx.y, q0 = blockIdx.x * BQ;
  const int qlen = seg_len(qs, b);
  if (q0 >= qlen) return;
  const int qst = seg_start(qs, b), kst = seg_start(ks, b), klen = seg_len(ks, b), ost = seg_start(os, b);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // warp ty owns rows ty*8..ty*8+7
  const float scale = rsqrtf(static_cast<float>(DH));
  for (int i = threadIdx.x; i < BQ * DH; i += 128) {
    int r = i / DH, c = i % DH;
    sQ[r][c] = (q0 + r < qlen) ? Q[(size_t)(qst + q0 + r) * ldq + h * DH + c] : 0.f;
  }
  float m[8], l[8], acc[8][PER];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    m[i] = -FLT_MAX;
    l[i] = 0.f;
#pragma unroll
    for (int p = 0; p < PER; ++p) acc[i][p] = 0.f;
  }
  for (int k0 = 0; k0 < klen; k0 += BKV) {
    __syncthreads();
    for (int i = threadIdx.x; i < BKV * DH; i += 128) {
      int r = i / DH, c = i % DH;
      bool ok = k0 + r < klen;
      sK[r][c] = ok ? K[(size_t)(kst + k0 + r) * ldk + h * DH + c] : 0.f;
      sV[r][c] = ok ? V[(size_t)(kst + k0 + r) * ldv + h * DH + c] : 0.f;
    }
    __syncthreads();
    const bool valid = k0 + tx < klen;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = ty * 8 + i;
      float s = 0.f;
#pragma unroll 8
      for (int c = 0; c < DH; ++c) s += sQ[r][c] * sK[tx][c];
      s = valid ? s * scale : -FLT_MAX;
      float mx = fmaxf(m[i], warp_max(s));
      float p = valid ? __expf(s - mx) : 0.f;
      float corr = __expf(m[i] - mx);
      l[i] = l[i] * corr + warp_sum(p);
      m[i] = mx;
#pragma unroll
      for (int q = 0; q < PER; ++q) acc[i][q] *= corr;
      sP[r][tx] = p;
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = ty * 8 + i;
      for (int j = 0; j < BKV; ++j) {
        float p = sP[r][j];
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          int c = tx + 32 * q;
          if (c < DH) acc[i][q] += p * sV[j][c];
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = q0 + ty * 8 + i;
    if (r >= qlen) continue;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      int c = tx + 32 * q;
      if (c < DH) O[(size_t)(ost + r) * ldo + h * DH + c] = acc[i][q] / l[i];
    }
  }
}

// ---------------------------------------------------------------------------
// bf16 mma.sync flash attention
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  uint32_t s = smem_u32(smem);
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int DH>
struct AttnSmem {
  static constexpr int BQ = 64, BKV = 64, LD = DH + 8;  // +16 B per row: conflict-free ldmatrix
  static constexpr int BYTES = (BQ * LD + 4 * BKV * LD) * 2;
};

template <int DH>
__global__ void __launch_bounds__(128) attn_bf16_kernel(int heads, const __nv_bfloat16* __restrict__ Q, int ldq,
                                                         const __nv_bfloat16* __restrict__ K, int ldk,
                                                         const __nv_bfloat16* __restrict__ V, int ldv,
                                                         __nv_bfloat16* __restrict__ O, int ldo, Seg qs, Seg ks,
                                                         Seg os) {
  pdl_begin();
  using S = AttnSmem<DH>;
  constexpr int BQ = S::BQ, BKV = S::BKV, LD = S::LD;
  constexpr int CH = DH / 8;  // 16-byte chunks per row
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sK = sQ + BQ * LD;        // [2][BKV][LD]
  __nv_bfloat16* sV = sK + 2 * BKV * LD;   // [2][BKV][LD]
  const int b = blockIdx.z, h = blockIdx.y, q0 = blockIdx.x * BQ;
  const int qlen = seg_len(qs, b);
  if (q0 >= qlen) return;
  const int qst = seg_start(qs, b), kst = seg_start(ks, b), klen = seg_len(ks, b), ost = seg_start(os, b);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (klen + BKV - 1) / BKV;

  for (int i = threadIdx.x; i < BQ * CH; i += 128) {
    int r = i / CH, c = (i % CH) * 8;
    bool ok = q0 + r < qlen;
    const __nv_bfloat16* src = Q + (size_t)(qst + (ok ? q0 + r : 0)) * ldq + h * DH + c;
    cp_async16(sQ + r * LD + c, src, ok);
  }
  auto load_kv = [&](int tile, int buf) {
    const int k0 = tile * BKV;
    for (int i = threadIdx.x; i < BKV * CH; i += 128) {
      int r = i / CH, c = (i % CH) * 8;
      bool ok = k0 + r < klen;
      size_t row = (size_t)(kst + (ok ? k0 + r : 0));
      cp_async16(sK + (buf * BKV + r) * LD + c, K + row * ldk + h * DH + c, ok);
      cp_async16(sV + (buf * BKV + r) * LD + c, V + row * ldv + h * DH + c, ok);
    }
  };
  load_kv(0, 0);
  cp_async_commit();

  const float scale_log2 = rsqrtf(static_cast<float>(DH)) * 1.4426950408889634f;
  float m_r[2] = {-FLT_MAX, -FLT_MAX}, l_r[2] = {0.f, 0.f};
  float o[DH / 8][4];
#pragma unroll
  for (int n = 0; n < DH / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  uint32_t qf[DH / 16][4];

  for (int t = 0; t < ntiles; ++t) {
    const int buf = t & 1;
    if (t + 1 < ntiles) load_kv(t + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (t == 0) {
#pragma unroll
      for (int kk = 0; kk < DH / 16; ++kk) {
        uint32_t addr = smem_u32(sQ + (warp * 16 + (lane & 15)) * LD + kk * 16 + (lane >> 4) * 8);
        ldsm_x4(addr, qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    // S = Q K^T : 16 x 64 per warp
    float s[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
    const __nv_bfloat16* kb = sK + buf * BKV * LD;
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {  // pairs of n-tiles (16 keys)
        int key = np * 16 + (lane & 7) + ((lane >> 4) << 3);
        int col = kk * 16 + ((lane >> 3) & 1) * 8;
        uint32_t r0, r1, r2, r3;
        ldsm_x4(smem_u32(kb + key * LD + col), r0, r1, r2, r3);
        mma_bf16(s[2 * np], qf[kk], r0, r1);
        mma_bf16(s[2 * np + 1], qf[kk], r2, r3);
      }
    }
    // mask + online softmax (rows lane/4 and lane/4+8)
    const int kbase = t * BKV;
    float mx[2] = {m_r[0], m_r[1]};
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      int c = kbase + n * 8 + 2 * (lane & 3);
      if (c >= klen) s[n][0] = s[n][2] = -FLT_MAX;
      if (c + 1 >= klen) s[n][1] = s[n][3] = -FLT_MAX;
      mx[0] = fmaxf(mx[0], fmaxf(s[n][0], s[n][1]));
      mx[1] = fmaxf(mx[1], fmaxf(s[n][2], s[n][3]));
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 1));
      mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 2));
    }
    float corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 2; ++i) corr[i] = exp2f((m_r[i] - mx[i]) * scale_log2);
    uint32_t pf[4][4];  // P as A fragments, 4 k-steps of 16 keys
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      float p0 = exp2f((s[n][0] - mx[0]) * scale_log2);
      float p1 = exp2f((s[n][1] - mx[0]) * scale_log2);
      float p2 = exp2f((s[n][2] - mx[1]) * scale_log2);
      float p3 = exp2f((s[n][3] - mx[1]) * scale_log2);
      rs[0] += p0 + p1;
      rs[1] += p2 + p3;
      pf[n >> 1][(n & 1) * 2 + 0] = pack_bf16(p0, p1);
      pf[n >> 1][(n & 1) * 2 + 1] = pack_bf16(p2, p3);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      rs[i] += __shfl_xor_sync(0xffffffffu, rs[i], 1);
      rs[i] += __shfl_xor_sync(0xffffffffu, rs[i], 2);
      l_r[i] = l_r[i] * corr[i] + rs[i];
      m_r[i] = mx[i];
    }
#pragma unroll
    for (int n = 0; n < DH / 8; ++n) {
      o[n][0] *= corr[0];
      o[n][1] *= corr[0];
      o[n][2] *= corr[1];
      o[n][3] *= corr[1];
    }
    // O += P V
    const __nv_bfloat16* vb = sV + buf * BKV * LD;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      // pf[kk] order must be {rows r k0-7, rows r+8 k0-7, rows r k8-15, rows r+8 k8-15}
      uint32_t a[4] = {pf[kk][0], pf[kk][1], pf[kk][2], pf[kk][3]};
#pragma unroll
      for (int np = 0; np < DH / 16; ++np) {
        int key = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        int col = np * 16 + (lane >> 4) * 8;
        uint32_t r0, r1, r2, r3;
        ldsm_x4_t(smem_u32(vb + key * LD + col), r0, r1, r2, r3);
        mma_bf16(o[2 * np], a, r0, r1);
        mma_bf16(o[2 * np + 1], a, r2, r3);
      }
    }
    __syncthreads();
  }
  // write O / l
  const float inv0 = 1.f / l_r[0], inv1 = 1.f / l_r[1];
  const int r0 = q0 + warp * 16 + (lane >> 2), r1 = r0 + 8;
#pragma unroll
  for (int n = 0; n < DH / 8; ++n) {
    int c = h * DH + n * 8 + 2 * (lane & 3);
    if (r0 < qlen)
      *reinterpret_cast<uint32_t*>(O + (size_t)(ost + r0) * ldo + c) = pack_bf16(o[n][0] * inv0, o[n][1] * inv0);
    if (r1 < qlen)
      *reinterpret_cast<uint32_t*>(O + (size_t)(ost + r1) * ldo + c) = pack_bf16(o[n][2] * inv1, o[n][3] * inv1);
  }
}

template <int DH>
void launch_f32(int B, int max_q, int heads, const float* Q, int ldq, const float* K, int ldk, const float* V, int ldv,
                float* O, int ldo, Seg q, Seg k, Seg o, cudaStream_t s) {
  constexpr int smem = (32 * DH + 32 * (DH + 1) + 32 * DH + 32 * 33) * 4;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(attn_f32_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    set = true;
  }
  dim3 grid((max_q + 31) / 32, heads, B);
  launch_pdl(attn_f32_kernel<DH>, grid, 128, smem, s, heads, Q, ldq, K, ldk, V, ldv, O, ldo, q, k, o);
}

template <int DH>
void launch_b16(int B, int max_q, int heads, const __nv_bfloat16* Q, int ldq, const __nv_bfloat16* K, int ldk,
                const __nv_bfloat16* V, int ldv, __nv_bfloat16* O, int ldo, Seg q, Seg k, Seg o, cudaStream_t s) {
  constexpr int smem = AttnSmem<DH>::BYTES;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(attn_bf16_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    set = true;
  }
  dim3 grid((max_q + 63) / 64, heads, B);
  launch_pdl(attn_bf16_kernel<DH>, grid, 128, smem, s, heads, Q, ldq, K, ldk, V, ldv, O, ldo, q, k, o);
}

}  // namespace

template <>
void launch_attention<float>(int B, int max_q, int heads, int dh, const float* Q, int ldq, const float* K, int ldk,
                             const float* V, int ldv, float* O, int ldo, Seg q, Seg k, Seg o, cudaStream_t s, double flops) {
  if (B <= 0 || max_q <= 0) return;
  ProfScope ps(PROF_ATTN, s, flops, 0.0);
  switch (dh) {
    case 8: launch_f32<8>(B, max_q, heads, Q, ldq, K, ldk, V, ldv, O, ldo, q, k, o, s); break;
    case 16: launch_f32<16>(B, max_q, heads, Q, ldq, K, ldk, V, ldv, O, ldo, q, k, o, s); break;
    case 32: launch_f32<32>(B, max_q, heads, Q, ldq, K, ldk, V, ldv, O, ldo, q, k, o, s); break;
    case 64: launch_f32<64>(B, max_q, heads, Q, ldq, K, ldk, V, ldv, O, ldo, q, k, o, s); break;
    case 128: launch_f32<128>(B, max_q, heads, Q, ldq, K, ldk, V, ldv, O, ldo, q, k, o, s); break;
    default: throw std::invalid_argument("attention: unsupported head dim " + std::to_string(dh));
  }
  ++launch_counter();
}

template <>
void launch_attention<__nv_bfloat16>(int B, int max_q, int heads, int dh, const __nv_bfloat16* Q, int ldq,
                                     const __nv_bfloat16* K, int ldk, const __nv_bfloat16* V, int ldv,
                                     __nv_bfloat16* O, int ldo, Seg q, Seg k, Seg o, cudaStream_t s, double flops) {
  if (B <= 0 || max_q <= 0) return;
  ProfScope ps(PROF_ATTN, s, flops, 0.0);
  switch (dh) {
    case 32: launch_b16<32>(B, max_q, heads, Q, ldq, K, ldk, V, ldv, O, ldo, q, k, o, s); break;
    case 64: launch_b16<64>(B, max_q, heads, Q, ldq, K, ldk, V, ldv, O, ldo, q, k, o, s); break;
    case 128: launch_b16<128>(B, max_q, heads, Q, ldq, K, ldk, V, ldv, O, ldo, q, k, o, s); break;
    default: throw std::invalid_argument("bf16 attention: unsupported head dim " + std::to_string(dh));
  }
  ++launch_counter();
}

}  // namespace orx
