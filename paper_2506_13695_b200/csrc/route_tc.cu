// MoE gate scores on the tensor pipe (bf16 engine): s = RMSNorm(h) . W_g with
// the RMSNorm gain folded into W_g, computed as 3xTF32 on tcgen05 so routing
// keeps fp32-grade scores (moe_forward, nn.cpp:117-147):
//   x = x_hi + x_lo, w = w_hi + w_lo (x_hi, w_hi tf32-exact, x_lo = x - x_hi)
//   x.w ~= x_hi.w_hi + x_lo.w_hi + x_hi.w_lo     (dropped term ~2^-21 relative)
// Split-K over two CTAs per 128-row tile (work item = tile x K half), two
// CTAs per SM: a single CTA walking all 32 K blocks of its tile was bound by
// the serial latency of its stage ring (23 us for the TMA / barrier skeleton
// alone at 16384 rows), so each half runs its 16 K blocks concurrently.
//   warp 0    TMA: h tile (128 rows x 32 fp32, 128-byte swizzled rows) and the
//             pre-split gate (32 expert rows x 32) per K block, 3-stage ring
//   warps 2-5 thread = row: split the staged fp32 row into tf32 hi (in place)
//             and lo (a 2-deep ring of its own), accumulate the row's partial
//             sum of squares; at the end of the half read the row's 32 partial
//             scores from TMEM and store them (with the partial sum) to a
//             scratch slot; the second CTA of the tile to finish (atomic
//             ticket) adds the other half's partials in a fixed order
//             (half 0 + half 1), scales by rsqrt(mean(x^2) + eps), and does
//             the stable top-k by score + bias (ties -> lower id,
//             nn.cpp:127-136), softmax over the selected raw scores
//             (nn.cpp:139-147), ids ascending
//   warp 1    one thread issues tcgen05.mma kind::tf32 (M=128, N=32, K=8), three
//             per K step (one TMEM accumulator per term), double-buffered
//             across work items
// The h tile is read once from HBM (4 d bytes per row); the per-row work is
// ~30 instructions per 32 columns.
#include <cfloat>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"
#include "gemm.cuh"
#include "kernels.cuh"

namespace orx {

namespace {

constexpr int kRtBM = 128;      // rows per tile
constexpr int kRtBK = 32;       // fp32 columns per K block (128-byte rows)
constexpr int kRtN = 32;        // expert slots (E <= 32)
constexpr int kRtStages = 3;
constexpr int kRtAcc = 3;                     // accumulators per work item (3 terms)
constexpr int kRtLo = 2;                      // lo ring depth
constexpr int kRtPart = 33;                   // partial scores (32) + partial sum of squares per row
constexpr uint32_t kRtA = kRtBM * kRtBK * 4;  // 16 KB
constexpr uint32_t kRtB = kRtN * kRtBK * 4;   // 4 KB
constexpr uint32_t kRtStage = kRtA + 2 * kRtB;  // A (hi in place) + B hi + B lo
constexpr size_t kRtSmem = kRtStages * kRtStage + kRtLo * kRtA + 1024 + 512;

// kind::tf32 instruction descriptor: fp32 accumulate, A/B tf32, both K-major
constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}
ORX_DEV void tc_mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
ORX_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__global__ void __launch_bounds__(192, 2)
    moe_route_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmBh,
                        const __grid_constant__ CUtensorMap tmBl, int rows, int d, int E, int k,
                        const float* __restrict__ bias, int32_t* __restrict__ sel, float* __restrict__ wts,
                        int32_t* __restrict__ counts, float* __restrict__ part, int32_t* __restrict__ ticket) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* lo_ring = smem + kRtStages * kRtStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(lo_ring + kRtLo * kRtA);
  uint64_t* conv = full + kRtStages;
  uint64_t* empty = conv + kRtStages;
  uint64_t* lo_empty = empty + kRtStages;   // [kRtLo]
  uint64_t* acc_full = lo_empty + kRtLo;    // [2]
  uint64_t* acc_empty = acc_full + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  int* hist = reinterpret_cast<int*>(tmem_slot + 4);  // [32]
  int* last_flag = hist + 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRtStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 4);
    }
    for (int a = 0; a < kRtLo; ++a) mbar_init(&lo_empty[a], 1);
    fence_mbar_init();
    tma_prefetch(&tmX);
    tma_prefetch(&tmBh);
    tma_prefetch(&tmBl);
  }
  if (threadIdx.x < 32) hist[threadIdx.x] = 0;
  if (warp == 1) tmem_alloc(tmem_slot, 256);  // 2 work items x 3 accumulators x 32 columns
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_begin();
  const int tiles = (rows + kRtBM - 1) / kRtBM;
  const int kblocks = d / kRtBK;
  const int items = 2 * tiles;  // (tile, K half)
  auto kb_begin = [&](int half) { return half ? kblocks / 2 : 0; };
  auto kb_end = [&](int half) { return half ? kblocks : kblocks / 2; };

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_x = l2_policy_evict_first(), pol_b = l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int w = blockIdx.x; w < items; w += gridDim.x) {
        const int t = w >> 1, k0 = kb_begin(w & 1), nk = kb_end(w & 1) - k0;
        for (int i = 0; i < nk; ++i) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * kRtStage;
          mbar_arrive_expect_tx(&full[stage], kRtA + 2 * kRtB);
          // K blocks in a per-CTA rotated order: in lockstep every CTA would read the
          // same 8 KB of the gate at the same time (one L2 hot spot for all readers)
          const int kr = k0 + (i + blockIdx.x) % nk;
          tma_load_2d(st, &tmX, &full[stage], kr * kRtBK, t * kRtBM, pol_x);
          tma_load_2d(st + kRtA, &tmBh, &full[stage], kr * kRtBK, 0, pol_b);
          tma_load_2d(st + kRtA + kRtB, &tmBl, &full[stage], kr * kRtBK, 0, pol_b);
          if (++stage == kRtStages) stage = 0, phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(kRtBM, kRtN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int lslot = 0;
      for (int w = blockIdx.x; w < items; w += gridDim.x) {
        const int nk = kb_end(w & 1) - kb_begin(w & 1);
        mbar_wait(&acc_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t dt = tmem + acc * kRtAcc * kRtN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          mbar_wait(&conv[stage], phase);
          tc_fence_after();
          const uint32_t ah = smem_u32(smem + stage * kRtStage), al = smem_u32(lo_ring + lslot * kRtA);
          const uint32_t bh = ah + kRtA, bl = bh + kRtB;
#pragma unroll
          for (int ks = 0; ks < kRtBK / 8; ++ks) {  // K = 8 tf32 = 32 bytes per step
            const uint32_t o = ks * 32;
            const uint32_t accum = kb > 0 || ks > 0;  // first use of each accumulator overwrites
            tc_mma_tf32(dt, umma_desc_sw128(ah + o), umma_desc_sw128(bh + o), idesc, accum);
            tc_mma_tf32(dt + kRtN, umma_desc_sw128(al + o), umma_desc_sw128(bh + o), idesc, accum);
            tc_mma_tf32(dt + 2 * kRtN, umma_desc_sw128(ah + o), umma_desc_sw128(bl + o), idesc, accum);
          }
          tc_commit(&empty[stage]);
          tc_commit(&lo_empty[lslot]);
          if (++stage == kRtStages) stage = 0, phase ^= 1;
          if (++lslot == kRtLo) lslot = 0;
        }
        tc_commit(&acc_full[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    const int q = warp & 3;   // TMEM lane quadrant = row block of the tile
    const int r = q * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int lslot = 0;
    uint32_t lphase = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x) {
      const int t = w >> 1, half = w & 1, nk = kb_end(half) - kb_begin(half);
      float ss = 0.f;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&full[stage], phase);
        mbar_wait(&lo_empty[lslot], lphase ^ 1);  // the MMAs of the lo buffer's previous use are done
        uint8_t* st = smem + stage * kRtStage;
        float4* hi = reinterpret_cast<float4*>(st + r * 128);
        float4* lo = reinterpret_cast<float4*>(lo_ring + lslot * kRtA + r * 128);
#pragma unroll
        for (int j = 0; j < 8; ++j) {  // the row's 8 16-byte units, elementwise: visit them XOR-rotated
          const int u = j ^ (r & 7);   // so the 8 lanes of a phase hit 8 different bank groups
          float4 x = hi[u];
          ss += x.x * x.x + x.y * x.y + x.z * x.z + x.w * x.w;
          float4 h4, l4;
          h4.x = __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
          h4.y = __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
          h4.z = __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
          h4.w = __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
          l4.x = x.x - h4.x, l4.y = x.y - h4.y, l4.z = x.z - h4.z, l4.w = x.w - h4.w;
          hi[u] = h4;
          lo[u] = l4;
        }
        fence_proxy_async_smem();  // generic-proxy writes -> the tensor core's reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[stage]);
        if (++stage == kRtStages) stage = 0, phase ^= 1;
        if (++lslot == kRtLo) lslot = 0, lphase ^= 1;
      }
      // epilogue: this row's expert scores
      mbar_wait(&acc_full[acc], acc_phase);
      __syncwarp();
      tc_fence_after();
      float sum[32];
#pragma unroll 1
      for (int a = 0; a < kRtAcc; ++a) {  // hi.hi, lo.hi, hi.lo
        uint32_t raw[32];
        tmem_ld32_async(tmem + lane_off + (acc * kRtAcc + a) * kRtN, raw);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) sum[e] = a == 0 ? __uint_as_float(raw[e]) : sum[e] + __uint_as_float(raw[e]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      // this half's partials into its scratch slot [item][33][128] (coalesced over rows)
      float* mine = part + (size_t)w * kRtPart * kRtBM + r;
#pragma unroll
      for (int e = 0; e < 32; ++e) mine[e * kRtBM] = sum[e];
      mine[32 * kRtBM] = ss;
      __threadfence();
      asm volatile("bar.sync 1, 128;" ::: "memory");  // the 4 epilogue warps
      if (threadIdx.x == 64) {
        const int old = atomicAdd(&ticket[t], 1);
        __threadfence();
        *last_flag = old;
        if (old == 1) ticket[t] = 0;  // both halves are in: reset for the next call
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (*last_flag == 0) continue;  // the other half finishes the tile
      const float* other = part + (size_t)(w ^ 1) * kRtPart * kRtBM + r;
      float tot[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {  // fixed order: K half 0 + K half 1
        const float o = __ldcg(other + e * kRtBM);
        tot[e] = half == 0 ? sum[e] + o : o + sum[e];
      }
      const float os = __ldcg(other + 32 * kRtBM);
      ss = half == 0 ? ss + os : os + ss;
      const int row = t * kRtBM + r;
      if (row >= rows) continue;
      const float inv = rsqrtf(ss / d + 1e-6f);
      float sc[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) sc[e] = tot[e] * inv;
      uint32_t taken = 0;
      int ids[8];
      float rw[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        ids[j] = 1 << 30;
        rw[j] = -FLT_MAX;
        if (j >= k) continue;
        int bi = -1;
        float bk = -FLT_MAX;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          if (e >= E || ((taken >> e) & 1u)) continue;
          const float key = sc[e] + __ldg(bias + e);
          if (bi < 0 || key > bk) bk = key, bi = e;  // strict >: ties keep the lower id
        }
        taken |= 1u << bi;
        ids[j] = bi;
      }
      // ids ascending, raw scores in that order (nn.cpp:139-147)
      int n = 0;
#pragma unroll
      for (int e = 0; e < 32; ++e)
        if ((taken >> e) & 1u) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j == n) ids[j] = e, rw[j] = sc[e];
          ++n;
        }
      float mx = -FLT_MAX;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < k) mx = fmaxf(mx, rw[j]);
      float den = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < k) den += __expf(rw[j] - mx);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < k) {
          sel[(size_t)row * k + j] = ids[j];
          wts[(size_t)row * k + j] = __expf(rw[j] - mx) / den;
          atomicAdd(&hist[ids[j]], 1);
        }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < E && hist[threadIdx.x]) atomicAdd(&counts[threadIdx.x], hist[threadIdx.x]);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

CUtensorMap map_f32(const void* ptr, long long rows, long long cols, long long ld, int box_rows) {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeFn>(p);
  }
  CUtensorMap m;
  cuuint64_t gdim[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t gstride[1] = {static_cast<cuuint64_t>(ld) * 4};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kRtBK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), gdim, gstride, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("route tensor map encode failed (" + std::to_string(int(r)) + ")");
  return m;
}

}  // namespace

bool moe_route_tc_supported(int d, int E, int k, int ldx) {
  return E <= kRtN && k >= 1 && k <= 8 && d % kRtBK == 0 && ldx % 4 == 0;
}

size_t moe_route_tc_scratch_floats(int max_rows) {
  return static_cast<size_t>(2) * ((max_rows + kRtBM - 1) / kRtBM) * kRtPart * kRtBM;
}
void launch_moe_route_tc(int rows, int d, int E, int k, const float* x, int ldx, const float* gate_hi,
                         const float* gate_lo, const float* bias, int32_t* sel, float* wts, int32_t* counts,
                         float* part, int32_t* ticket, cudaStream_t s) {
  if (rows <= 0) return;
  if (!moe_route_tc_supported(d, E, k, ldx)) throw std::invalid_argument("moe_route_tc: unsupported shape");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(moe_route_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kRtSmem));
    attr = true;
  }
  const CUtensorMap mx = map_f32(x, rows, d, ldx, kRtBM);
  const CUtensorMap mh = map_f32(gate_hi, kRtN, d, d, kRtN);
  const CUtensorMap ml = map_f32(gate_lo, kRtN, d, d, kRtN);
  const int tiles = (rows + kRtBM - 1) / kRtBM;
  const int grid = std::min(2 * tiles, 2 * num_sms());
  ProfScope ps(PROF_MOE_ROUTE, s, 2.0 * 3 * rows * d * kRtN, double(rows) * (4.0 * d + 8.0 * k));
  prof_note("moe_route_tc_kernel");
  launch_pdl(moe_route_tc_kernel, grid, 192, kRtSmem, s, mx, mh, ml, rows, d, E, k, bias, sel, wts, counts, part,
             ticket);
  ++launch_counter();
}

void gate_route4_layout(const float* gate, int E, int d, float* sw) {
  for (size_t i = 0; i < static_cast<size_t>(d) * 24; ++i) sw[i] = 0.f;
  for (int e = 0; e < E; ++e)
    for (int c = 0; c < d; ++c) {  // 4-column groups x 24 swizzled (4 experts x 1 column) units
      const int q = c >> 2, unit = ((c & 3) * 6 + (e >> 2)) ^ (q & 7);
      sw[(size_t)q * 96 + unit * 4 + (e & 3)] = gate[(size_t)e * d + c];
    }
}

void gate_tf32_split(const float* gate, int E, int d, float* hi, float* lo) {
  for (size_t i = 0; i < static_cast<size_t>(kRtN) * d; ++i) hi[i] = lo[i] = 0.f;
  for (size_t i = 0; i < static_cast<size_t>(E) * d; ++i) {
    uint32_t b;
    memcpy(&b, &gate[i], 4);
    b &= 0xFFFFE000u;  // tf32-exact part
    memcpy(&hi[i], &b, 4);
    lo[i] = gate[i] - hi[i];
  }
}

void debug_moe_route(int rows, int d, int E, int k, const float* x, const float* gate, const float* bias,
                     int variant, int32_t* sel, float* wts) {
  if (rows <= 0) return;
  if (variant < 0 || variant > 2) throw std::invalid_argument("debug_moe_route: variant 0, 1 or 2");
  if (variant == 1 && !(E <= 24 && d % 128 == 0)) throw std::invalid_argument("moe_route4 needs E <= 24, d % 128 == 0");
  if (variant == 2 && !moe_route_tc_supported(d, E, k, d)) throw std::invalid_argument("moe_route_tc: unsupported shape");
  std::vector<float> g2(static_cast<size_t>(kRtN) * d * 2);
  const size_t nx = static_cast<size_t>(rows) * d, ng = static_cast<size_t>(E) * d;
  float *dx, *dg, *dh, *dl, *dsw, *db, *dw;
  int32_t *ds, *dc;
  auto chk = [](cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("debug_moe_route: ") + cudaGetErrorString(e));
  };
  chk(cudaMalloc(&dx, nx * 4));
  chk(cudaMalloc(&dg, ng * 4));
  chk(cudaMalloc(&dh, g2.size() * 4));
  dl = dh + static_cast<size_t>(kRtN) * d;
  chk(cudaMalloc(&dsw, static_cast<size_t>(d) * 24 * 4));
  chk(cudaMalloc(&db, E * 4));
  chk(cudaMalloc(&ds, static_cast<size_t>(rows) * k * 4));
  chk(cudaMalloc(&dw, static_cast<size_t>(rows) * k * 4));
  chk(cudaMalloc(&dc, 32 * 4));
  chk(cudaMemcpy(dx, x, nx * 4, cudaMemcpyHostToDevice));
  chk(cudaMemcpy(dg, gate, ng * 4, cudaMemcpyHostToDevice));
  chk(cudaMemcpy(db, bias, E * 4, cudaMemcpyHostToDevice));
  chk(cudaMemset(dc, 0, 32 * 4));
  if (variant == 1) {
    std::vector<float> sw(static_cast<size_t>(d) * 24);
    gate_route4_layout(gate, E, d, sw.data());
    chk(cudaMemcpy(dsw, sw.data(), sw.size() * 4, cudaMemcpyHostToDevice));
  }
  if (variant == 2) {
    gate_tf32_split(gate, E, d, g2.data(), g2.data() + static_cast<size_t>(kRtN) * d);
    chk(cudaMemcpy(dh, g2.data(), g2.size() * 4, cudaMemcpyHostToDevice));
    float* part = nullptr;
    int32_t* ticket = nullptr;
    chk(cudaMalloc(&part, moe_route_tc_scratch_floats(rows) * 4));
    chk(cudaMalloc(&ticket, ((rows + kRtBM - 1) / kRtBM) * 4));
    chk(cudaMemset(ticket, 0, ((rows + kRtBM - 1) / kRtBM) * 4));
    launch_moe_route_tc(rows, d, E, k, dx, d, dh, dl, db, ds, dw, dc, part, ticket, 0);
    chk(cudaDeviceSynchronize());
    std::vector<int32_t> tk((rows + kRtBM - 1) / kRtBM);
    chk(cudaMemcpy(tk.data(), ticket, tk.size() * 4, cudaMemcpyDeviceToHost));
    for (int32_t v : tk)
      if (v != 0) throw std::runtime_error("moe_route_tc: tile tickets not reset");
    cudaFree(part);
    cudaFree(ticket);
  } else {
    launch_moe_route(rows, d, E, k, dx, d, nullptr, dg, dg, db, ds, dw, dc, 0, variant == 1 ? dsw : nullptr);
  }
  chk(cudaGetLastError());
  chk(cudaDeviceSynchronize());
  chk(cudaMemcpy(sel, ds, static_cast<size_t>(rows) * k * 4, cudaMemcpyDeviceToHost));
  chk(cudaMemcpy(wts, dw, static_cast<size_t>(rows) * k * 4, cudaMemcpyDeviceToHost));
  for (void* p : {static_cast<void*>(dx), static_cast<void*>(dg), static_cast<void*>(dh), static_cast<void*>(dsw),
                  static_cast<void*>(db), static_cast<void*>(ds), static_cast<void*>(dw), static_cast<void*>(dc)})
    cudaFree(p);
}

}  // namespace orx
