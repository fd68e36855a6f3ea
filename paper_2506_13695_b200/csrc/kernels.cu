#include <algorithm>
#include <cfloat>
#include <stdexcept>

#include "common.cuh"
#include "gemm.cuh"
#include "kernels.cuh"

namespace orx {

namespace {

__device__ __forceinline__ int hashed(int64_t id, int vocab) {  // policy.cpp:14-17
  int64_t m = id % vocab;
  return static_cast<int>(m < 0 ? m + vocab : m);
}

// Feature row of one record (policy.cpp:139-198):
// [vid row | aid row | tag | ts | playtime | duration | label multi-hot . emb]
template <class T>
__global__ void features_kernel(RecordsDev r, FeatureTables t, T* __restrict__ out, int ldo) {
  pdl_begin();
  const int d = t.d, ad = t.aid_dim, mn = t.minor;
  const int F = t.vid_only ? d : d + ad + 5 * mn;
  for (int row = blockIdx.x; row < r.n; row += gridDim.x) {
    const int vid = t.use_sid ? 0 : r.vid[row];  // indices hashed at staging
    const int aid = r.aid[row];
    const float sc[4] = {r.tag[row], r.ts[row], r.play[row], r.dur[row]};
    const uint32_t lab = r.labels[row];
    T* o = out + (size_t)row * ldo;
    for (int c = threadIdx.x; c < ldo; c += blockDim.x) {
      float v = 0.f;
      if (c < d) {
        if (t.use_sid) {
          for (int l = 0; l < t.n_code_layers; ++l) v += t.tokens[l][(size_t)r.sid[(size_t)row * t.n_code_layers + l] * d + c];
        } else {
          v = t.vid[(size_t)vid * d + c];
        }
      } else if (c < F) {
        int cc = c - d;
        if (cc < ad) {
          v = t.aid[(size_t)aid * ad + cc];
        } else {
          cc -= ad;
          int f = cc / mn, j = cc % mn;
          if (f < 4) {
            const float* p = f == 0 ? t.tag : f == 1 ? t.ts : f == 2 ? t.play : t.dur;
            v = sc[f] * p[j] + p[mn + j];
          } else {
            for (int b = 0; b < t.n_flags; ++b)
              if ((lab >> b) & 1u) v += t.label[b * mn + j];
          }
        }
      }
      o[c] = from_f<T>(v);
    }
  }
}

// 4 / 8 consecutive elements of T <-> floats
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ld4(const __nv_bfloat16* p) {
  uint2 u = *reinterpret_cast<const uint2*>(p);
  float2 a = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.x));
  float2 b = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ void st4(__nv_bfloat16* p, float4 v) {
  uint2 u;
  u.x = pack_bf16(v.x, v.y);
  u.y = pack_bf16(v.z, v.w);
  *reinterpret_cast<uint2*>(p) = u;
}
__device__ __forceinline__ void st8(float* p, const float (&v)[8]) {
  st4(p, make_float4(v[0], v[1], v[2], v[3]));
  st4(p + 4, make_float4(v[4], v[5], v[6], v[7]));
}
__device__ __forceinline__ void st8(__nv_bfloat16* p, const float (&v)[8]) {
  uint4 u;
  u.x = pack_bf16(v[0], v[1]);
  u.y = pack_bf16(v[2], v[3]);
  u.z = pack_bf16(v[4], v[5]);
  u.w = pack_bf16(v[6], v[7]);
  *reinterpret_cast<uint4*>(p) = u;
}

// Vectorised feature rows (same layout as features_kernel): warp per record,
// lane per 8-column group; every section width is a multiple of 8 here.
template <class T>
__global__ void __launch_bounds__(256) features8_kernel(RecordsDev r, FeatureTables t, T* __restrict__ out, int ldo) {
  pdl_begin();
  const int d = t.d, ad = t.aid_dim, mn = t.minor;
  const int F = t.vid_only ? d : d + ad + 5 * mn;
  const int lane = threadIdx.x & 31;
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < r.n; row += gridDim.x * (blockDim.x >> 5)) {
    const int vid = t.use_sid ? 0 : r.vid[row];  // indices hashed at staging
    const int aid = r.aid[row];
    const float sc[4] = {r.tag[row], r.ts[row], r.play[row], r.dur[row]};
    const uint32_t lab = r.labels[row];
    T* o = out + (size_t)row * ldo;
#pragma unroll 3
    for (int c0 = lane * 8; c0 < ldo; c0 += 256) {
      float v[8];
      if (c0 < d) {
        if (t.use_sid) {
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = 0.f;
          for (int l = 0; l < t.n_code_layers; ++l) {
            const float* src = t.tokens[l] + (size_t)r.sid[(size_t)row * t.n_code_layers + l] * d + c0;
            float4 a = ld4(src), b = ld4(src + 4);
            v[0] += a.x, v[1] += a.y, v[2] += a.z, v[3] += a.w, v[4] += b.x, v[5] += b.y, v[6] += b.z, v[7] += b.w;
          }
        } else {
          const float* src = t.vid + (size_t)vid * d + c0;
          float4 a = ld4(src), b = ld4(src + 4);
          v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
        }
      } else if (c0 < F) {
        int cc = c0 - d;
        if (cc < ad) {
          const float* src = t.aid + (size_t)aid * ad + cc;
          float4 a = ld4(src), b = ld4(src + 4);
          v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
        } else {
          cc -= ad;
          const int f = cc / mn, j0 = cc % mn;
          if (f < 4) {  // scalar feature x * w + b, (2 x minor) table (policy.cpp:175-188)
            const float* p = f == 0 ? t.tag : f == 1 ? t.ts : f == 2 ? t.play : t.dur;
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = sc[f] * p[j0 + j] + p[mn + j0 + j];
          } else {  // label multi-hot . (5 x minor) (policy.cpp:190-195)
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = 0.f;
            for (int b = 0; b < t.n_flags; ++b)
              if ((lab >> b) & 1u) {
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] += t.label[b * mn + j0 + j];
              }
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = 0.f;
      }
      st8(o + c0, v);
    }
  }
}

// bf16 engine, vid_only = 0, no sid history: warp per record, every lane first
// issues all of its 16-byte loads (vid / aid rows from the bf16 tables), then
// computes the scalar / label sections and stores (memory-level parallelism).
constexpr int kFeatMaxChunks = 12;  // ldo <= 3072
constexpr int kFeatBatch = 4;       // 16-byte loads in flight per lane
__global__ void __launch_bounds__(256, 4) features16_kernel(RecordsDev r, FeatureTables t,
                                                            __nv_bfloat16* __restrict__ out, int ldo) {
  pdl_begin();
  const int d = t.d, ad = t.aid_dim, mn = t.minor;
  const int F = d + ad + 5 * mn;
  const int lane = threadIdx.x & 31;
  // the minor-feature tables (4 x [2][mn] + [n_flags][mn] fp32) in shared
  // memory: read as float4 per 8-column chunk instead of scalar L1 loads
  extern __shared__ float4 sm4[];
  float* smt = reinterpret_cast<float*>(sm4);
  const int nt = 8 * mn + t.n_flags * mn;
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    const int f = i / (2 * mn), j = i - f * 2 * mn;
    smt[i] = f < 4 ? (f == 0 ? t.tag : f == 1 ? t.ts : f == 2 ? t.play : t.dur)[j] : t.label[i - 8 * mn];
  }
  __syncthreads();
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < r.n; row += gridDim.x * (blockDim.x >> 5)) {
    const int vid = r.vid[row];  // indices hashed at staging
    const int aid = r.aid[row];
    const __nv_bfloat16* vrow = t.vid16 + (size_t)vid * d;
    const __nv_bfloat16* arow = t.aid16 + (size_t)aid * ad;
    __nv_bfloat16* o = out + (size_t)row * ldo;
    for (int k0 = 0; k0 < kFeatMaxChunks; k0 += kFeatBatch) {
      if ((lane + 32 * k0) * 8 >= ldo) break;
      uint4 g[kFeatBatch];
#pragma unroll
      for (int k = 0; k < kFeatBatch; ++k) {
        const int c0 = (lane + 32 * (k0 + k)) * 8;
        if (c0 < d) g[k] = __ldg(reinterpret_cast<const uint4*>(vrow + c0));
        else if (c0 < d + ad) g[k] = __ldg(reinterpret_cast<const uint4*>(arow + (c0 - d)));
      }
#pragma unroll
      for (int k = 0; k < kFeatBatch; ++k) {
        const int c0 = (lane + 32 * (k0 + k)) * 8;
        if (c0 >= ldo) break;
        uint4 w = g[k];
        if (c0 >= d + ad) {
          float v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = 0.f;
          if (c0 < F) {
            const int cc = c0 - d - ad, f = cc / mn, j0 = cc % mn;
            if (f < 4) {  // x * w + b (policy.cpp:175-188)
              const float x = f == 0 ? r.tag[row] : f == 1 ? r.ts[row] : f == 2 ? r.play[row] : r.dur[row];
              const float4* w4 = reinterpret_cast<const float4*>(smt + f * 2 * mn + j0);
              const float4* b4 = reinterpret_cast<const float4*>(smt + f * 2 * mn + mn + j0);
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const float4 w = w4[h], b = b4[h];
                v[4 * h] = x * w.x + b.x, v[4 * h + 1] = x * w.y + b.y;
                v[4 * h + 2] = x * w.z + b.z, v[4 * h + 3] = x * w.w + b.w;
              }
            } else {  // labels multi-hot . (5 x minor) (policy.cpp:190-195)
              const uint32_t lab = r.labels[row];
              for (int b = 0; b < t.n_flags; ++b)
                if ((lab >> b) & 1u) {
                  const float4* l4 = reinterpret_cast<const float4*>(smt + 8 * mn + b * mn + j0);
#pragma unroll
                  for (int h = 0; h < 2; ++h) {
                    const float4 w = l4[h];
                    v[4 * h] += w.x, v[4 * h + 1] += w.y, v[4 * h + 2] += w.z, v[4 * h + 3] += w.w;
                  }
                }
            }
          }
          w = make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
        }
        *reinterpret_cast<uint4*>(o + c0) = w;
      }
    }
  }
}

// Folded pathway first layer: G warps per record, each owning 256 columns
// (two float4 per lane, 16-byte lane stride); the u vectors stay in registers
// across the rows a warp visits, the Pv / Pa / Pl rows (L2-resident per
// pathway) are gathered as float4. Replaces features16 + the fc1 GEMM
// (n x 2.125d x d) per pathway.
constexpr int kFoldMaxD4 = 512;  // d <= 2048
template <int G, bool PAL>
__global__ void __launch_bounds__(256, 3) fold_features_kernel(RecordsDev r, FoldTables f,
                                                               __nv_bfloat16* __restrict__ out, int ldo) {
  // the 4 scalar-section vectors in shared memory, not registers: 3 blocks per
  // SM instead of 2 (the kernel is bound by the latency of its gathers)
  __shared__ float4 su[4][kFoldMaxD4];
  pdl_begin();
  constexpr int RPB = 8 / G;  // records in flight per block
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d4 = f.d / 4, cg = warp % G, rl = warp / G;
  const unsigned lmask = (1u << f.n_flags) - 1u;
  for (int i = threadIdx.x; i < 4 * d4; i += blockDim.x)
    su[i / d4][i % d4] = __ldg(reinterpret_cast<const float4*>(f.u) + i);
  __syncthreads();
  int c4[2];
  bool ok[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    c4[h] = cg * 64 + h * 32 + lane;
    ok[h] = c4[h] < d4;
  }
  // Software-pipelined over this warp's records: the record fields of row k+2
  // and the table rows of row k+1 are in flight while row k is finished (the
  // loop is otherwise two dependent memory latencies per record).
  const int stride = gridDim.x * RPB;
  struct Rec {
    int vid, aid;
    unsigned lab;
    float x0, x1, x2, x3;
  };
  auto load_rec = [&](int row, Rec& q) {
    if (row < r.n) {
      q.vid = r.vid[row];
      q.aid = r.aid[row];
      q.lab = r.labels[row] & lmask;
      q.x0 = r.tag[row];
      q.x1 = r.ts[row];
      q.x2 = r.play[row];
      q.x3 = r.dur[row];
    }
  };
  auto gather = [&](int row, const Rec& q, float4 (&a)[2], float4 (&b)[2], float4 (&l)[2]) {
    if (row >= r.n) return;
    const float4* pv = reinterpret_cast<const float4*>(f.pv) + (size_t)q.vid * d4;
    if constexpr (PAL) {  // aid and label rows pre-added: two gathers per record
      const float4* pb = reinterpret_cast<const float4*>(f.pal) + ((size_t)q.aid << f.n_flags | q.lab) * d4;
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (ok[h]) a[h] = __ldg(pv + c4[h]), b[h] = __ldg(pb + c4[h]);
    } else {
      const float4* pa = reinterpret_cast<const float4*>(f.pa) + (size_t)q.aid * d4;
      const float4* pl = reinterpret_cast<const float4*>(f.pl) + (size_t)q.lab * d4;
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (ok[h]) a[h] = __ldg(pv + c4[h]), b[h] = __ldg(pa + c4[h]), l[h] = __ldg(pl + c4[h]);
    }
  };
  int row = blockIdx.x * RPB + rl;
  Rec q0{}, q1{}, q2{};
  float4 a0[2], b0[2], l0[2], a1[2], b1[2], l1[2];
  load_rec(row, q0);
  load_rec(row + stride, q1);
  gather(row, q0, a0, b0, l0);
  for (; row < r.n; row += stride) {
    load_rec(row + 2 * stride, q2);
    gather(row + stride, q1, a1, b1, l1);
    const float x0 = q0.x0, x1 = q0.x1, x2 = q0.x2, x3 = q0.x3;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!ok[h]) continue;
      float v[4];
      const float4 u0 = su[0][c4[h]], u1 = su[1][c4[h]], u2 = su[2][c4[h]], u3 = su[3][c4[h]];
      if constexpr (PAL) l0[h] = make_float4(-0.f, -0.f, -0.f, -0.f);  // x + -0 == x: folds away
      v[0] = a0[h].x + b0[h].x + l0[h].x + x0 * u0.x + x1 * u1.x + x2 * u2.x + x3 * u3.x;
      v[1] = a0[h].y + b0[h].y + l0[h].y + x0 * u0.y + x1 * u1.y + x2 * u2.y + x3 * u3.y;
      v[2] = a0[h].z + b0[h].z + l0[h].z + x0 * u0.z + x1 * u1.z + x2 * u2.z + x3 * u3.z;
      v[3] = a0[h].w + b0[h].w + l0[h].w + x0 * u0.w + x1 * u1.w + x2 * u2.w + x3 * u3.w;
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = v[j] > 0.f ? v[j] : 0.01f * v[j];  // tape.hpp:88
      *reinterpret_cast<uint2*>(out + (size_t)row * ldo + c4[h] * 4) = make_uint2(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]));
    }
    q0 = q1;
    q1 = q2;
#pragma unroll
    for (int h = 0; h < 2; ++h) a0[h] = a1[h], b0[h] = b1[h], l0[h] = l1[h];
  }
}

__global__ void fold_pal_kernel(int naid, int n_flags, int d, const float* __restrict__ pa,
                                const float* __restrict__ pl, float* __restrict__ pal) {
  const long long n = (long long)naid << n_flags;
  for (long long i = blockIdx.x; i < n; i += gridDim.x) {
    const long long a = i >> n_flags, m = i & ((1 << n_flags) - 1);
    for (int j = threadIdx.x; j < d; j += blockDim.x) pal[i * d + j] = pa[a * d + j] + pl[m * d + j];
  }
}

template <class T>
__global__ void static_features_kernel(int U, const int32_t* uid, const int32_t* gender, const int32_t* age,
                                       const float* ue, const float* ge, const float* ae, int sd, int uv, int gv,
                                       int av, T* out, int ldo) {
  pdl_begin();
  int u = blockIdx.x;
  if (u >= U) return;
  int iu = hashed(uid[u], uv), ig = hashed(gender[u], gv), ia = hashed(age[u], av);
  for (int c = threadIdx.x; c < ldo; c += blockDim.x) {
    float v = 0.f;
    if (c < sd) v = ue[(size_t)iu * sd + c];
    else if (c < 2 * sd) v = ge[(size_t)ig * sd + c - sd];
    else if (c < 3 * sd) v = ae[(size_t)ia * sd + c - 2 * sd];
    out[(size_t)u * ldo + c] = from_f<T>(v);
  }
}

__global__ void z_init_kernel(int U, int T, int d, const float* pos, const float* pad_s, const float* pad_p,
                              const int32_t* n_s, const int32_t* n_p, int Ls, int Lp, float* z) {
  pdl_begin();
  size_t row = blockIdx.x;
  int u = static_cast<int>(row / T), t = static_cast<int>(row % T);
  const float* pad = nullptr;
  if (t >= 1 && t < 1 + Ls) {
    if (t - 1 < Ls - n_s[u]) pad = pad_s;
  } else if (t >= 1 + Ls && t < 1 + Ls + Lp) {
    if (t - 1 - Ls < Lp - n_p[u]) pad = pad_p;
  }
  // every other row (static, records, QFormer queries) is written by a GEMM
  // whose residual operand is the position table itself (engine pos_resid)
  if (!pad) return;
  if (d % 4 == 0) {  // float4 path (the callers' buffers are 16-byte aligned)
    const float4* p4 = reinterpret_cast<const float4*>(pos + (size_t)t * d);
    const float4* q4 = reinterpret_cast<const float4*>(pad);
    float4* z4 = reinterpret_cast<float4*>(z + row * d);
    for (int c = threadIdx.x; c < d / 4; c += blockDim.x) {
      float4 v = __ldg(p4 + c);
      if (pad) {
        const float4 w = __ldg(q4 + c);
        v.x += w.x, v.y += w.y, v.z += w.z, v.w += w.w;
      }
      z4[c] = v;
    }
    return;
  }
  for (int c = threadIdx.x; c < d; c += blockDim.x) z[row * d + c] = pos[(size_t)t * d + c] + (pad ? pad[c] : 0.f);
}

// RMSNorm, warp per row (tape.cpp:462-503, eps 1e-6 nn.hpp:36).
template <class T>
__global__ void rmsnorm_kernel(int rows, int d, const float* __restrict__ x, int ldx, const float* __restrict__ g,
                               T* __restrict__ out, int ldo) {
  pdl_begin();
  int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (row >= rows) return;
  const float* xr = x + (size_t)row * ldx;
  float ss = 0.f;
  for (int c = lane; c < d; c += 32) ss += xr[c] * xr[c];
  ss = warp_sum(ss);
  float r = rsqrtf(ss / d + 1e-6f);
  T* o = out + (size_t)row * ldo;
  for (int c = lane; c < d; c += 32) o[c] = from_f<T>(xr[c] * r * g[c]);
}

// Vectorised variant: cols % 4 == 0, rows 16-byte aligned; thread per 4 elements.
template <class T>
__global__ void convert4_kernel(int rows, int cols, const float* __restrict__ x, int ldx, T* __restrict__ out,
                                int ldo) {
  pdl_begin();
  const int q = cols / 4;
  const long long n = (long long)rows * q;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(i / q), c = static_cast<int>(i % q) * 4;
    st4(out + (size_t)r * ldo + c, __ldg(reinterpret_cast<const float4*>(x + (size_t)r * ldx + c)));
  }
}

template <class T>
__global__ void convert_kernel(int rows, int cols, const float* x, int ldx, T* out, int ldo) {
  pdl_begin();
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t n = (size_t)rows * cols;
  for (; i < n; i += (size_t)gridDim.x * blockDim.x) {
    size_t r = i / cols, c = i % cols;
    out[r * ldo + c] = from_f<T>(x[r * ldx + c]);
  }
}

template <class T>
__global__ void fill_rows_kernel(int rows, int cols, const float* src, T* out, int ldo, const int32_t* idx) {
  pdl_begin();
  int r = blockIdx.x;
  if (r >= rows) return;
  int orow = idx ? idx[r] : r;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) out[(size_t)orow * ldo + c] = from_f<T>(src[c]);
}

__global__ void dec_embed_kernel(int rows, int d, const float* table, const int32_t* code, int code_stride,
                                 float* h) {
  pdl_begin();
  int r = blockIdx.x;
  if (r >= rows) return;
  size_t src = code ? (size_t)code[(size_t)r * code_stride] * d : 0;
  if (d % 4 == 0) {
    const float4* t4 = reinterpret_cast<const float4*>(table + src);
    float4* h4 = reinterpret_cast<float4*>(h + (size_t)r * d);
    for (int c = threadIdx.x; c < d / 4; c += blockDim.x) h4[c] = __ldg(t4 + c);
    return;
  }
  for (int c = threadIdx.x; c < d; c += blockDim.x) h[(size_t)r * d + c] = table[src + c];
}

// dec_embed + the first decoder layer's RMSNorm in one pass (bf16 engine,
// d = 128 * NC): warp per row, the embedding row in registers.
template <int NC>
__global__ void __launch_bounds__(256) dec_embed_norm_kernel(int rows, int d, const float* __restrict__ table,
                                                             const int32_t* __restrict__ code, int code_stride,
                                                             float* __restrict__ h, const float* __restrict__ gain,
                                                             __nv_bfloat16* __restrict__ out) {
  pdl_begin();
  const int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (r >= rows) return;
  const float4* t4 = reinterpret_cast<const float4*>(table + (code ? (size_t)code[(size_t)r * code_stride] * d : 0));
  float4 v[NC];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    v[i] = __ldg(t4 + lane + 32 * i);
    ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
  }
  float4* h4 = reinterpret_cast<float4*>(h + (size_t)r * d);
#pragma unroll
  for (int i = 0; i < NC; ++i) h4[lane + 32 * i] = v[i];
  ss = warp_sum(ss);
  const float rs = rsqrtf(ss / d + 1e-6f);
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int c = (lane + 32 * i) * 4;
    const float4 g = __ldg(reinterpret_cast<const float4*>(gain + c));
    *reinterpret_cast<uint2*>(out + (size_t)r * d + c) =
        make_uint2(pack_bf16(v[i].x * rs * g.x, v[i].y * rs * g.y), pack_bf16(v[i].z * rs * g.z, v[i].w * rs * g.w));
  }
}

// K / V of position p < step for a row: the K|V columns of that position's
// QKV GEMM output (kv[p * L + layer], [rows_p][3d]) at the ancestor row.
template <class T>
__device__ __forceinline__ const T* kv_at(T* const* kv, int p, int L, int layer, int row, int d) {
  return kv[p * L + layer] + (size_t)row * 3 * d + d;
}

// Warp per (row, head): keys are positions 0..step; position p < step is read
// from that position's QKV output at row anc[r][p], position `step` is the
// row's own K/V (this step's QKV output stays in place as its cache entry).
template <class T>
__global__ void dec_self_attn_kernel(int rows, int d, int heads, int step, int layer, int L, const T* __restrict__ qkv,
                                     T* const* __restrict__ kv, const int32_t* __restrict__ anc, int anc_stride,
                                     T* __restrict__ out) {
  pdl_begin();
  int gw = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
  int r = gw / heads, h = gw % heads;
  if (r >= rows) return;
  const int dh = d / heads;
  const T* q = qkv + (size_t)r * 3 * d + h * dh;
  const T* kown = q + d;
  const T* vown = q + 2 * d;
  const float scale = rsqrtf(static_cast<float>(dh));
  float sc[8];
  float mx = -FLT_MAX;
  for (int p = 0; p <= step; ++p) {
    const T* k = p == step ? kown : kv_at(kv, p, L, layer, anc[(size_t)r * anc_stride + p], d) + h * dh;
    float s = 0.f;
    for (int c = lane; c < dh; c += 32) s += to_f(q[c]) * to_f(k[c]);
    s = warp_sum(s) * scale;
    sc[p] = s;
    mx = fmaxf(mx, s);
  }
  float den = 0.f;
  for (int p = 0; p <= step; ++p) {
    sc[p] = __expf(sc[p] - mx);
    den += sc[p];
  }
  for (int c = lane; c < dh; c += 32) {
    float acc = 0.f;
    for (int p = 0; p <= step; ++p) {
      const T* v = p == step ? vown : kv_at(kv, p, L, layer, anc[(size_t)r * anc_stride + p], d) + d + h * dh;
      acc += sc[p] * to_f(v[c]);
    }
    out[(size_t)r * d + h * dh + c] = from_f<T>(acc / den);
  }
}

// Vectorised variant (dh % 4 == 0, dh <= 128): lane owns 4 consecutive
// head dims; same math and order of operations as dec_self_attn_kernel.
template <class T>
__global__ void __launch_bounds__(256) dec_self_attn4_kernel(int rows, int d, int heads, int step, int layer, int L,
                                                             const T* __restrict__ qkv, T* const* __restrict__ kv,
                                                             const int32_t* __restrict__ anc, int anc_stride,
                                                             T* __restrict__ out) {
  pdl_begin();
  const int gw = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
  const int r = gw / heads, h = gw % heads;
  if (r >= rows) return;
  const int dh = d / heads;
  const bool on = lane * 4 < dh;
  const int c = on ? lane * 4 : 0;
  const T* q = qkv + (size_t)r * 3 * d + h * dh;
  const float4 q4 = ld4(q + c);
  const float4 k4 = ld4(q + d + c);
  const float4 v4 = ld4(q + 2 * d + c);
  const float scale = rsqrtf(static_cast<float>(dh));
  float sc[8];
  float mx = -FLT_MAX;
  for (int p = 0; p <= step; ++p) {
    float4 kk = k4;
    if (p < step) kk = ld4(kv_at(kv, p, L, layer, anc[(size_t)r * anc_stride + p], d) + h * dh + c);
    float s = on ? q4.x * kk.x + q4.y * kk.y + q4.z * kk.z + q4.w * kk.w : 0.f;
    s = warp_sum(s) * scale;
    sc[p] = s;
    mx = fmaxf(mx, s);
  }
  float den = 0.f;
  for (int p = 0; p <= step; ++p) {
    sc[p] = __expf(sc[p] - mx);
    den += sc[p];
  }
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int p = 0; p <= step; ++p) {
    float4 vv = v4;
    if (p < step) vv = ld4(kv_at(kv, p, L, layer, anc[(size_t)r * anc_stride + p], d) + d + h * dh + c);
    acc.x += sc[p] * vv.x, acc.y += sc[p] * vv.y, acc.z += sc[p] * vv.z, acc.w += sc[p] * vv.w;
  }
  if (on) {
    const float inv = 1.f / den;
    st4(out + (size_t)r * d + h * dh + c, make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv));
  }
}

// four consecutive expert-output elements (fp32, or bf16 in the bf16 engine)
__device__ __forceinline__ float4 ldy4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 ldy4(const __nv_bfloat16* p) {
  const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

// h[r] += sum_j (ascending expert) y[slot[r][j]], float4 per thread (d % 4 == 0).
template <class YT>
__global__ void __launch_bounds__(256) moe_combine4_kernel(int rows, int k, int d, const YT* __restrict__ yg,
                                                           const int32_t* __restrict__ slot, float* __restrict__ h,
                                                           int ldh, int32_t* __restrict__ zero, int nzero) {
  pdl_begin();
  if (blockIdx.x == 0 && threadIdx.x < nzero) zero[threadIdx.x] = 0;  // routing counters, for the next MoE layer
  const int q = d / 4;
  const long long n = (long long)rows * q;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(i / q), c = static_cast<int>(i % q) * 4;
    float4 acc = ldy4(yg + (size_t)slot[(size_t)r * k] * d + c);
    for (int j = 1; j < k; ++j) {
      const float4 y = ldy4(yg + (size_t)slot[(size_t)r * k + j] * d + c);
      acc.x += y.x, acc.y += y.y, acc.z += y.z, acc.w += y.w;
    }
    float4* hp = reinterpret_cast<float4*>(h + (size_t)r * ldh + c);
    float4 hv = *hp;
    hv.x += acc.x, hv.y += acc.y, hv.z += acc.z, hv.w += acc.w;
    *hp = hv;
  }
}

// Gate scores, top-k (stable: score+bias desc, ties -> lower id), selected ids
// ascending, softmax over selected raw scores (nn.cpp:121-147). The gate input
// RMSNorm(x) is recomputed here in fp32 from the fp32 residual stream so that
// routing decisions do not see bf16 rounding. Gate matrix staged in smem;
// warp per row (grid-stride), lane e owns expert e (E <= 32).
constexpr int kRouteMaxPer = 64;  // d <= 2048
__device__ __forceinline__ void moe_route_row(int r, int d, int E, int k, const float* __restrict__ xr,
                                              const float* __restrict__ gain, const float* __restrict__ sg,
                                              const float* __restrict__ bias, int32_t* __restrict__ sel,
                                              float* __restrict__ wts, int32_t* __restrict__ counts, int lane) {
  float xv[kRouteMaxPer];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < kRouteMaxPer; ++i) {
    int c = lane + 32 * i;
    xv[i] = c < d ? xr[c] : 0.f;
    ss += xv[i] * xv[i];
  }
  ss = warp_sum(ss);
  const float rr = rsqrtf(ss / d + 1e-6f);
#pragma unroll
  for (int i = 0; i < kRouteMaxPer; ++i) {
    int c = lane + 32 * i;
    if (c < d) xv[i] = xv[i] * rr * gain[c];
  }
  float my = -FLT_MAX;  // lane e's raw score
  for (int e = 0; e < E; ++e) {
    const float* g = sg + (size_t)e * d;
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < kRouteMaxPer; ++i) {
      int c = lane + 32 * i;
      if (c < d) s += xv[i] * g[c];
    }
    s = warp_sum(s);
    if (lane == e) my = s;
  }
  float key = lane < E ? my + bias[lane] : -FLT_MAX;
  bool taken = false;
  uint32_t chosen = 0;
  for (int j = 0; j < k; ++j) {
    float v = taken ? -FLT_MAX : key;
    int idx = lane < E && !taken ? lane : 1 << 30;
    for (int o = 16; o > 0; o >>= 1) {
      float v2 = __shfl_xor_sync(0xffffffffu, v, o);
      int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
      if (v2 > v || (v2 == v && i2 < idx)) {
        v = v2;
        idx = i2;
      }
    }
    if (lane == idx) taken = true;
    chosen |= 1u << idx;
  }
  float mx = -FLT_MAX;
  for (int e = 0; e < E; ++e)
    if (chosen >> e & 1u) mx = fmaxf(mx, __shfl_sync(0xffffffffu, my, e));
  float den = 0.f;
  for (int e = 0; e < E; ++e)
    if (chosen >> e & 1u) den += __expf(__shfl_sync(0xffffffffu, my, e) - mx);
  if (lane < E && (chosen >> lane & 1u)) {
    int j = __popc(chosen & ((1u << lane) - 1u));
    sel[(size_t)r * k + j] = lane;
    wts[(size_t)r * k + j] = __expf(my - mx) / den;
    atomicAdd(&counts[lane], 1);
  }
}

__global__ void __launch_bounds__(256) moe_route_kernel(int rows, int d, int E, int k, const float* __restrict__ x,
                                                        int ldx, const float* __restrict__ gain,
                                                        const float* __restrict__ gate_t,
                                                        const float* __restrict__ bias, int32_t* __restrict__ sel,
                                                        float* __restrict__ wts, int32_t* __restrict__ counts) {
  pdl_begin();
  extern __shared__ float sg[];  // [E][d]
  for (int i = threadIdx.x; i < E * d; i += blockDim.x) sg[i] = gate_t[i];
  __syncthreads();
  const int lane = threadIdx.x % 32, wpb = blockDim.x / 32;
  for (int r = blockIdx.x * wpb + threadIdx.x / 32; r < rows; r += gridDim.x * wpb)
    moe_route_row(r, d, E, k, x + (size_t)r * ldx, gain, sg, bias, sel, wts, counts, lane);
}

// Routing v2 (d % 4 == 0): warp per 2 rows, lane owns columns {128 i + 4 lane ..+3};
// the gate is pre-multiplied by the RMSNorm gain (gg[e][c] = gain[c] * W_g[c][e])
// so score_e = rsqrt(mean(x^2) + eps) * sum_c x_c gg[e][c] = RMSNorm(x) . W_g[:, e]
// (nn.cpp:117-120). 64 partial sums per lane (2 rows x 32 expert slots) are
// reduce-scattered with a 5-level butterfly (lane l ends with slots 2l, 2l+1),
// then selection runs with lane = expert as above. Per-expert counts go
// through a block histogram (one global atomic per expert per block).
constexpr int kRoutePerWarp = 2;
__device__ __forceinline__ void butterfly64(float (&v)[64], int lane) {
#pragma unroll
  for (int lvl = 0; lvl < 5; ++lvl) {
    const int o = 16 >> lvl;
    const int h = 32 >> lvl;
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const float send = up ? v[i] : v[i + h];
      const float keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
}

__global__ void __launch_bounds__(256, 2) moe_route2_kernel(int rows, int d, int E, int k, const float* __restrict__ x,
                                                            int ldx, const float* __restrict__ gg,
                                                            const float* __restrict__ bias, int32_t* __restrict__ sel,
                                                            float* __restrict__ wts, int32_t* __restrict__ counts) {
  pdl_begin();
  extern __shared__ float sg[];  // [E][d]
  __shared__ int hist[32];
  for (int i = threadIdx.x; i < E * d / 4; i += blockDim.x)
    reinterpret_cast<float4*>(sg)[i] = reinterpret_cast<const float4*>(gg)[i];
  if (threadIdx.x < 32) hist[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
  const float bias_l = lane < E ? bias[lane] : 0.f;
  for (int r0 = (blockIdx.x * wpb + (threadIdx.x >> 5)) * kRoutePerWarp; r0 < rows;
       r0 += gridDim.x * wpb * kRoutePerWarp) {
    float p[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) p[i] = 0.f;
    float ss0 = 0.f, ss1 = 0.f;
    const bool has1 = r0 + 1 < rows;
    const float* x0 = x + (size_t)r0 * ldx;
    const float* x1 = x + (size_t)(has1 ? r0 + 1 : r0) * ldx;
    for (int c = lane * 4; c < d; c += 128) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(x0 + c));
      float4 b = __ldg(reinterpret_cast<const float4*>(x1 + c));
      if (!has1) b = make_float4(0.f, 0.f, 0.f, 0.f);
      ss0 += a.x * a.x + a.y * a.y + a.z * a.z + a.w * a.w;
      ss1 += b.x * b.x + b.y * b.y + b.z * b.z + b.w * b.w;
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        if (e < E) {
          const float4 g = *reinterpret_cast<const float4*>(sg + (size_t)e * d + c);
          p[e] += a.x * g.x + a.y * g.y + a.z * g.z + a.w * g.w;
          p[32 + e] += b.x * g.x + b.y * g.y + b.z * g.z + b.w * g.w;
        }
      }
    }
    butterfly64(p, lane);
    ss0 = warp_sum(ss0);
    ss1 = warp_sum(ss1);
#pragma unroll
    for (int rr = 0; rr < kRoutePerWarp; ++rr) {
      const int r = r0 + rr;
      if (r >= rows) break;
      const float inv = rsqrtf((rr ? ss1 : ss0) / d + 1e-6f);
      // slot (rr, e) lives in lane rr*16 + e/2, element e&1
      const float v0 = __shfl_sync(0xffffffffu, p[0], rr * 16 + (lane >> 1));
      const float v1 = __shfl_sync(0xffffffffu, p[1], rr * 16 + (lane >> 1));
      const float my = ((lane & 1) ? v1 : v0) * inv;  // raw gate score of expert `lane`
      const float key = lane < E ? my + bias_l : -FLT_MAX;
      bool taken = false;
      uint32_t chosen = 0;
      for (int j = 0; j < k; ++j) {  // stable top-k: (score + bias) desc, ties -> lower id (nn.cpp:127-136)
        float v = taken ? -FLT_MAX : key;
        int idx = lane < E && !taken ? lane : 1 << 30;
        for (int o = 16; o > 0; o >>= 1) {
          float v2 = __shfl_xor_sync(0xffffffffu, v, o);
          int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
          if (v2 > v || (v2 == v && i2 < idx)) {
            v = v2;
            idx = i2;
          }
        }
        if (lane == idx) taken = true;
        chosen |= 1u << idx;
      }
      // softmax over the selected raw scores (nn.cpp:139-147); ids ascending
      float mx = -FLT_MAX;
      for (int e = 0; e < E; ++e)
        if (chosen >> e & 1u) mx = fmaxf(mx, __shfl_sync(0xffffffffu, my, e));
      float den = 0.f;
      for (int e = 0; e < E; ++e)
        if (chosen >> e & 1u) den += __expf(__shfl_sync(0xffffffffu, my, e) - mx);
      if (lane < E && (chosen >> lane & 1u)) {
        const int j = __popc(chosen & ((1u << lane) - 1u));
        sel[(size_t)r * k + j] = lane;
        wts[(size_t)r * k + j] = __expf(my - mx) / den;
        atomicAdd(&hist[lane], 1);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < E && hist[threadIdx.x]) atomicAdd(&counts[threadIdx.x], hist[threadIdx.x]);
}

// Routing v4 (E <= 24, k <= 8, d % 128 == 0): warp per 4 rows. Lane owns
// columns {128 i + 4 lane .. +3}. The gain-folded gate sits in shared memory
// as 16-byte units (g_e.c .. g_e+3.c) of one column and 4 experts, 24 units per
// 4-column group, XOR-swizzled by the group index (conflict-free LDS.128):
// one unit feeds 2 packed FFMA2 (expert pairs x the row's x_c broadcast) per
// row, so every gate load serves 4 rows with no operand shuffling. The 96
// partial sums (4 rows x 24 expert slots) are reduce-scattered with a 5-level
// butterfly: lane l ends with row (l >> 3) & 3, experts 3 (l & 7) .. +2, so each
// row's selection runs in one 8-lane group (stable top-k by score + bias,
// ties -> lower id, nn.cpp:127-136; softmax over the selected raw scores,
// nn.cpp:139-147; ids ascending).
constexpr int kRoute4Rows = 4;
__global__ void __launch_bounds__(256, 1) moe_route4_kernel(int rows, int d, int E, int k, const float* __restrict__ x,
                                                            int ldx, const float* __restrict__ gsw,
                                                            const float* __restrict__ bias, int32_t* __restrict__ sel,
                                                            float* __restrict__ wts, int32_t* __restrict__ counts) {
  extern __shared__ float sg[];  // [d / 4 groups][24 units][4], pre-swizzled by the engine (gsw)
  __shared__ int hist[32];
  // The gate is a weight: staged before griddepcontrol.wait (overlaps the
  // previous kernel's tail), 8 independent 16-byte loads in flight per thread.
  {
    const int n4 = 24 * d / 4;
    float4* s4 = reinterpret_cast<float4*>(sg);
    const float4* g4 = reinterpret_cast<const float4*>(gsw);
    for (int i0 = threadIdx.x; i0 < n4; i0 += 8 * blockDim.x) {
      float4 t[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = i0 + j * blockDim.x;
        if (i < n4) t[j] = __ldg(g4 + i);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (i0 + j * blockDim.x < n4) s4[i0 + j * blockDim.x] = t[j];
    }
  }
  if (threadIdx.x < 32) hist[threadIdx.x] = 0;
  pdl_begin();
  __syncthreads();
  const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
  const int grp = (lane >> 3) & 3, sub = lane & 7;
  float bias3[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const int e = 3 * sub + j;
    bias3[j] = e < E ? bias[e] : 0.f;
  }
  const float4* sg4 = reinterpret_cast<const float4*>(sg);
  // x streams as one flat sequence of (row group, 128-column block) steps per
  // warp, two steps of loads in flight across row-group boundaries
  const int gstride = gridDim.x * wpb;
  const int nb = d >> 7;
  int pg = blockIdx.x * wpb + (threadIdx.x >> 5), pi = 0;  // next step to load
  float4 an[2][4];
  auto load_step = [&](float4 (&dst)[4]) {
    if (pg * kRoute4Rows < rows) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
        dst[r] = __ldg(reinterpret_cast<const float4*>(x + (size_t)min(pg * kRoute4Rows + r, rows - 1) * ldx +
                                                       pi * 128 + lane * 4));
    }
    if (++pi == nb) {
      pi = 0;
      pg += gstride;
      const int rn = pg * kRoute4Rows + gstride * kRoute4Rows + (lane & 3);  // the group after, into L2
      if (lane < 4 && rn < rows)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x + (size_t)rn * ldx), "r"(d * 4) : "memory");
    }
  };
  load_step(an[0]);
  load_step(an[1]);
  for (int r0 = (blockIdx.x * wpb + (threadIdx.x >> 5)) * kRoute4Rows; r0 < rows; r0 += gstride * kRoute4Rows) {
    float2 acc[4][12];  // [row][expert pair]
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int p = 0; p < 12; ++p) acc[r][p] = make_float2(0.f, 0.f);
    float ss[4] = {0.f, 0.f, 0.f, 0.f};
    for (int c = lane * 4; c < d; c += 128) {
      float4 a[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        a[r] = an[0][r];
        an[0][r] = an[1][r];
      }
      load_step(an[1]);
#pragma unroll
      for (int r = 0; r < 4; ++r)
        ss[r] += a[r].x * a[r].x + a[r].y * a[r].y + a[r].z * a[r].z + a[r].w * a[r].w;
      const int q = c >> 2;
      const float4* gq = sg4 + (size_t)q * 24;
#pragma unroll
      for (int cl = 0; cl < 4; ++cl) {
#pragma unroll
        for (int u = 0; u < 6; ++u) {
          const float4 g = gq[(cl * 6 + u) ^ (lane & 7)];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const float xc = cl == 0 ? a[r].x : cl == 1 ? a[r].y : cl == 2 ? a[r].z : a[r].w;
            acc[r][2 * u] = ffma2(make_float2(g.x, g.y), make_float2(xc, xc), acc[r][2 * u]);
            acc[r][2 * u + 1] = ffma2(make_float2(g.z, g.w), make_float2(xc, xc), acc[r][2 * u + 1]);
          }
        }
      }
    }
    // flat v[r * 24 + e]
    float v[96];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int p = 0; p < 12; ++p) {
        v[r * 24 + 2 * p] = acc[r][p].x;
        v[r * 24 + 2 * p + 1] = acc[r][p].y;
      }
#pragma unroll
    for (int lvl = 0; lvl < 5; ++lvl) {
      const int o = 16 >> lvl;
      const int h = 48 >> lvl;
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < h; ++i) {
        const float send = up ? v[i] : v[i + h];
        const float keep = up ? v[i + h] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) ss[r] = warp_sum(ss[r]);
    const int r = r0 + grp;
    const float my_ss = grp == 0 ? ss[0] : grp == 1 ? ss[1] : grp == 2 ? ss[2] : ss[3];
    const float inv = rsqrtf(my_ss / d + 1e-6f);
    float sc[3], key[3];
    bool taken[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      sc[j] = v[j] * inv;
      key[j] = 3 * sub + j < E ? sc[j] + bias3[j] : -FLT_MAX;
      taken[j] = 3 * sub + j >= E;
    }
    int ids[8];
    float raw[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      ids[t] = 1 << 30;
      raw[t] = -FLT_MAX;
      if (t >= k) continue;
      float bk = -FLT_MAX, bs = 0.f;
      int bi = 1 << 30;
#pragma unroll
      for (int j = 0; j < 3; ++j)
        if (!taken[j] && (key[j] > bk || bi == (1 << 30))) {
          bk = key[j];
          bs = sc[j];
          bi = 3 * sub + j;
        }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {  // within the 8-lane group
        const float k2 = __shfl_xor_sync(0xffffffffu, bk, o);
        const float s2 = __shfl_xor_sync(0xffffffffu, bs, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        if (k2 > bk || (k2 == bk && i2 < bi)) {
          bk = k2;
          bs = s2;
          bi = i2;
        }
      }
#pragma unroll
      for (int j = 0; j < 3; ++j)
        if (3 * sub + j == bi) taken[j] = true;
      ids[t] = bi;
      raw[t] = bs;
    }
    // ids ascending (odd-even transposition network; unused slots hold 1 << 30)
#pragma unroll
    for (int pass = 0; pass < 8; ++pass)
#pragma unroll
      for (int a2 = pass & 1; a2 + 1 < 8; a2 += 2)
        if (ids[a2] > ids[a2 + 1]) {
          const int ti = ids[a2];
          ids[a2] = ids[a2 + 1];
          ids[a2 + 1] = ti;
          const float tr = raw[a2];
          raw[a2] = raw[a2 + 1];
          raw[a2 + 1] = tr;
        }
    float mx = -FLT_MAX;
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (t < k) mx = fmaxf(mx, raw[t]);
    float den = 0.f;
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (t < k) den += __expf(raw[t] - mx);
    if (r < rows && sub < k) {
      float rt = raw[0];
      int it = ids[0];
#pragma unroll
      for (int t = 1; t < 8; ++t)
        if (t == sub) rt = raw[t], it = ids[t];
      sel[(size_t)r * k + sub] = it;
      wts[(size_t)r * k + sub] = __expf(rt - mx) / den;
      atomicAdd(&hist[it], 1);
    }
  }
  __syncthreads();
  if (threadIdx.x < E && hist[threadIdx.x]) atomicAdd(&counts[threadIdx.x], hist[threadIdx.x]);
}

// Segment offsets padded to the GEMM expert tile (128 rows, 256 for the CTA-pair kernel); tile -> expert table.
// The grouped-GEMM plan inside the scatter (no separate launch): every CTA
// derives the expert segments (padded to the tile) from the final routing
// histogram, CTA 0 also writes the tile -> expert table; a pair's slot is its
// expert's segment start + an atomic on the zeroed per-expert fill counter.
__device__ __forceinline__ void moe_plan_block(const MoePlan& p, int* seg0) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int nt = lane < p.E ? (p.counts[lane] + p.tile_rows - 1) / p.tile_rows : 0;
    int incl = nt;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    seg0[lane] = incl - nt;  // first tile of expert `lane`
    if (lane == 31) seg0[32] = min(incl, p.max_tiles);
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    const int total = seg0[32];
    if (threadIdx.x == 0) *p.n_mtiles = total;
    for (int i = threadIdx.x; i < p.max_tiles; i += blockDim.x) {
      int e = -1;
      if (i < total)
        for (int x = 0; x < p.E; ++x)
          if (i >= seg0[x]) e = x;
      p.tile_expert[i] = e;
    }
  }
}

template <class T>
__global__ void moe_scatter_kernel(int rows, int k, int d, const T* __restrict__ x, int ldx,
                                   const int32_t* __restrict__ sel, const float* __restrict__ wts, MoePlan plan,
                                   int32_t* __restrict__ slot, T* __restrict__ xg, float* __restrict__ row_scale) {
  __shared__ int seg0[33];
  pdl_begin();
  moe_plan_block(plan, seg0);
  int gw = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (gw >= rows * k) return;
  int r = gw / k;
  int e = sel[gw];
  int s = 0;
  if (lane == 0) s = seg0[e] * plan.tile_rows + atomicAdd(&plan.fill[e], 1);
  s = __shfl_sync(0xffffffffu, s, 0);
  if (lane == 0) {
    slot[gw] = s;
    row_scale[s] = wts[gw];
    if (plan.row_rsq) {
      float ss = 0.f;
      for (int i = 0; i < plan.ssq_n; ++i) ss += plan.ssq[(long long)i * plan.ssq_ld + r];
      plan.row_rsq[s] = rsqrtf(ss * plan.inv_d + 1e-6f);
    }
  }
  const T* src = x + (size_t)r * ldx;
  T* dst = xg + (size_t)s * d;
  if (sizeof(T) == 2 && d % 8 == 0) {
    for (int c = lane * 8; c < d; c += 256) *reinterpret_cast<uint4*>(dst + c) = *reinterpret_cast<const uint4*>(src + c);
  } else {
    for (int c = lane; c < d; c += 32) dst[c] = src[c];
  }
}

// Same permutation with warp-aggregated slot allocation: a warp takes 32
// (row, expert) pairs, lanes routed to the same expert share one atomic
// (hot experts take a large share of the tokens under random-init routing),
// then the warp copies the 32 rows with 16-byte accesses (bf16, d % 8 == 0).
__global__ void __launch_bounds__(256) moe_scatter32_kernel(int rows, int k, int d, const __nv_bfloat16* __restrict__ x,
                                                            int ldx, const int32_t* __restrict__ sel,
                                                            const float* __restrict__ wts, MoePlan plan,
                                                            int32_t* __restrict__ slot, __nv_bfloat16* __restrict__ xg,
                                                            float* __restrict__ row_scale) {
  __shared__ int seg0[33];
  pdl_begin();
  moe_plan_block(plan, seg0);
  const int lane = threadIdx.x & 31;
  const int base_pair = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32;
  const int n_pairs = rows * k;
  if (base_pair >= n_pairs) return;
  const int gw = base_pair + lane;
  const bool on = gw < n_pairs;
  const int e = on ? sel[gw] : -1;
  const unsigned act = __ballot_sync(0xffffffffu, on);
  const unsigned peers = __match_any_sync(0xffffffffu, e);
  const int leader = __ffs(peers) - 1;
  int base = 0;
  if (on && lane == leader) base = seg0[e] * plan.tile_rows + atomicAdd(&plan.fill[e], __popc(peers));
  base = __shfl_sync(0xffffffffu, base, leader);
  const int my_slot = base + __popc(peers & ((1u << lane) - 1u));
  if (on) {
    slot[gw] = my_slot;
    row_scale[my_slot] = wts[gw];
    if (plan.row_rsq) {
      const int r = gw / k;
      float ss = 0.f;
      for (int i = 0; i < plan.ssq_n; ++i) ss += plan.ssq[(long long)i * plan.ssq_ld + r];
      plan.row_rsq[my_slot] = rsqrtf(ss * plan.inv_d + 1e-6f);
    }
  }
  for (int i = 0; i < 32; ++i) {
    if (!((act >> i) & 1u)) break;
    const int s = __shfl_sync(0xffffffffu, my_slot, i);
    const int r = (base_pair + i) / k;
    const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)r * ldx);
    uint4* dst = reinterpret_cast<uint4*>(xg + (size_t)s * d);
    for (int c = lane; c < d / 8; c += 32) dst[c] = src[c];
  }
}

// h[r] += sum_j (ascending expert) y[slot[r][j]]; y already carries the gate weight.
template <class YT>
__global__ void moe_combine_kernel(int rows, int k, int d, const YT* __restrict__ yg,
                                   const int32_t* __restrict__ slot, float* __restrict__ h, int ldh,
                                   int32_t* __restrict__ zero, int nzero) {
  pdl_begin();
  if (blockIdx.x == 0 && threadIdx.x < nzero) zero[threadIdx.x] = 0;
  int r = blockIdx.x;
  if (r >= rows) return;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float acc = 0.f;
    for (int j = 0; j < k; ++j) acc += to_f(yg[(size_t)slot[(size_t)r * k + j] * d + c]);
    h[(size_t)r * ldh + c] += acc;
  }
}

__global__ void swiglu_mul_kernel(long long n, const float* a, const float* b, float* out) {
  pdl_begin();
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i < n; i += (long long)gridDim.x * blockDim.x) {
    float x = a[i];
    out[i] = x / (1.f + __expf(-x)) * b[i];
  }
}

// ---- expert-parallel exchange over peer memory -----------------------------
__device__ __forceinline__ void st_release_sys_add(uint32_t* p) {
  asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void ep_signal_all(const EpPeers& P, int phase) {
  __threadfence_system();
  for (int p = 0; p < P.world; ++p) st_release_sys_add(P.flag[p] + phase * P.world + P.me);
}

__global__ void ep_counts_kernel(int E, const int32_t* __restrict__ counts, EpPeers P) {
  pdl_begin();
  for (int i = threadIdx.x; i < P.world * E; i += blockDim.x) {
    const int p = i / E, e = i - p * E;
    P.cnt[p][P.me * E + e] = counts[e];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) ep_signal_all(P, EP_COUNTS);
}

__global__ void ep_signal_kernel(EpPeers P, int phase) {
  pdl_begin();
  if (threadIdx.x == 0) ep_signal_all(P, phase);
}

// One thread spins (acquire, system scope) on the local arrival counters of
// every source for this exchange; gives up after 30 s (err = 1) so a lost
// peer cannot hang the GPU.
__global__ void ep_wait_kernel(EpPeers P, int phase) {
  pdl_begin();
  if (threadIdx.x != 0) return;
  const uint32_t target = P.epoch[phase] + 1;
  const uint32_t* f = P.flag[P.me] + phase * P.world;
  const uint64_t t0 = globaltimer_ns();
  for (int p = 0; p < P.world; ++p) {
    while (ld_acquire_sys(f + p) < target) {
      if (globaltimer_ns() - t0 > 30ull * 1000000000ull) {
        *P.err = 1;
        break;
      }
      __nanosleep(200);
    }
  }
  P.epoch[phase] = target;
  __threadfence();
}

// Device plan (the same arithmetic as ep_plan_placed, ep_plan.hpp, on every
// rank from the same histograms): rank p's grouped buffer holds, per local slot
// j (global expert list[p][j]), a segment of that expert's rows -- every rank's
// (source-rank major) for an owned expert, p's own for a replicated one
// (owner -1) -- padded to `tile`. Also accumulates the layer's global expert
// loads (placement statistics) and marks the padding rows (no source).
__global__ void ep_plan_kernel(int E, EpPeers P, int tile, int max_tiles, int32_t* __restrict__ cursor,
                               int32_t* __restrict__ tile_expert, int32_t* __restrict__ n_mtiles,
                               int32_t* __restrict__ seg, const int32_t* __restrict__ owner,
                               const int32_t* __restrict__ slot, const int32_t* __restrict__ list, int C,
                               long long* __restrict__ load) {
  pdl_begin();
  const int32_t* cnt = P.cnt[P.me];  // local copy [W][E]
  const int W = P.world;
  __shared__ int32_t tot[32], seg_start[kEpMaxWorld * 32], seg_rows[kEpMaxWorld * 32];
  const int e = threadIdx.x;
  if (e < E) {
    int t = 0;
    for (int q = 0; q < W; ++q) t += cnt[q * E + e];
    tot[e] = t;
    if (load) load[e] += t;
  }
  __syncthreads();
  if (threadIdx.x < W) {
    const int p = threadIdx.x;
    int off = 0;
    for (int j = 0; j < C; ++j) {
      const int g = list[p * C + j];
      const int n = g < 0 ? 0 : (owner[g] < 0 ? cnt[p * E + g] : tot[g]);
      seg_start[p * 32 + j] = off;
      seg_rows[p * 32 + j] = n;
      off += (n + tile - 1) / tile * tile;
    }
    if (p == P.me && off > P.recv_cap) *P.err = 2;
  }
  __syncthreads();
  if (e < E) {
    const int o = owner[e];
    int before = 0;
    if (o >= 0)
      for (int q = 0; q < P.me; ++q) before += cnt[q * E + e];
    cursor[e] = seg_start[(o < 0 ? P.me : o) * 32 + slot[e]] + before;
  }
  const int* my_start = seg_start + P.me * 32;
  const int* my_rows = seg_rows + P.me * 32;
  if (threadIdx.x == 0) {
    int nt = 0;
    for (int j = 0; j < C; ++j) {
      seg[2 * j] = my_start[j];
      seg[2 * j + 1] = my_rows[j];
      for (int i = 0; i < (my_rows[j] + tile - 1) / tile && nt < max_tiles; ++i) tile_expert[nt++] = j;
    }
    *n_mtiles = nt;
    for (int i = nt; i < max_tiles; ++i) tile_expert[i] = -1;
  }
  // padding rows of the local segments: no source (the fused return skips them)
  for (int j = 0; j < C; ++j) {
    const int end = min(my_start[j] + (my_rows[j] + tile - 1) / tile * tile, P.recv_cap);
    for (int i = my_start[j] + my_rows[j] + threadIdx.x; i < end; i += blockDim.x) P.src[P.me][i] = -1;
  }
}

template <class T>
__global__ void ep_dispatch_kernel(int rows, int k, int d, const T* __restrict__ x, int ldx,
                                   const int32_t* __restrict__ sel, const float* __restrict__ wts,
                                   int32_t* __restrict__ cursor, int32_t* __restrict__ slot,
                                   const int32_t* __restrict__ owner_of, EpPeers P) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const int n_pairs = rows * k;
  for (int base_pair = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; base_pair < n_pairs;
       base_pair += gridDim.x * (blockDim.x >> 5) * 32) {
    const int gw = base_pair + lane;
    const bool on = gw < n_pairs;
    const int e = on ? sel[gw] : -1;
    const unsigned act = __ballot_sync(0xffffffffu, on);
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (on && lane == leader) base = atomicAdd(&cursor[e], __popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    const int pos = base + __popc(peers & ((1u << lane) - 1u));
    const int own = on ? owner_of[e] : 0;
    const int owner = own < 0 ? P.me : own;  // replicated experts run where the token lives
    const bool fits = pos < P.recv_cap;
    if (on && fits) {
      slot[gw] = gw;
      P.wr[owner][pos] = wts[gw];
      P.src[owner][pos] = (P.me << 24) | gw;
    } else if (on) {
      *P.err = 2;
    }
    for (int i = 0; i < 32; ++i) {
      if (!((act >> i) & 1u)) break;
      const int s = __shfl_sync(0xffffffffu, pos, i);
      const int o = __shfl_sync(0xffffffffu, owner, i);
      if (s >= P.recv_cap) continue;
      const int r = (base_pair + i) / k;
      const T* a = x + (size_t)r * ldx;
      T* b = reinterpret_cast<T*>(P.xr[o]) + (size_t)s * d;
      if (sizeof(T) == 2 && d % 8 == 0) {
        for (int c = lane * 8; c < d; c += 256)
          *reinterpret_cast<uint4*>(b + c) = *reinterpret_cast<const uint4*>(a + c);
      } else if (d % 4 == 0) {
        for (int c = lane * 4; c < d; c += 128)
          *reinterpret_cast<uint4*>(b + c) = *reinterpret_cast<const uint4*>(a + c);
      } else {
        for (int c = lane; c < d; c += 32) b[c] = a[c];
      }
    }
  }
}

// Row-major form for bf16, d = 256 * NV, k | 32: a warp assigns 32 (token,
// expert) pairs (= 32 / k tokens) as above, then loads each token row ONCE
// (coalesced, NV x 16 B per lane) and stores it to its k destinations -- the
// peer stores are posted writes, so the next row's loads overlap them.
template <int NV>
__global__ void __launch_bounds__(256) ep_dispatch_rows_kernel(int rows, int k, int d,
                                                               const __nv_bfloat16* __restrict__ x, int ldx,
                                                               const int32_t* __restrict__ sel,
                                                               const float* __restrict__ wts,
                                                               int32_t* __restrict__ cursor, int32_t* __restrict__ slot,
                                                               const int32_t* __restrict__ owner_of, EpPeers P) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const int n_pairs = rows * k, tpw = 32 / k;
  for (int base_pair = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; base_pair < n_pairs;
       base_pair += gridDim.x * (blockDim.x >> 5) * 32) {
    const int gw = base_pair + lane;
    const bool on = gw < n_pairs;
    const int e = on ? sel[gw] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (on && lane == leader) base = atomicAdd(&cursor[e], __popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    const int pos = base + __popc(peers & ((1u << lane) - 1u));
    const int own = on ? owner_of[e] : 0;
    const int owner = own < 0 ? P.me : own;
    if (on && pos < P.recv_cap) {
      slot[gw] = gw;
      P.wr[owner][pos] = wts[gw];
      P.src[owner][pos] = (P.me << 24) | gw;
    } else if (on) {
      *P.err = 2;
    }
    const int r0 = base_pair / k;
#pragma unroll 2
    for (int t = 0; t < tpw; ++t) {
      const int r = r0 + t;
      if (r >= rows) break;
      const uint4* a = reinterpret_cast<const uint4*>(x + (size_t)r * ldx);
      uint4 v[NV];
#pragma unroll
      for (int q = 0; q < NV; ++q) v[q] = __ldg(a + lane + 32 * q);
      for (int j = 0; j < k; ++j) {
        const int s = __shfl_sync(0xffffffffu, pos, t * k + j);
        const int o = __shfl_sync(0xffffffffu, owner, t * k + j);
        if (s >= P.recv_cap) continue;
        uint4* b = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(P.xr[o]) + (size_t)s * d);
#pragma unroll
        for (int q = 0; q < NV; ++q) b[lane + 32 * q] = v[q];
      }
    }
  }
}

// Warp per received row: the weighted expert output goes back to yr[slot] on the
// token's rank (fp32 engine; the bf16 engine stores from the W2 GEMM epilogue).
template <class T>
__global__ void ep_return_kernel(int El, int d, const int32_t* __restrict__ seg, const T* __restrict__ yg,
                                 EpPeers P) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const int wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), nw = gridDim.x * (blockDim.x >> 5);
  const int32_t* src = P.src[P.me];
  for (int el = 0; el < El; ++el) {
    const int s0 = seg[2 * el], n = seg[2 * el + 1];
    for (int i = wid; i < n; i += nw) {
      const int code = src[s0 + i];
      const int q = code >> 24, gw = code & 0xFFFFFF;
      const T* a = yg + (size_t)(s0 + i) * d;
      T* b = static_cast<T*>(P.yr[q]) + (size_t)gw * d;
      constexpr int V = 16 / sizeof(T);
      if (d % V == 0) {
        for (int c = lane * V; c < d; c += 32 * V)
          *reinterpret_cast<uint4*>(b + c) = *reinterpret_cast<const uint4*>(a + c);
      } else {
        for (int c = lane; c < d; c += 32) b[c] = a[c];
      }
    }
  }
}

// K|V of the empty-history pad key rows (kv = pad.lifelong . Wkv, fp32 [2 nkv]):
// K part row-major into kvl[row][0 .. nkv), V part transposed like the split
// K|V GEMM's epilogue (column n of layer n / d at vt[u][n % d][t]).
template <class T>
__global__ void fill_kv_pad_kernel(int n_pad, const int32_t* __restrict__ rows, const int32_t* __restrict__ row_user,
                                   const int32_t* __restrict__ row_pos, const float* __restrict__ kv, int nkv,
                                   T* __restrict__ kvl, int ldk, T* __restrict__ vt, int vt_ld,
                                   long long vt_user_stride, long long vt_layer_stride, int d) {
  pdl_begin();
  for (int i = blockIdx.x; i < n_pad; i += gridDim.x) {
    const int r = rows[i], u = row_user[r], t = row_pos[r];
    for (int n = threadIdx.x; n < nkv; n += blockDim.x) {
      kvl[(size_t)r * ldk + n] = from_f<T>(kv[n]);
      const int l = n / d, m = n - l * d;
      vt[(long long)u * vt_user_stride + t + (long long)m * vt_ld + (long long)l * vt_layer_stride] =
          from_f<T>(kv[nkv + n]);
    }
  }
}

inline int grid_for(long long n, int block, int cap = 148 * 32) {
  long long g = (n + block - 1) / block;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

#define ORX_LAUNCH_CAT(cat, ...)          \
  do {                                    \
    ProfScope ps__(cat, s, 0.0, 0.0);     \
    __VA_ARGS__;                          \
    prof_note_launch(#__VA_ARGS__);         \
    ++launch_counter();                   \
  } while (0)
#define ORX_LAUNCH(...) ORX_LAUNCH_CAT(PROF_MISC, __VA_ARGS__)
// with the launch's algorithmic HBM bytes (bench.py's per-class GB/s)
#define ORX_LAUNCH_CATB(cat, bytes, ...)    \
  do {                                      \
    ProfScope ps__(cat, s, 0.0, (bytes));   \
    __VA_ARGS__;                            \
    prof_note_launch(#__VA_ARGS__);         \
    ++launch_counter();                     \
  } while (0)

template <class T>
void launch_features(const RecordsDev& r, const FeatureTables& t, T* out, int ldo, cudaStream_t s) {
  if (r.n <= 0) return;
  const double nb = double(r.n) * (double(ldo) * sizeof(T) + 28.0);  // feature rows out, scalar inputs in
  const bool vec = t.d % 8 == 0 && ldo % 8 == 0 && (t.vid_only || (t.aid_dim % 8 == 0 && t.minor % 8 == 0));
  if constexpr (sizeof(T) == 2) {
    if (vec && t.vid16 && t.aid16 && !t.use_sid && !t.vid_only && ldo <= 8 * 32 * kFeatMaxChunks) {
      const size_t tsm = sizeof(float) * (8 + t.n_flags) * t.minor;
      if (tsm > 48 * 1024) cudaFuncSetAttribute(features16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(tsm));
      ORX_LAUNCH_CATB(PROF_FEAT, nb, launch_pdl(features16_kernel, grid_for(r.n, 8, num_sms() * 8), 256, tsm, s, 
          r, t, reinterpret_cast<__nv_bfloat16*>(out), ldo));
      return;
    }
  }
  if (vec) {
    ORX_LAUNCH_CATB(PROF_FEAT, nb, launch_pdl(features8_kernel<T>, grid_for(r.n, 8, num_sms() * 8), 256, 0, s, r, t, out, ldo));
    return;
  }
  ORX_LAUNCH_CATB(PROF_FEAT, nb, launch_pdl(features_kernel<T>, grid_for(r.n, 1, 148 * 16), 256, 0, s, r, t, out, ldo));
}
bool fold_features_supported(int d, int n_flags) {
  const int g = (d + 255) / 256;
  return d % 4 == 0 && d <= 2048 && 8 % g == 0 && n_flags >= 0 && n_flags <= 8;
}
void launch_fold_features(const RecordsDev& r, const FoldTables& f, __nv_bfloat16* out, int ldo, cudaStream_t s) {
  if (r.n <= 0) return;
  if (!fold_features_supported(f.d, f.n_flags) || ldo % 4 != 0)
    throw std::invalid_argument("fold_features: unsupported shape");
  const int g = (f.d + 255) / 256, rpb = 8 / g;
  const int grid = static_cast<int>(std::min<long long>((r.n + rpb - 1) / rpb, num_sms() * 3LL));  // 3 blocks per SM
  // records' scalar inputs in, bf16 hidden rows out (the table gathers are L2 hits)
  const double nb = double(r.n) * (2.0 * f.d + 28.0);
  auto go = [&](auto kern) { ORX_LAUNCH_CATB(PROF_FEAT, nb, launch_pdl(kern, grid, 256, 0, s, r, f, out, ldo)); };
  if (f.pal) {
    if (g == 1) go(fold_features_kernel<1, true>);
    else if (g == 2) go(fold_features_kernel<2, true>);
    else if (g == 4) go(fold_features_kernel<4, true>);
    else go(fold_features_kernel<8, true>);
  } else {
    if (g == 1) go(fold_features_kernel<1, false>);
    else if (g == 2) go(fold_features_kernel<2, false>);
    else if (g == 4) go(fold_features_kernel<4, false>);
    else go(fold_features_kernel<8, false>);
  }
}
void launch_fold_pal(int naid, int n_flags, int d, const float* pa, const float* pl, float* pal, cudaStream_t s) {
  const long long n = (long long)naid << n_flags;
  fold_pal_kernel<<<static_cast<int>(std::min<long long>(n, 148LL * 16)), 256, 0, s>>>(naid, n_flags, d, pa, pl, pal);
}
template <class T>
void launch_static_features(int U, const int32_t* uid, const int32_t* gender, const int32_t* age, const float* ue,
                            const float* ge, const float* ae, int sd, int uv, int gv, int av, T* out, int ldo,
                            cudaStream_t s) {
  ORX_LAUNCH(launch_pdl(static_features_kernel<T>, U, 128, 0, s, U, uid, gender, age, ue, ge, ae, sd, uv, gv, av, out, ldo));
}
void launch_z_init(int U, int T, int d, const float* pos, const float* pad_s, const float* pad_p, const int32_t* n_s,
                   const int32_t* n_p, int Ls, int Lp, float* z, cudaStream_t s) {
  const bool al = reinterpret_cast<uintptr_t>(pos) % 16 == 0 && reinterpret_cast<uintptr_t>(z) % 16 == 0 &&
                  reinterpret_cast<uintptr_t>(pad_s) % 16 == 0 && reinterpret_cast<uintptr_t>(pad_p) % 16 == 0;
  if (!al && d % 4 == 0) throw std::invalid_argument("z_init: buffers must be 16-byte aligned");
  ORX_LAUNCH(launch_pdl(z_init_kernel, U * T, d % 4 == 0 ? std::min(256, d / 4) : 256, 0, s, U, T, d, pos, pad_s, pad_p,
                        n_s, n_p, Ls, Lp, z));
}
// Warp per row, the row held in registers: one float4 load per lane per 128
// columns, all NC issued before the reduction (the scalar kernel above ran at
// ~60% of HBM bandwidth on 4-byte loads).
template <class T, int NC>
__global__ void __launch_bounds__(256, 2) rmsnorm4_kernel(int rows, int d, const float* __restrict__ x, int ldx,
                                                       const float* __restrict__ g, T* __restrict__ out, int ldo) {
  pdl_begin();
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (row >= rows) return;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)row * ldx);
  float4 v[NC];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int c4 = lane + 32 * i;
    v[i] = c4 * 4 < d ? __ldg(xr + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int i = 0; i < NC; ++i) ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / d + 1e-6f);
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int c = (lane + 32 * i) * 4;
    if (c >= d) continue;
    const float4 gg = __ldg(reinterpret_cast<const float4*>(g + c));
    const float a = v[i].x * r * gg.x, b = v[i].y * r * gg.y, cc = v[i].z * r * gg.z, e = v[i].w * r * gg.w;
    if constexpr (sizeof(T) == 2) {
      *reinterpret_cast<uint2*>(out + (size_t)row * ldo + c) = make_uint2(pack_bf16(a, b), pack_bf16(cc, e));
    } else {
      *reinterpret_cast<float4*>(out + (size_t)row * ldo + c) = make_float4(a, b, cc, e);
    }
  }
}

template <class T>
void launch_rmsnorm(int rows, int d, const float* x, int ldx, const float* gain, T* out, int ldo, cudaStream_t s) {
  if (rows <= 0) return;
  const double nb = double(rows) * d * (4.0 + sizeof(T));  // fp32 row in, normalised row out
  const bool vec = d % 4 == 0 && ldx % 4 == 0 && ldo % 4 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(gain) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0;
  if (vec && d <= 512) {
    ORX_LAUNCH_CATB(PROF_NORM, nb, launch_pdl(rmsnorm4_kernel<T, 4>, (rows + 7) / 8, 256, 0, s, rows, d, x, ldx, gain, out, ldo));
  } else if (vec && d <= 1024) {
    ORX_LAUNCH_CATB(PROF_NORM, nb, launch_pdl(rmsnorm4_kernel<T, 8>, (rows + 7) / 8, 256, 0, s, rows, d, x, ldx, gain, out, ldo));
  } else if (vec && d <= 2048) {
    ORX_LAUNCH_CATB(PROF_NORM, nb, launch_pdl(rmsnorm4_kernel<T, 16>, (rows + 7) / 8, 256, 0, s, rows, d, x, ldx, gain, out, ldo));
  } else {
    ORX_LAUNCH_CATB(PROF_NORM, nb, launch_pdl(rmsnorm_kernel<T>, (rows + 7) / 8, 256, 0, s, rows, d, x, ldx, gain, out, ldo));
  }
}
template <class T>
void launch_convert(int rows, int cols, const float* x, int ldx, T* out, int ldo, cudaStream_t s) {
  if (rows <= 0) return;
  if (cols % 4 == 0 && ldx % 4 == 0 && ldo % 4 == 0) {
    ORX_LAUNCH(launch_pdl(convert4_kernel<T>, grid_for((long long)rows * cols / 4, 256), 256, 0, s, rows, cols, x, ldx, out,
                                                                                          ldo));
    return;
  }
  ORX_LAUNCH(launch_pdl(convert_kernel<T>, grid_for((long long)rows * cols, 256), 256, 0, s, rows, cols, x, ldx, out, ldo));
}
template <class T>
void launch_fill_rows(int rows, int cols, const float* src, T* out, int ldo, const int32_t* idx, cudaStream_t s) {
  if (rows <= 0) return;
  ORX_LAUNCH(launch_pdl(fill_rows_kernel<T>, rows, 128, 0, s, rows, cols, src, out, ldo, idx));
}
void launch_dec_embed(int rows, int d, const float* table, const int32_t* code, int code_stride, float* h,
                      cudaStream_t s) {
  if (rows <= 0) return;
  if (d % 4 == 0 && (reinterpret_cast<uintptr_t>(table) % 16 || reinterpret_cast<uintptr_t>(h) % 16))
    throw std::invalid_argument("dec_embed: buffers must be 16-byte aligned");
  ORX_LAUNCH(launch_pdl(dec_embed_kernel, rows, d % 4 == 0 ? std::min(256, d / 4) : 256, 0, s, rows, d, table, code,
                        code_stride, h));
}
bool launch_dec_embed_norm(int rows, int d, const float* table, const int32_t* code, int code_stride, float* h,
                           const float* gain, __nv_bfloat16* out, cudaStream_t s) {
  if (d % 128 != 0 || d > 1024 || reinterpret_cast<uintptr_t>(table) % 16 || reinterpret_cast<uintptr_t>(h) % 16 ||
      reinterpret_cast<uintptr_t>(out) % 16 || reinterpret_cast<uintptr_t>(gain) % 16)
    return false;
  if (rows <= 0) return true;
  const int nc = d / 128;
  const double nb = double(rows) * d * (4.0 + 4.0 + 2.0);
  auto go = [&](auto kern) {
    ORX_LAUNCH_CATB(PROF_NORM, nb, launch_pdl(kern, (rows + 7) / 8, 256, 0, s, rows, d, table, code, code_stride, h,
                                              gain, out));
  };
  switch (nc) {
    case 1: go(dec_embed_norm_kernel<1>); break;
    case 2: go(dec_embed_norm_kernel<2>); break;
    case 4: go(dec_embed_norm_kernel<4>); break;
    case 8: go(dec_embed_norm_kernel<8>); break;
    default: return false;
  }
  return true;
}
// bf16 decoder self-attention, one warp per ROW (all heads): lane l owns
// columns [l * EPL, (l + 1) * EPL) of q / k / v (16-byte loads), a head spans
// dh / EPL lanes, so each position's dot product is a per-lane partial plus a
// log2(dh / EPL)-step shuffle; the ancestor row of each cached position is
// loaded once per row instead of once per head (the warp-per-head kernel
// above was issue bound on shuffles and index math).
template <int EPL>
__global__ void __launch_bounds__(256) dec_self_attn_row_kernel(int rows, int d, int heads, int step, int layer, int L,
                                                                const __nv_bfloat16* __restrict__ qkv,
                                                                __nv_bfloat16* const* __restrict__ kv,
                                                                const int32_t* __restrict__ anc, int anc_stride,
                                                                __nv_bfloat16* __restrict__ out) {
  pdl_begin();
  constexpr int NV = EPL / 8;  // uint4 (8 x bf16) per lane
  const int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (r >= rows) return;
  const int dh = d / heads, lph = dh / EPL;  // lanes per head (power of two)
  const int c0 = lane * EPL;
  const __nv_bfloat16* qr = qkv + (size_t)r * 3 * d + c0;
  uint4 q[NV], kv_own[2][NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    q[i] = __ldg(reinterpret_cast<const uint4*>(qr) + i);
    kv_own[0][i] = __ldg(reinterpret_cast<const uint4*>(qr + d) + i);
    kv_own[1][i] = __ldg(reinterpret_cast<const uint4*>(qr + 2 * d) + i);
  }
  const int a_l = lane < step ? anc[(size_t)r * anc_stride + lane] : 0;
  auto bf2 = [](uint32_t w) { return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w)); };
  auto dot = [&](const uint4* k) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const uint32_t qw[4] = {q[i].x, q[i].y, q[i].z, q[i].w}, kw[4] = {k[i].x, k[i].y, k[i].z, k[i].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 a = bf2(qw[j]), b = bf2(kw[j]);
        s = fmaf(a.x, b.x, s);
        s = fmaf(a.y, b.y, s);
      }
    }
    for (int o = lph >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
  };
  const float scale = rsqrtf(static_cast<float>(dh));
  float sc[8];
  float mx = -FLT_MAX;
  for (int p = 0; p <= step; ++p) {
    float sp;
    if (p < step) {
      const int ar = __shfl_sync(0xffffffffu, a_l, p);
      const uint4* kp = reinterpret_cast<const uint4*>(kv_at(kv, p, L, layer, ar, d) + c0);
      uint4 kk[NV];
#pragma unroll
      for (int i = 0; i < NV; ++i) kk[i] = kp[i];
      sp = dot(kk);
    } else {
      sp = dot(kv_own[0]);
    }
    sc[p] = sp * scale;
    mx = fmaxf(mx, sc[p]);
  }
  float den = 0.f;
  for (int p = 0; p <= step; ++p) {
    sc[p] = __expf(sc[p] - mx);
    den += sc[p];
  }
  float acc[EPL];
#pragma unroll
  for (int e = 0; e < EPL; ++e) acc[e] = 0.f;
  for (int p = 0; p <= step; ++p) {
    uint4 vv[NV];
    if (p < step) {
      const int ar = __shfl_sync(0xffffffffu, a_l, p);
      const uint4* vp = reinterpret_cast<const uint4*>(kv_at(kv, p, L, layer, ar, d) + d + c0);
#pragma unroll
      for (int i = 0; i < NV; ++i) vv[i] = vp[i];
    } else {
#pragma unroll
      for (int i = 0; i < NV; ++i) vv[i] = kv_own[1][i];
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const uint32_t vw[4] = {vv[i].x, vv[i].y, vv[i].z, vv[i].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 b = bf2(vw[j]);
        acc[8 * i + 2 * j] = fmaf(sc[p], b.x, acc[8 * i + 2 * j]);
        acc[8 * i + 2 * j + 1] = fmaf(sc[p], b.y, acc[8 * i + 2 * j + 1]);
      }
    }
  }
  const float inv = 1.f / den;
  uint4* o = reinterpret_cast<uint4*>(out + (size_t)r * d + c0);
#pragma unroll
  for (int i = 0; i < NV; ++i)
    o[i] = make_uint4(pack_bf16(acc[8 * i] * inv, acc[8 * i + 1] * inv), pack_bf16(acc[8 * i + 2] * inv, acc[8 * i + 3] * inv),
                      pack_bf16(acc[8 * i + 4] * inv, acc[8 * i + 5] * inv), pack_bf16(acc[8 * i + 6] * inv, acc[8 * i + 7] * inv));
}

template <class T>
void launch_dec_self_attn(int rows, int d, int heads, int step, int layer, int L, const T* qkv, T* const* kv,
                          const int32_t* anc, int anc_stride, T* out, cudaStream_t s) {
  if (rows <= 0) return;
  // per row: q, k, v in; the ancestors' k, v; out row
  const double nb = double(rows) * d * sizeof(T) * (3.0 + 2.0 * step + 1.0);
  long long warps = (long long)rows * heads;
  if constexpr (sizeof(T) == 2) {
    const int dh = d / heads, epl = d / 32, lph = epl > 0 ? dh / epl : 0;
    if (d % 256 == 0 && epl <= 64 && dh % epl == 0 && (lph & (lph - 1)) == 0 && step < 8) {  // whole row per warp
      auto go = [&](auto kern) {
        ORX_LAUNCH_CATB(PROF_DEC_SELF, nb, launch_pdl(kern, (rows + 7) / 8, 256, 0, s, rows, d, heads, step, layer, L,
                                                 reinterpret_cast<const __nv_bfloat16*>(qkv),
                                                 reinterpret_cast<__nv_bfloat16* const*>(kv), anc, anc_stride,
                                                 reinterpret_cast<__nv_bfloat16*>(out)));
      };
      if (epl == 8) go(dec_self_attn_row_kernel<8>);
      else if (epl == 16) go(dec_self_attn_row_kernel<16>);
      else if (epl == 32) go(dec_self_attn_row_kernel<32>);
      else go(dec_self_attn_row_kernel<64>);
      return;
    }
  }
  if ((d / heads) % 4 == 0 && d / heads <= 128 && d % 4 == 0) {
    ORX_LAUNCH_CATB(PROF_DEC_SELF, nb, launch_pdl(dec_self_attn4_kernel<T>, static_cast<int>((warps + 7) / 8), 256, 0, s, 
        rows, d, heads, step, layer, L, qkv, kv, anc, anc_stride, out));
    return;
  }
  ORX_LAUNCH_CATB(PROF_DEC_SELF, nb, launch_pdl(dec_self_attn_kernel<T>, static_cast<int>((warps + 7) / 8), 256, 0, s, 
      rows, d, heads, step, layer, L, qkv, kv, anc, anc_stride, out));
}
void launch_moe_route(int rows, int d, int E, int k, const float* x, int ldx, const float* gain, const float* gate_t,
                      const float* gate_gain, const float* bias, int32_t* sel, float* wts, int32_t* counts,
                      cudaStream_t s, const float* gate_sw) {
  if (rows <= 0) return;
  if (E > 32) throw std::invalid_argument("moe routing supports at most 32 experts");
  const int smem = E * d * 4;
  if (gate_sw && E <= 24 && k <= 8 && d % 128 == 0 && ldx % 4 == 0 && !getenv("ORX_ROUTE_V2")) {
    const int smem4 = 24 * d * 4;
    const int per_block = 8 * kRoute4Rows;
    const int blocks = std::min((rows + per_block - 1) / per_block, num_sms());  // one 8-warp block per SM
    static int set4 = 0;
    if (smem4 > 48 * 1024 && smem4 > set4) {
      cudaFuncSetAttribute(moe_route4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem4);
      set4 = smem4;
    }
    ProfScope ps(PROF_MOE_ROUTE, s, 0.0, double(rows) * (4.0 * d + 8.0 * k));
    launch_pdl(moe_route4_kernel, blocks, 256, smem4, s, rows, d, E, k, x, ldx, gate_sw, bias, sel, wts, counts);
    ++launch_counter();
    return;
  }
  if (gate_gain && d % 4 == 0 && ldx % 4 == 0) {
    const int per_block = 8 * kRoutePerWarp;
    int blocks = std::min((rows + per_block - 1) / per_block, num_sms() * 2);
    static int set2 = 0;
    if (smem > 48 * 1024 && smem > set2) {
      cudaFuncSetAttribute(moe_route2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      set2 = smem;
    }
    ORX_LAUNCH_CAT(PROF_MOE_ROUTE, launch_pdl(moe_route2_kernel, blocks, 256, smem, s, rows, d, E, k, x, ldx, gate_gain, bias,
                                              sel, wts, counts));
    return;
  }
  if (d > 32 * kRouteMaxPer) throw std::invalid_argument("moe routing supports d_model <= 2048");
  static int set = 0;
  if (smem > 48 * 1024 && smem > set) {
    cudaFuncSetAttribute(moe_route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    set = smem;
  }
  int blocks = std::min((rows + 7) / 8, num_sms() * 2);
  ORX_LAUNCH_CAT(PROF_MOE_ROUTE, launch_pdl(moe_route_kernel, blocks, 256, smem, s, rows, d, E, k, x, ldx, gain, gate_t, bias,
                                                                            sel, wts, counts));
}
template <class T>
void launch_moe_scatter(int rows, int k, int d, const T* x, int ldx, const int32_t* sel, const float* wts,
                        const MoePlan& plan, int32_t* slot, T* xg, float* row_scale, cudaStream_t s) {
  if (plan.E > 32) throw std::invalid_argument("moe_scatter: at most 32 experts");
  const double nb = double(rows) * d * sizeof(T) * (1.0 + k);  // token rows in, k expert-sorted copies out
  if (rows <= 0) return;
  long long warps = (long long)rows * k;
  if constexpr (sizeof(T) == 2) {
    if (d % 8 == 0 && ldx % 8 == 0 && warps >= 8192) {  // many pairs: aggregate the slot atomics per warp
      const long long w32 = (warps + 31) / 32;
      ORX_LAUNCH_CATB(PROF_MOE_ROUTE, nb, launch_pdl(moe_scatter32_kernel, static_cast<int>((w32 + 7) / 8), 256, 0, s, 
                                         rows, k, d, reinterpret_cast<const __nv_bfloat16*>(x), ldx, sel, wts, plan,
                                         slot, reinterpret_cast<__nv_bfloat16*>(xg), row_scale));
      return;
    }
  }
  ORX_LAUNCH_CATB(PROF_MOE_ROUTE, nb, launch_pdl(moe_scatter_kernel<T>, static_cast<int>((warps + 7) / 8), 256, 0, s, rows, k, d, x, ldx, sel, wts,
                                                                                      plan, slot, xg, row_scale));
}
// h += sum_j yg[slot[r][j]] (as moe_combine4_kernel, same order), then the
// NEXT op's input from the updated row while it is in registers: the next
// layer's RMSNorm (gain) or, for the head, a plain bf16 copy (gain null) —
// as rmsnorm4_kernel / convert would compute it, one pass over h instead of two.
template <int NC, class YT>
__global__ void __launch_bounds__(256) moe_combine_norm_kernel(int rows, int k, int d, const YT* __restrict__ yg,
                                                               const int32_t* __restrict__ slot, float* __restrict__ h,
                                                               int ldh, const float* __restrict__ gain,
                                                               __nv_bfloat16* __restrict__ out, int ldo,
                                                               int32_t* __restrict__ zero, int nzero) {
  pdl_begin();
  if (blockIdx.x == 0 && threadIdx.x < nzero) zero[threadIdx.x] = 0;
  const int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (r >= rows) return;
  // every load of a pass is issued before its first use (the row's h segment and
  // the first expert output, then one pass per further expert): k round trips
  // to memory per row instead of one per column chunk
  float4 v[NC], acc[NC];
  float4* hr = reinterpret_cast<float4*>(h + (size_t)r * ldh);
  const YT* y0 = yg + (size_t)slot[(size_t)r * k] * d;
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    v[i] = hr[lane + 32 * i];
    acc[i] = ldy4(y0 + 4 * (lane + 32 * i));
  }
  for (int j = 1; j < k; ++j) {  // ascending expert order, as the reference combines (nn.cpp:152-169)
    const YT* yj = yg + (size_t)slot[(size_t)r * k + j] * d;
    float4 y[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) y[i] = ldy4(yj + 4 * (lane + 32 * i));
#pragma unroll
    for (int i = 0; i < NC; ++i) acc[i].x += y[i].x, acc[i].y += y[i].y, acc[i].z += y[i].z, acc[i].w += y[i].w;
  }
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    v[i].x += acc[i].x, v[i].y += acc[i].y, v[i].z += acc[i].z, v[i].w += acc[i].w;
    hr[lane + 32 * i] = v[i];
  }
  float rs = 1.f;
  if (gain) {
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < NC; ++i) ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
    ss = warp_sum(ss);
    rs = rsqrtf(ss / d + 1e-6f);
  }
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int c = (lane + 32 * i) * 4;
    float a = v[i].x, b = v[i].y, cc = v[i].z, e = v[i].w;
    if (gain) {
      const float4 g4 = __ldg(reinterpret_cast<const float4*>(gain + c));
      a = a * rs * g4.x, b = b * rs * g4.y, cc = cc * rs * g4.z, e = e * rs * g4.w;
    }
    *reinterpret_cast<uint2*>(out + (size_t)r * ldo + c) = make_uint2(pack_bf16(a, b), pack_bf16(cc, e));
  }
}

template <class YT>
bool launch_moe_combine_norm(int rows, int k, int d, const YT* yg, const int32_t* slot, float* h, int ldh,
                             const float* gain, __nv_bfloat16* out, int ldo, cudaStream_t s, int32_t* zero,
                             int nzero) {
  if (nzero > 256) throw std::invalid_argument("moe_combine: at most 256 counters to zero");
  if ((d != 512 && d != 1024) || ldh % 4 || ldo % 4 || reinterpret_cast<uintptr_t>(h) % 16 ||
      reinterpret_cast<uintptr_t>(out) % 16 || (gain && reinterpret_cast<uintptr_t>(gain) % 16) ||
      getenv("ORX_NO_COMBINE_NORM"))
    return false;
  if (rows <= 0) return true;
  const double nb = double(rows) * d * (sizeof(YT) * k + 8.0 + 2.0);  // k expert outputs + residual in/out + bf16 row
  if (d == 1024)
    ORX_LAUNCH_CATB(PROF_MOE_ROUTE, nb, launch_pdl(moe_combine_norm_kernel<8, YT>, (rows + 7) / 8, 256, 0, s, rows, k, d, yg,
                                              slot, h, ldh, gain, out, ldo, zero, nzero));
  else
    ORX_LAUNCH_CATB(PROF_MOE_ROUTE, nb, launch_pdl(moe_combine_norm_kernel<4, YT>, (rows + 7) / 8, 256, 0, s, rows, k, d, yg,
                                              slot, h, ldh, gain, out, ldo, zero, nzero));
  return true;
}

template <class YT>
void launch_moe_combine(int rows, int k, int d, const YT* yg, const int32_t* slot, float* h, int ldh,
                        cudaStream_t s, int32_t* zero, int nzero) {
  if (nzero > 256) throw std::invalid_argument("moe_combine: at most 256 counters to zero");
  const double nb = double(rows) * d * (sizeof(YT) * k + 8.0);  // k expert outputs + residual in/out
  if (rows <= 0) return;
  if (d % 4 == 0 && ldh % 4 == 0) {
    ORX_LAUNCH_CATB(PROF_MOE_ROUTE, nb, launch_pdl(moe_combine4_kernel<YT>, grid_for((long long)rows * d / 4, 256, num_sms() * 8), 256, 0, s, rows, k, d, yg, slot, h, ldh, zero, nzero));
    return;
  }
  ORX_LAUNCH_CATB(PROF_MOE_ROUTE, nb, launch_pdl(moe_combine_kernel<YT>, rows, 256, 0, s, rows, k, d, yg, slot, h, ldh, zero, nzero));
}
void launch_swiglu_mul(long long n, const float* a, const float* b, float* out, cudaStream_t s) {
  if (n <= 0) return;
  ORX_LAUNCH(launch_pdl(swiglu_mul_kernel, grid_for(n, 256), 256, 0, s, n, a, b, out));
}

void launch_ep_counts(int E, const int32_t* counts, const EpPeers& P, cudaStream_t s) {
  ORX_LAUNCH_CATB(PROF_MOE_ROUTE, double(P.world) * E * 4, launch_pdl(ep_counts_kernel, 1, 256, 0, s, E, counts, P));
}
void launch_ep_signal(const EpPeers& P, int phase, cudaStream_t s) {
  ORX_LAUNCH_CAT(PROF_MOE_ROUTE, launch_pdl(ep_signal_kernel, 1, 32, 0, s, P, phase));
}
void launch_ep_wait(const EpPeers& P, int phase, cudaStream_t s) {
  ORX_LAUNCH_CAT(PROF_MOE_ROUTE, launch_pdl(ep_wait_kernel, 1, 32, 0, s, P, phase));
}
void launch_ep_plan(int E, const EpPeers& P, int tile, int max_tiles, int32_t* cursor, int32_t* tile_expert,
                    int32_t* n_mtiles, int32_t* seg, const int32_t* owner, const int32_t* slot, const int32_t* list,
                    int C, long long* load, cudaStream_t s) {
  if (E > 32 || C > 32 || P.world > kEpMaxWorld) throw std::invalid_argument("ep_plan: at most 32 experts / slots");
  ORX_LAUNCH_CAT(PROF_MOE_ROUTE, launch_pdl(ep_plan_kernel, 1, 32, 0, s, E, P, tile, max_tiles, cursor, tile_expert,
                                            n_mtiles, seg, owner, slot, list, C, load));
}
template <class T>
void launch_ep_dispatch(int rows, int k, int d, const T* x, int ldx, const int32_t* sel, const float* wts,
                        int32_t* cursor, int32_t* slot, const int32_t* owner, const EpPeers& P, cudaStream_t s) {
  if (rows <= 0) return;
  const double nb = double(rows) * k * (d * sizeof(T) + 8.0) + double(rows) * d * sizeof(T);
  const long long warps = ((long long)rows * k + 31) / 32;
  if constexpr (sizeof(T) == 2) {
    const int nv = d / 256;
    if (d % 256 == 0 && 32 % k == 0 && ldx % 8 == 0 && (nv == 1 || nv == 2 || nv == 4)) {
      auto kern = nv == 4 ? ep_dispatch_rows_kernel<4> : nv == 2 ? ep_dispatch_rows_kernel<2> : ep_dispatch_rows_kernel<1>;
      ORX_LAUNCH_CATB(PROF_MOE_ROUTE, nb,
                      launch_pdl(kern, grid_for(warps, 8, num_sms() * 8), 256, 0, s, rows, k, d,
                                 reinterpret_cast<const __nv_bfloat16*>(x), ldx, sel, wts, cursor, slot, owner, P));
      return;
    }
  }
  ORX_LAUNCH_CATB(PROF_MOE_ROUTE, nb,
                  launch_pdl(ep_dispatch_kernel<T>, grid_for(warps, 8, num_sms() * 8), 256, 0, s, rows, k, d, x, ldx,
                             sel, wts, cursor, slot, owner, P));
}
template <class T>
void launch_ep_return(int El, int d, const int32_t* seg, const T* yg, const EpPeers& P, cudaStream_t s) {
  ORX_LAUNCH_CAT(PROF_MOE_ROUTE, launch_pdl(ep_return_kernel<T>, num_sms() * 4, 256, 0, s, El, d, seg, yg, P));
}

template <class T>
void launch_fill_kv_pad(int n_pad, const int32_t* rows, const int32_t* row_user, const int32_t* row_pos,
                        const float* kv, int nkv, T* kvl, int ldk, T* vt, int vt_ld, long long vt_user_stride,
                        long long vt_layer_stride, int d, cudaStream_t s) {
  if (n_pad <= 0) return;
  ORX_LAUNCH(launch_pdl(fill_kv_pad_kernel<T>, std::min(n_pad, num_sms() * 4), 256, 0, s, n_pad, rows, row_user,
                        row_pos, kv, nkv, kvl, ldk, vt, vt_ld, vt_user_stride, vt_layer_stride, d));
}

#define INST(T)                                                                                                   \
  template void launch_features<T>(const RecordsDev&, const FeatureTables&, T*, int, cudaStream_t);              \
  template void launch_static_features<T>(int, const int32_t*, const int32_t*, const int32_t*, const float*,     \
                                          const float*, const float*, int, int, int, int, T*, int, cudaStream_t); \
  template void launch_rmsnorm<T>(int, int, const float*, int, const float*, T*, int, cudaStream_t);              \
  template void launch_convert<T>(int, int, const float*, int, T*, int, cudaStream_t);                           \
  template void launch_fill_rows<T>(int, int, const float*, T*, int, const int32_t*, cudaStream_t);              \
  template void launch_fill_kv_pad<T>(int, const int32_t*, const int32_t*, const int32_t*, const float*, int, T*, \
                                      int, T*, int, long long, long long, int, cudaStream_t);                      \
  template void launch_dec_self_attn<T>(int, int, int, int, int, int, const T*, T* const*, const int32_t*, int,   \
                                        T*, cudaStream_t);                                                       \
  template void launch_moe_scatter<T>(int, int, int, const T*, int, const int32_t*, const float*, const MoePlan&, \
                                      int32_t*, T*, float*, cudaStream_t);                                        \
  template void launch_ep_dispatch<T>(int, int, int, const T*, int, const int32_t*, const float*, int32_t*,       \
                                      int32_t*, const int32_t*, const EpPeers&, cudaStream_t);                               \
  template void launch_ep_return<T>(int, int, const int32_t*, const T*, const EpPeers&, cudaStream_t);           \
  template void launch_moe_combine<T>(int, int, int, const T*, const int32_t*, float*, int, cudaStream_t, int32_t*, \
                                      int);                                                                        \
  template bool launch_moe_combine_norm<T>(int, int, int, const T*, const int32_t*, float*, int, const float*,    \
                                           __nv_bfloat16*, int, cudaStream_t, int32_t*, int);
INST(float)
INST(__nv_bfloat16)

}  // namespace orx
