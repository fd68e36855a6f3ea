// Lifelong-history compression on the GPU: the
// reference's compress_lifelong (policy.cpp:447-510) over hierarchical
// K-means (kmeans.cpp:22-183), one CTA per user, bit-identical to the f64
// CPU code:
//  * every squared distance is summed sequentially over the content columns
//    with explicitly rounded f64 operations (no FMA contraction), as sq_dist;
//  * every order-dependent f64 sum (k-means++ total and pick scan, the
//    objective, centroid sums, leaf centres and feature means) runs in the
//    reference's index order;
//  * the xoshiro256** stream (rng.cpp) is consumed in the same order: the
//    recursive splits are replayed depth-first with an explicit stack;
//  * ties break like the reference (lowest centroid / index, first minimum).
// Parallelism is across points inside a CTA and across users over the grid.
#include <cfloat>
#include <stdexcept>
#include <string>
#include <vector>

#include "compress.cuh"
#include "gemm.cuh"
#include "model.hpp"

namespace orx {

namespace {

constexpr int kCT = 256;

struct DevRng {  // rng.cpp:23-70 (state seeded on the host)
  uint64_t s[4];
  __device__ static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  __device__ uint64_t next() {
    const uint64_t result = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
  __device__ double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  __device__ int64_t randint(int64_t n) {
    const uint64_t un = static_cast<uint64_t>(n);
    const uint64_t limit = UINT64_MAX - UINT64_MAX % un;
    uint64_t v = next();
    while (v >= limit) v = next();
    return static_cast<int64_t>(v % un);
  }
};

__device__ __forceinline__ double sq_dist(const double* a, const double* b, int d) {
  double s = 0.0;
  for (int i = 0; i < d; ++i) {
    const double diff = __dsub_rn(a[i], b[i]);
    s = __dadd_rn(s, __dmul_rn(diff, diff));
  }
  return s;
}

struct UserWs {  // per-user global workspace (offsets prepared on the host)
  int* idx;        // [n] point ids, permuted into child ranges
  int* tmp;        // [n]
  int* assign;     // [n]
  int* stack;      // [2 n] (start, len | flag)
  double* d2;      // [n]
  double* cent;    // [kmax * D]
  int* counts;     // [kmax]
  unsigned char* taken;  // [n]
};

__device__ int cube_root_count(int n) {  // kmeans.cpp:133-137
  int c = 0;
  while (static_cast<long long>(c + 1) * (c + 1) * (c + 1) <= n) ++c;
  return c;
}

// kmeans(points[idx[s..s+n)], k, rng) -> assign[0..n) (kmeans.cpp:22-131)
__device__ void kmeans_block(const double* __restrict__ pts, int D, const int* __restrict__ idx, int n, int k,
                             DevRng& rng, UserWs& w) {
  __shared__ int sh_pick;
  __shared__ int sh_conv;
  __shared__ double red_d[kCT];
  __shared__ int red_i[kCT];
  const int tid = threadIdx.x;
  auto P = [&](int r) { return pts + (size_t)idx[r] * D; };
  // k-means++ seeding
  if (tid == 0) sh_pick = static_cast<int>(rng.randint(n));
  __syncthreads();
  for (int j = tid; j < D; j += kCT) w.cent[j] = P(sh_pick)[j];
  for (int r = tid; r < n; r += kCT) w.d2[r] = DBL_MAX;
  __syncthreads();
  for (int c = 1; c < k; ++c) {
    for (int r = tid; r < n; r += kCT) {
      const double d = sq_dist(P(r), w.cent + (size_t)(c - 1) * D, D);
      w.d2[r] = fmin(w.d2[r], d);
    }
    __syncthreads();
    if (tid == 0) {
      double total = 0.0;
      for (int r = 0; r < n; ++r) total = __dadd_rn(total, w.d2[r]);
      int pick = 0;
      if (total > 0) {
        const double rr = __dmul_rn(rng.uniform(), total);
        double acc = 0.0;
        for (int r = 0; r < n; ++r) {
          acc = __dadd_rn(acc, w.d2[r]);
          pick = r;
          if (acc >= rr) break;
        }
      } else {
        pick = static_cast<int>(rng.randint(n));
      }
      sh_pick = pick;
    }
    __syncthreads();
    for (int j = tid; j < D; j += kCT) w.cent[(size_t)c * D + j] = P(sh_pick)[j];
    __syncthreads();
  }
  double prev_obj = DBL_MAX;
  for (int iter = 0; iter < 50; ++iter) {  // KMeansOptions{max_iters = 50, rel_tol = 1e-6}
    // assignment: ties to the lowest centroid
    for (int r = tid; r < n; r += kCT) {
      int best = 0;
      double bd = sq_dist(P(r), w.cent, D);
      for (int c = 1; c < k; ++c) {
        const double d = sq_dist(P(r), w.cent + (size_t)c * D, D);
        if (d < bd) bd = d, best = c;
      }
      w.assign[r] = best;
      w.d2[r] = bd;
    }
    __syncthreads();
    if (tid == 0) {
      double obj = 0.0;
      for (int r = 0; r < n; ++r) obj = __dadd_rn(obj, w.d2[r]);
      sh_conv = prev_obj != DBL_MAX && __dsub_rn(prev_obj, obj) <= 1e-6 * fmax(prev_obj, 1e-300);
      prev_obj = obj;
      for (int c = 0; c < k; ++c) w.counts[c] = 0;
      for (int r = 0; r < n; ++r) ++w.counts[w.assign[r]];
    }
    __syncthreads();
    // update: means of the assigned points, summed in index order
    for (int cj = tid; cj < k * D; cj += kCT) {
      const int c = cj / D, j = cj % D;
      if (w.counts[c] == 0) continue;
      double sum = 0.0;
      for (int r = 0; r < n; ++r)
        if (w.assign[r] == c) sum = __dadd_rn(sum, P(r)[j]);
      w.cent[cj] = __ddiv_rn(sum, static_cast<double>(w.counts[c]));
    }
    for (int r = tid; r < n; r += kCT) w.taken[r] = 0;
    __syncthreads();
    // reseed empty clusters to the farthest point from its assigned centroid
    for (int c = 0; c < k; ++c) {
      if (w.counts[c] > 0) continue;
      double bd = -1.0;
      int bi = -1;
      for (int r = tid; r < n; r += kCT) {
        if (w.taken[r]) continue;
        const double d = sq_dist(P(r), w.cent + (size_t)w.assign[r] * D, D);
        if (d > bd) bd = d, bi = r;  // first maximum in this thread's (ascending) stride
      }
      red_d[tid] = bd;
      red_i[tid] = bi;
      __syncthreads();
      if (tid == 0) {
        double best = -1.0;
        int far = -1;
        for (int t = 0; t < kCT; ++t)
          if (red_i[t] >= 0 && (red_d[t] > best || (red_d[t] == best && red_i[t] < far))) best = red_d[t], far = red_i[t];
        sh_pick = far;
        if (far >= 0) {
          w.taken[far] = 1;
          w.assign[far] = c;
          sh_conv = 0;
        }
      }
      __syncthreads();
      if (sh_pick >= 0)
        for (int j = tid; j < D; j += kCT) w.cent[(size_t)c * D + j] = P(sh_pick)[j];
      __syncthreads();
    }
    if (sh_conv) break;
    __syncthreads();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kCT) compress_kernel(CompressArgs a, const int64_t* __restrict__ ws_off,
                                                       const int64_t* __restrict__ cent_off, int* ws_int,
                                                       double* ws_dbl, unsigned char* ws_u8,
                                                       const uint64_t* __restrict__ rng_state) {
  const int u = blockIdx.x, tid = threadIdx.x;
  const int64_t i0 = a.offsets[u];
  const int n = static_cast<int>(a.offsets[u + 1] - i0);
  const int64_t o0 = a.out_offsets[u];
  const int n_out = static_cast<int>(a.out_offsets[u + 1] - o0);
  const int skip = n - n_out;  // oldest records dropped when n > max_out (policy.cpp:506-507)
  auto emit = [&](int out_i, int src, int rep, double tag, double play, double dur) {
    const int64_t dst = o0 + out_i, s = i0 + src, rp = i0 + rep;
    a.out_vid[dst] = a.vid[rp];
    a.out_aid[dst] = a.aid[rp];
    a.out_labels[dst] = a.labels[rp];
    a.out_tag[dst] = tag;
    a.out_ts[dst] = a.ts[s];
    a.out_playtime[dst] = play;
    a.out_duration[dst] = dur;
    if (a.sid)
      for (int l = 0; l < a.n_code_layers; ++l) a.out_sid[dst * a.n_code_layers + l] = a.sid[rp * a.n_code_layers + l];
  };
  if (n <= a.threshold) {  // kept as is
    for (int i = tid; i < n_out; i += kCT) {
      const int src = skip + i;
      emit(i, src, src, a.tag[i0 + src], a.playtime[i0 + src], a.duration[i0 + src]);
    }
    return;
  }
  UserWs w;
  const int64_t wo = ws_off[u];
  w.idx = ws_int + 6 * wo;
  w.tmp = w.idx + n;
  w.assign = w.tmp + n;
  w.stack = w.assign + n;  // 2 n
  int* labels = w.stack + 2 * n;  // n
  w.d2 = ws_dbl + wo;
  w.cent = ws_dbl + a.total_points + cent_off[u] * a.D;
  w.counts = reinterpret_cast<int*>(ws_u8) + cent_off[u];  // kmax ints per user (u8 arena holds them as ints)
  w.taken = ws_u8 + 4 * a.total_kmax + wo;
  const double* pts = a.content + i0 * a.D;
  DevRng rng;
  for (int q = 0; q < 4; ++q) rng.s[q] = rng_state[4 * u + q];
  __shared__ int sh_sp, sh_next, sh_s, sh_len, sh_flag;
  for (int i = tid; i < n; i += kCT) w.idx[i] = i;
  if (tid == 0) {
    sh_sp = 0;
    sh_next = 0;
    w.stack[0] = 0;
    w.stack[1] = n << 1;
    sh_sp = 1;
  }
  __syncthreads();
  while (true) {  // split_recursive (kmeans.cpp:141-171), depth first
    if (tid == 0) {
      if (sh_sp == 0) {
        sh_len = -1;
      } else {
        --sh_sp;
        sh_s = w.stack[2 * sh_sp];
        sh_len = w.stack[2 * sh_sp + 1] >> 1;
        sh_flag = w.stack[2 * sh_sp + 1] & 1;
      }
    }
    __syncthreads();
    const int s = sh_s, len = sh_len;
    if (len < 0) break;
    if (len <= a.threshold || sh_flag) {  // leaf (or a degenerate split's single child)
      const int lab = sh_next;
      for (int r = tid; r < len; r += kCT) labels[w.idx[s + r]] = lab;
      __syncthreads();
      if (tid == 0) ++sh_next;
      __syncthreads();
      continue;
    }
    const int k = min(max(2, cube_root_count(len)), len);
    kmeans_block(pts, a.D, w.idx + s, len, k, rng, w);
    if (tid == 0) {
      // children in cluster order, members in subset order; pushed reversed so child 0 runs first
      int pos = 0;
      for (int c = 0; c < k; ++c) {
        const int start = pos;
        for (int r = 0; r < len; ++r)
          if (w.assign[r] == c) w.tmp[pos++] = w.idx[s + r];
        w.counts[c] = pos - start;
      }
      for (int r = 0; r < len; ++r) w.idx[s + r] = w.tmp[r];
      int end = s + len;
      for (int c = k - 1; c >= 0; --c) {
        const int cnt = w.counts[c];
        end -= cnt;
        if (cnt == 0) continue;
        w.stack[2 * sh_sp] = end;
        w.stack[2 * sh_sp + 1] = (cnt << 1) | (cnt == len ? 1 : 0);
        ++sh_sp;
      }
    }
    __syncthreads();
  }
  // compress_lifelong (policy.cpp:459-501): leaf members (ascending), centre,
  // representative nearest the centre, mean tag / ts / playtime / duration
  const int n_leaves = sh_next;
  __shared__ double red_d[kCT];
  __shared__ int red_i[kCT];
  int* mem = w.tmp;          // members grouped by leaf
  int* leaf_start = w.stack;  // n_leaves + 1 (n_leaves <= n)
  if (tid == 0) {
    for (int l = 0; l <= n_leaves; ++l) leaf_start[l] = 0;
    for (int i = 0; i < n; ++i) ++leaf_start[labels[i] + 1];
    for (int l = 0; l < n_leaves; ++l) leaf_start[l + 1] += leaf_start[l];
    // stable fill: members ascending per leaf
    for (int i = 0; i < n; ++i) w.assign[i] = 0;
    for (int i = 0; i < n; ++i) {
      const int l = labels[i];
      mem[leaf_start[l] + w.assign[l]++] = i;
    }
  }
  __syncthreads();
  int* rep_of = w.idx;  // leaf -> representative
  for (int l = 0; l < n_leaves; ++l) {
    const int b = leaf_start[l], m = leaf_start[l + 1] - b;
    double* center = w.cent;
    const double inv_m = static_cast<double>(m);
    for (int j = tid; j < a.D; j += kCT) {
      double c = 0.0;
      for (int q = 0; q < m; ++q) c = __dadd_rn(c, __ddiv_rn(pts[(size_t)mem[b + q] * a.D + j], inv_m));
      center[j] = c;
    }
    __syncthreads();
    double bd = DBL_MAX;
    int bq = -1;
    for (int q = tid; q < m; q += kCT) {
      const double d = sq_dist(pts + (size_t)mem[b + q] * a.D, center, a.D);
      if (d < bd) bd = d, bq = q;
    }
    red_d[tid] = bd;
    red_i[tid] = bq;
    __syncthreads();
    if (tid == 0) {
      double best = 1e300;  // policy.cpp:473-483: strict <, first minimum, starting from members[0]
      int rq = 0;
      for (int t = 0; t < kCT; ++t)
        if (red_i[t] >= 0 && (red_d[t] < best || (red_d[t] == best && red_i[t] < rq))) best = red_d[t], rq = red_i[t];
      rep_of[l] = mem[b + rq];
      double tg = 0.0, pl = 0.0, du = 0.0;
      for (int q = 0; q < m; ++q) {
        const int64_t i = i0 + mem[b + q];
        tg = __dadd_rn(tg, __ddiv_rn(a.tag[i], inv_m));
        pl = __dadd_rn(pl, __ddiv_rn(a.playtime[i], inv_m));
        du = __dadd_rn(du, __ddiv_rn(a.duration[i], inv_m));
      }
      pl = fmin(pl, du);  // policy.cpp:495
      a.leaf_tag[wo + l] = tg;
      a.leaf_play[wo + l] = pl;
      a.leaf_dur[wo + l] = du;
    }
    __syncthreads();
  }
  for (int i = tid; i < n_out; i += kCT) {
    const int src = skip + i, l = labels[src];
    emit(i, src, rep_of[l], a.leaf_tag[wo + l], a.leaf_play[wo + l], a.leaf_dur[wo + l]);
  }
}

}  // namespace

void compress_lifelong_gpu(const CompressHost& h, int device) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) {
    cudaGetLastError();
    throw RuntimeError("no CUDA device available (the engine has no CPU fallback)");
  }
  require(device >= 0 && device < ndev, "device index out of range");
  require(h.threshold >= 1, "hierarchical_clusters: threshold must be >= 1");
  require(h.max_out >= 1, "compress_lifelong: max_out must be >= 1");
  require(h.D >= 1, "compress_lifelong: content width must be >= 1");
  cudaSetDevice(device);
  const int U = h.n_users;
  std::vector<int64_t> out_off(U + 1, 0), ws_off(U + 1, 0), cent_off(U + 1, 0);
  for (int u = 0; u < U; ++u) {
    const int64_t n = h.offsets[u + 1] - h.offsets[u];
    require(n >= 0, "offsets must be non-decreasing");
    out_off[u + 1] = out_off[u] + std::min<int64_t>(n, h.max_out);
    ws_off[u + 1] = ws_off[u] + n;
    int64_t c = 0;
    while ((c + 1) * (c + 1) * (c + 1) <= n) ++c;
    cent_off[u + 1] = cent_off[u] + std::max<int64_t>(2, c);
  }
  const int64_t N = ws_off[U], K = cent_off[U];
  require(N < (int64_t(1) << 30), "compress_lifelong: too many records");
  // device arenas
  std::vector<void*> allocs;
  auto dalloc = [&](size_t bytes) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(bytes, 16)) != cudaSuccess) {
      for (void* q : allocs) cudaFree(q);
      throw RuntimeError("CUDA: out of memory in compress_lifelong");
    }
    allocs.push_back(p);
    return p;
  };
  auto up = [&](const void* src, size_t bytes) {
    void* p = dalloc(bytes);
    if (bytes) cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice);
    return p;
  };
  const int L = h.n_code_layers;
  CompressArgs a{};
  a.D = h.D;
  a.threshold = h.threshold;
  a.n_code_layers = L;
  a.total_points = N;
  a.total_kmax = K;
  a.offsets = static_cast<int64_t*>(up(h.offsets, (U + 1) * 8));
  a.out_offsets = static_cast<int64_t*>(up(out_off.data(), (U + 1) * 8));
  a.vid = static_cast<int64_t*>(up(h.vid, N * 8));
  a.aid = static_cast<int32_t*>(up(h.aid, N * 4));
  a.labels = static_cast<uint32_t*>(up(h.labels, N * 4));
  a.tag = static_cast<double*>(up(h.tag, N * 8));
  a.ts = static_cast<double*>(up(h.ts, N * 8));
  a.playtime = static_cast<double*>(up(h.playtime, N * 8));
  a.duration = static_cast<double*>(up(h.duration, N * 8));
  a.sid = h.sid ? static_cast<int32_t*>(up(h.sid, N * L * 4)) : nullptr;
  a.content = static_cast<double*>(up(h.content, N * h.D * 8));
  const int64_t NO = out_off[U];
  a.out_vid = static_cast<int64_t*>(dalloc(NO * 8));
  a.out_aid = static_cast<int32_t*>(dalloc(NO * 4));
  a.out_labels = static_cast<uint32_t*>(dalloc(NO * 4));
  a.out_tag = static_cast<double*>(dalloc(NO * 8));
  a.out_ts = static_cast<double*>(dalloc(NO * 8));
  a.out_playtime = static_cast<double*>(dalloc(NO * 8));
  a.out_duration = static_cast<double*>(dalloc(NO * 8));
  a.out_sid = h.sid ? static_cast<int32_t*>(dalloc(NO * L * 4)) : nullptr;
  a.leaf_tag = static_cast<double*>(dalloc(N * 8));
  a.leaf_play = static_cast<double*>(dalloc(N * 8));
  a.leaf_dur = static_cast<double*>(dalloc(N * 8));
  std::vector<uint64_t> st(static_cast<size_t>(U) * 4);
  for (int u = 0; u < U; ++u) {
    Rng r(h.rng_seeds[u]);
    for (int q = 0; q < 4; ++q) st[4 * u + q] = r.s_[q];
  }
  auto* d_state = static_cast<uint64_t*>(up(st.data(), st.size() * 8));
  auto* d_wsoff = static_cast<int64_t*>(up(ws_off.data(), (U + 1) * 8));
  auto* d_centoff = static_cast<int64_t*>(up(cent_off.data(), (U + 1) * 8));
  auto* ws_int = static_cast<int*>(dalloc(static_cast<size_t>(N) * 6 * 4));
  auto* ws_dbl = static_cast<double*>(dalloc((static_cast<size_t>(N) + static_cast<size_t>(K) * h.D) * 8));
  auto* ws_u8 = static_cast<unsigned char*>(dalloc(static_cast<size_t>(K) * 4 + N));
  if (U > 0) compress_kernel<<<U, kCT>>>(a, d_wsoff, d_centoff, ws_int, ws_dbl, ws_u8, d_state);
  cudaError_t err = cudaDeviceSynchronize();
  if (err == cudaSuccess) err = cudaGetLastError();
  if (err == cudaSuccess) {
    auto down = [&](void* dst, const void* src, size_t bytes) {
      if (bytes) cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost);
    };
    h.out_offsets[0] = 0;
    for (int u = 0; u < U; ++u) h.out_offsets[u + 1] = out_off[u + 1];
    down(h.out_vid, a.out_vid, NO * 8);
    down(h.out_aid, a.out_aid, NO * 4);
    down(h.out_labels, a.out_labels, NO * 4);
    down(h.out_tag, a.out_tag, NO * 8);
    down(h.out_ts, a.out_ts, NO * 8);
    down(h.out_playtime, a.out_playtime, NO * 8);
    down(h.out_duration, a.out_duration, NO * 8);
    if (h.sid && h.out_sid) down(h.out_sid, a.out_sid, NO * L * 4);
  }
  for (void* p : allocs) cudaFree(p);
  if (err != cudaSuccess) throw RuntimeError(std::string("CUDA: ") + cudaGetErrorString(err));
  ++launch_counter();
}

}  // namespace orx
