// Host-side plan of one expert-parallel MoE exchange.
//
// Input: cnt[p * E + e] = rows rank p routes to (global) expert e, for every
// rank p (an all-gather of the per-rank routing histograms). Rank r owns
// experts [r * El, (r + 1) * El).
//   send  : rank r sends its rows sorted by expert; the rows for rank p's
//           experts are the contiguous block [send_off[p], +send_cnt[p]).
//   recv  : from rank p it receives recv_cnt[p] rows at recv_off[p], sorted
//           by (local) expert.
//   group : received rows are regrouped expert-major, source-rank minor,
//           each expert's segment padded to `tile` rows for the grouped GEMM:
//           tab[(p * El + el) * 3 + {0,1,2}] = (src row, dst row, count) and
//           tiles[i] = local expert of grouped-GEMM M tile i (-1 past the end).
// Plain C++ (no CUDA) so the CPU tests can call it through the C-ABI.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <vector>

namespace orx {

struct EpPlan {
  std::vector<int64_t> send_cnt, send_off, recv_cnt, recv_off;
  int64_t total_send = 0, total_recv = 0;
  int n_tiles = 0;  // grouped-GEMM M tiles in use
};

inline EpPlan ep_plan(int W, int rank, int E, const int32_t* cnt, int tile, int max_tiles, int32_t* tab,
                      int32_t* tiles) {
  if (W < 1 || rank < 0 || rank >= W || E % W != 0 || tile < 1)
    throw std::invalid_argument("ep_plan: bad world / rank / expert count / tile");
  const int El = E / W, e0 = rank * El;
  EpPlan pl;
  pl.send_cnt.assign(W, 0);
  pl.send_off.assign(W, 0);
  pl.recv_cnt.assign(W, 0);
  pl.recv_off.assign(W, 0);
  for (int p = 0; p < W; ++p)
    for (int e = p * El; e < (p + 1) * El; ++e) pl.send_cnt[p] += cnt[static_cast<size_t>(rank) * E + e];
  for (int p = 0; p < W; ++p)
    for (int e = e0; e < e0 + El; ++e) pl.recv_cnt[p] += cnt[static_cast<size_t>(p) * E + e];
  for (int p = 1; p < W; ++p) {
    pl.send_off[p] = pl.send_off[p - 1] + pl.send_cnt[p - 1];
    pl.recv_off[p] = pl.recv_off[p - 1] + pl.recv_cnt[p - 1];
  }
  pl.total_send = pl.send_off[W - 1] + pl.send_cnt[W - 1];
  pl.total_recv = pl.recv_off[W - 1] + pl.recv_cnt[W - 1];
  int64_t dst = 0;
  for (int el = 0; el < El; ++el) {
    int64_t r_e = 0;
    for (int p = 0; p < W; ++p) {
      int64_t src = pl.recv_off[p];
      for (int e2 = e0; e2 < e0 + el; ++e2) src += cnt[static_cast<size_t>(p) * E + e2];
      const int n = cnt[static_cast<size_t>(p) * E + e0 + el];
      int32_t* t = tab + 3 * (static_cast<size_t>(p) * El + el);
      t[0] = static_cast<int32_t>(src);
      t[1] = static_cast<int32_t>(dst + r_e);
      t[2] = n;
      r_e += n;
    }
    const int nt = static_cast<int>((r_e + tile - 1) / tile);
    for (int i = 0; i < nt; ++i) {
      if (pl.n_tiles >= max_tiles) throw std::runtime_error("ep_plan: grouped tile table overflow");
      tiles[pl.n_tiles++] = el;
    }
    dst += static_cast<int64_t>(nt) * tile;
  }
  for (int i = pl.n_tiles; i < max_tiles; ++i) tiles[i] = -1;
  return pl;
}

}  // namespace orx
