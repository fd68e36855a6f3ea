// Expert placement and the per-exchange plan of an expert-parallel engine
// (SURVEY.md §8(e)). Plain C++ (no CUDA): the engine uploads the placement
// tables, the device plan (ep_plan_kernel, kernels.cu) computes the same
// layout as ep_plan_placed below, and the CPU tests drive this restatement
// through the C-ABI.
//
// Placement: owner[li * E + e] = the rank that computes expert e of MoE layer
// li, or -1 = replicated (every rank holds the expert and computes it for its
// own tokens, so those rows never cross NVLink). Rank p's local slots of layer
// li are the replicated experts (ascending id) followed by the experts it owns
// (ascending id); slot[li * E + e] is e's slot index on the rank(s) computing
// it. The default placement is contiguous blocks of E / W experts per rank.
//
// Exchange layout (one MoE call, cnt[q * E + e] = rows rank q routes to
// expert e, all-gathered): rank p's receive buffer holds, per local slot j
// in order, the rows of expert g = list[p][j] -- every rank's rows, source-rank
// major, for an owned expert; p's own rows for a replicated one -- padded to
// `tile` rows for the grouped GEMM.
#pragma once

#include <algorithm>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <vector>

namespace orx {

struct EpPlacement {
  int layers = 0, E = 0, W = 1;
  std::vector<int32_t> owner;  // [layers][E]

  static EpPlacement contiguous(int layers, int E, int W) {
    if (W < 1 || E % W != 0) throw std::invalid_argument("expert count must divide evenly over the ranks");
    EpPlacement p;
    p.layers = layers, p.E = E, p.W = W;
    p.owner.resize(static_cast<size_t>(layers) * E);
    for (int li = 0; li < layers; ++li)
      for (int e = 0; e < E; ++e) p.owner[static_cast<size_t>(li) * E + e] = e / (E / W);
    return p;
  }
  void validate() const {
    if (W < 1 || E < 1 || E > 32 || owner.size() != static_cast<size_t>(layers) * E)
      throw std::invalid_argument("expert placement: bad shape (at most 32 experts)");
    for (int32_t o : owner)
      if (o < -1 || o >= W) throw std::invalid_argument("expert placement: owner must be -1 or a rank");
    if (capacity() > 32) throw std::invalid_argument("expert placement: more than 32 local experts per rank");
  }
  // local experts of rank p in layer li (replicated first, then owned; ascending ids)
  std::vector<int> local(int li, int p) const {
    std::vector<int> out;
    for (int pass = 0; pass < 2; ++pass)
      for (int e = 0; e < E; ++e) {
        const int o = owner[static_cast<size_t>(li) * E + e];
        if ((pass == 0 && o < 0) || (pass == 1 && o == p)) out.push_back(e);
      }
    return out;
  }
  // local slots per rank (the weight buffers and grouped GEMMs are sized for it)
  int capacity() const {
    int c = 0;
    for (int li = 0; li < layers; ++li)
      for (int p = 0; p < W; ++p) c = std::max(c, static_cast<int>(local(li, p).size()));
    return c;
  }
  // list[(li * W + p) * C + j] = global expert of slot j on rank p (-1 = empty);
  // slot[li * E + e] = e's slot on the rank(s) computing it
  void tables(int C, std::vector<int32_t>& list, std::vector<int32_t>& slot) const {
    list.assign(static_cast<size_t>(layers) * W * C, -1);
    slot.assign(static_cast<size_t>(layers) * E, -1);
    for (int li = 0; li < layers; ++li)
      for (int p = 0; p < W; ++p) {
        const std::vector<int> l = local(li, p);
        for (size_t j = 0; j < l.size(); ++j) {
          list[(static_cast<size_t>(li) * W + p) * C + j] = l[j];
          slot[static_cast<size_t>(li) * E + l[j]] = static_cast<int32_t>(j);
        }
      }
  }
  bool operator==(const EpPlacement& o) const {
    return layers == o.layers && E == o.E && W == o.W && owner == o.owner;
  }
};

// Load-balanced placement from per-layer expert loads (rows routed to each
// expert, summed over every rank and some calls; EngineT accumulates them).
// Per layer, for r = min_replicas .. max_replicas: the r heaviest experts are replicated
// (their load splits evenly over the ranks, as the token batches do) and the
// rest are packed onto the ranks heaviest-first, each to the least-loaded rank
// with a free slot (at most ceil((E - r) / W) + 1 owned experts per rank),
// then refined by moves / swaps that lower the busiest rank's load; the first
// r whose busiest rank is within `tolerance` of the mean wins, else the best
// r. A replicated expert's rows never cross NVLink, so min_replicas > 0
// trades expert memory for exchange traffic. Deterministic: every rank
// computes the same placement from the same (all-gathered) loads.
inline EpPlacement ep_place_balanced(const int64_t* load, int layers, int E, int W, int max_replicas,
                                     double tolerance = 1.05, std::vector<double>* predicted = nullptr,
                                     int min_replicas = 0) {
  if (W < 1 || E < 1 || E > 32 || layers < 0 || max_replicas < 0 || min_replicas < 0 || min_replicas > max_replicas)
    throw std::invalid_argument("ep_place: bad layers / experts / world / replicas");
  EpPlacement p;
  p.layers = layers, p.E = E, p.W = W;
  p.owner.assign(static_cast<size_t>(layers) * E, 0);
  if (predicted) predicted->assign(static_cast<size_t>(layers), 1.0);
  for (int li = 0; li < layers; ++li) {
    const int64_t* l = load + static_cast<size_t>(li) * E;
    std::vector<int> order(E);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return l[a] > l[b]; });
    double total = 0;
    for (int e = 0; e < E; ++e) total += static_cast<double>(l[e]);
    const double mean = total / W;
    std::vector<int32_t> best;
    double best_imb = 1e300;
    for (int r = std::min(min_replicas, E); r <= std::min(max_replicas, E); ++r) {
      std::vector<int32_t> own(E, -1);
      std::vector<double> rank_load(W, 0.0);
      std::vector<int> n_owned(W, 0);
      double repl = 0;
      for (int i = 0; i < r; ++i) repl += static_cast<double>(l[order[i]]);
      for (int q = 0; q < W; ++q) rank_load[q] = repl / W;
      const int cap = (E - r + W - 1) / W + 1;
      for (int i = r; i < E; ++i) {
        int pick = -1;
        for (int q = 0; q < W; ++q)
          if (n_owned[q] < cap && (pick < 0 || rank_load[q] < rank_load[pick])) pick = q;
        own[order[i]] = pick;
        rank_load[pick] += static_cast<double>(l[order[i]]);
        ++n_owned[pick];
      }
      // refinement: move one expert off the busiest rank, or swap it for a
      // lighter one, whichever lowers the pair's maximum the most
      for (int it = 0; it < 4 * E; ++it) {
        const int b = static_cast<int>(std::max_element(rank_load.begin(), rank_load.end()) - rank_load.begin());
        double best_max = rank_load[b];
        int bx = -1, bq = -1, by = -1;
        for (int x = 0; x < E; ++x) {
          if (own[x] != b) continue;
          const double lx = static_cast<double>(l[x]);
          for (int q = 0; q < W; ++q) {
            if (q == b) continue;
            if (n_owned[q] < cap) {
              const double m = std::max(rank_load[b] - lx, rank_load[q] + lx);
              if (m < best_max - 1e-9) best_max = m, bx = x, bq = q, by = -1;
            }
            for (int y = 0; y < E; ++y) {
              if (own[y] != q || l[y] >= l[x]) continue;
              const double dl = lx - static_cast<double>(l[y]);
              const double m = std::max(rank_load[b] - dl, rank_load[q] + dl);
              if (m < best_max - 1e-9) best_max = m, bx = x, bq = q, by = y;
            }
          }
        }
        if (bx < 0) break;
        const double lx = static_cast<double>(l[bx]), ly = by < 0 ? 0.0 : static_cast<double>(l[by]);
        own[bx] = bq;
        rank_load[b] -= lx - ly;
        rank_load[bq] += lx - ly;
        if (by >= 0) {
          own[by] = b;
        } else {
          --n_owned[b];
          ++n_owned[bq];
        }
      }
      const double imb = mean > 0 ? *std::max_element(rank_load.begin(), rank_load.end()) / mean : 1.0;
      if (imb < best_imb - 1e-12) best_imb = imb, best = own;
      if (imb <= tolerance) break;
    }
    std::copy(best.begin(), best.end(), p.owner.begin() + static_cast<size_t>(li) * E);
    if (predicted) (*predicted)[li] = best_imb;
  }
  return p;
}

// Host restatement of ep_plan_kernel for rank `rank`: cursor[e] = first row
// of this rank's expert-e rows in the destination buffer (destination rank =
// owner, or this rank for a replicated expert); seg[2j], seg[2j+1] = start and
// row count of local slot j; tiles[i] = local slot of grouped-GEMM M tile i
// (-1 past the end). Returns the rows this rank's buffer needs.
inline int64_t ep_plan_placed(int W, int rank, int E, const int32_t* cnt, const int32_t* owner, int tile,
                              int max_tiles, int32_t* cursor, int32_t* seg, int C, int32_t* tiles,
                              int32_t* n_tiles) {
  if (W < 1 || rank < 0 || rank >= W || E < 1 || E > 32 || tile < 1)
    throw std::invalid_argument("ep_plan: bad world / rank / expert count / tile");
  EpPlacement pl;
  pl.layers = 1, pl.E = E, pl.W = W;
  pl.owner.assign(owner, owner + E);
  pl.validate();
  if (C < pl.capacity()) throw std::invalid_argument("ep_plan: slot capacity below the placement's");
  std::vector<int32_t> list, slot;
  pl.tables(C, list, slot);
  std::vector<int64_t> tot(E, 0);
  for (int e = 0; e < E; ++e)
    for (int q = 0; q < W; ++q) tot[e] += cnt[static_cast<size_t>(q) * E + e];
  std::vector<int64_t> start(static_cast<size_t>(W) * C), rows(static_cast<size_t>(W) * C);
  int64_t need = 0;
  for (int p = 0; p < W; ++p) {
    int64_t off = 0;
    for (int j = 0; j < C; ++j) {
      const int g = list[static_cast<size_t>(p) * C + j];
      const int64_t n = g < 0 ? 0 : (owner[g] < 0 ? cnt[static_cast<size_t>(p) * E + g] : tot[g]);
      start[static_cast<size_t>(p) * C + j] = off;
      rows[static_cast<size_t>(p) * C + j] = n;
      off += (n + tile - 1) / tile * tile;
    }
    if (p == rank) need = off;
  }
  for (int e = 0; e < E; ++e) {
    const int dest = owner[e] < 0 ? rank : owner[e];
    int64_t before = 0;
    if (owner[e] >= 0)
      for (int q = 0; q < rank; ++q) before += cnt[static_cast<size_t>(q) * E + e];
    cursor[e] = static_cast<int32_t>(start[static_cast<size_t>(dest) * C + slot[e]] + before);
  }
  int nt = 0;
  for (int j = 0; j < C; ++j) {
    const int64_t n = rows[static_cast<size_t>(rank) * C + j];
    seg[2 * j] = static_cast<int32_t>(start[static_cast<size_t>(rank) * C + j]);
    seg[2 * j + 1] = static_cast<int32_t>(n);
    for (int64_t i = 0; i < (n + tile - 1) / tile; ++i) {
      if (nt >= max_tiles) throw std::runtime_error("ep_plan: grouped tile table overflow");
      tiles[nt++] = j;
    }
  }
  for (int i = nt; i < max_tiles; ++i) tiles[i] = -1;
  *n_tiles = nt;
  return need;
}

}  // namespace orx
