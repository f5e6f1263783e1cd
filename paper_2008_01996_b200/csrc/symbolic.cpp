// Nested-dissection symbolic analysis (host C++). See symbolic.h.
//
// Ordering: recursive graph bisection. For each connected vertex set a
// pseudo-peripheral BFS level structure is built (from both ends of the
// pseudo-diameter); the separator is the smallest level whose two sides are
// within 2:1 of each other, thinned by moving separator vertices without an
// upper-side neighbour to the lower side. Sets at or below `leaf_size`
// vertices become dense leaf fronts. Every separator is one supernode, so
// every front has a dense p x p pivot block and a sorted list of q update
// rows; the elimination order is the postorder of the dissection tree, which
// is what the reference's etree postorder achieves for its MMD ordering
// (sparse_direct.py:71-109, :144-145).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include "symbolic.h"

#include <algorithm>
#include <cstdio>
#include <numeric>
#include <atomic>
#include <thread>

namespace kh {
namespace {
std::atomic<long long> g_sep_ns[8];

struct Graph {
  int64_t n = 0;
  std::vector<int64_t> xadj, adj;
};

// rows [0, n) split over up to 8 threads: fn(r0, r1)
template <class F>
void parallel_rows(int64_t n, F fn) {
  const int nth = (int)std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  if (n < 4096 || nth == 1) {
    fn((int64_t)0, n);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 1; t < nth; ++t) th.emplace_back(fn, n * t / nth, n * (t + 1) / nth);
  fn((int64_t)0, n / nth);
  for (auto& x : th) x.join();
}

// Fast path of build_graph: a canonical (rows sorted, no duplicates) and
// structurally symmetric pattern -- what scipy hands over for M + A -- is its
// own graph minus the diagonal. Returns false if the pattern is not of that kind.
bool graph_from_symmetric(int64_t n, const int64_t* indptr, const int64_t* indices, Graph& g) {
  std::atomic<bool> ok{true};
  parallel_rows(n, [&](int64_t r0, int64_t r1) {
    for (int64_t i = r0; i < r1 && ok.load(std::memory_order_relaxed); ++i)
      for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
        const int64_t j = indices[e];
        if (e > indptr[i] && indices[e - 1] >= j) { ok = false; break; }
        if (j == i) continue;
        if (!std::binary_search(indices + indptr[j], indices + indptr[j + 1], i)) { ok = false; break; }
      }
  });
  if (!ok) return false;
  g.n = n;
  g.xadj.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    int64_t d = indptr[i + 1] - indptr[i];
    for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) d -= indices[e] == i;
    g.xadj[i + 1] = g.xadj[i] + d;
  }
  g.adj.resize(g.xadj[n]);
  parallel_rows(n, [&](int64_t r0, int64_t r1) {
    for (int64_t i = r0; i < r1; ++i) {
      int64_t w = g.xadj[i];
      for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e)
        if (indices[e] != i) g.adj[w++] = indices[e];
    }
  });
  return true;
}

Graph build_graph(int64_t n, const int64_t* indptr, const int64_t* indices) {
  Graph g;
  if (graph_from_symmetric(n, indptr, indices, g)) return g;
  g.n = n;
  std::vector<int64_t> deg(n, 0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
      int64_t j = indices[e];
      if (j != i) { ++deg[i]; ++deg[j]; }
    }
  g.xadj.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) g.xadj[i + 1] = g.xadj[i] + deg[i];
  g.adj.resize(g.xadj[n]);
  std::vector<int64_t> fill(g.xadj.begin(), g.xadj.end() - 1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
      int64_t j = indices[e];
      if (j != i) { g.adj[fill[i]++] = j; g.adj[fill[j]++] = i; }
    }
  // sort + unique each row, then compact
  int64_t w = 0;
  std::vector<int64_t> nx(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    auto b = g.adj.begin() + g.xadj[i], e = g.adj.begin() + g.xadj[i + 1];
    std::sort(b, e);
    auto last = std::unique(b, e);
    nx[i] = w;
    for (auto it = b; it != last; ++it) g.adj[w++] = *it;
  }
  nx[n] = w;
  g.adj.resize(w);
  g.xadj.swap(nx);
  return g;
}

// A dissection subtree in local postorder: piv[f] are the pivots (original
// ids) of local front f, kids[f] its children (local indices).
struct Sub {
  std::vector<std::vector<int64_t>> piv;
  std::vector<std::vector<int32_t>> kids;
};

// Shared, thread-safe state: vertex sets handled concurrently are disjoint,
// so `dist` is only written for a thread's own vertices; `in_set` stamps are
// globally unique (atomic counter) and read with relaxed atomics.
struct Shared {
  const Graph& g;
  int32_t leaf;
  std::vector<std::atomic<int32_t>> in_set;
  std::vector<int32_t> dist, dist2;  // two level structures per vertex set (both ends of the diameter)
  std::atomic<int32_t> stamp{0};
  Shared(const Graph& gr, int32_t lf) : g(gr), leaf(lf), in_set(gr.n), dist(gr.n, -1), dist2(gr.n, -1) {
    for (auto& x : in_set) x.store(0, std::memory_order_relaxed);
  }
};

struct Builder {
  Shared& sh;
  const Graph& g;
  std::vector<int64_t> queue;  // per-thread BFS queue, sized to the largest set it handles

  explicit Builder(Shared& s) : sh(s), g(s.g) {}

  int32_t in(int64_t v) const { return sh.in_set[v].load(std::memory_order_relaxed); }
  void mark(int64_t v, int32_t s) { sh.in_set[v].store(s, std::memory_order_relaxed); }

  // BFS restricted to vertices stamped s; fills queue and level starts.
  int64_t bfs(int64_t root, int32_t s, std::vector<int64_t>& lvl_start) {
    return bfs_into(root, s, lvl_start, queue, sh.dist);
  }
  int64_t bfs_into(int64_t root, int32_t s, std::vector<int64_t>& lvl_start, std::vector<int64_t>& q,
                   std::vector<int32_t>& dist) {
    lvl_start.clear();
    int64_t head = 0, tail = 0;
    q[tail++] = root;
    dist[root] = 0;
    int32_t cur = -1;
    while (head < tail) {
      int64_t v = q[head];
      const int32_t dv = dist[v];
      if (dv != cur) { cur = dv; lvl_start.push_back(head); }
      ++head;
      for (int64_t e = g.xadj[v]; e < g.xadj[v + 1]; ++e) {
        int64_t u = g.adj[e];
        if (dist[u] < 0 && in(u) == s) { dist[u] = dv + 1; q[tail++] = u; }
      }
    }
    lvl_start.push_back(tail);
    return tail;
  }

  // A rooted level structure of the current set: BFS order, level starts and
  // per-vertex levels (in one of the two shared dist arrays).
  struct Levels {
    std::vector<int64_t> order, ls;
    std::vector<int32_t>* dist = nullptr;
    int64_t N = 0;
  };
  Levels lv[2];  // per-thread level-structure slots
  void levels(int64_t root, int32_t s, const std::vector<int64_t>& V, Levels& L) {
    if (L.order.size() < V.size()) L.order.resize(V.size());
    for (int64_t v : V) (*L.dist)[v] = -1;
    L.N = bfs_into(root, s, L.ls, L.order, *L.dist);
  }

  void reset_dist(const std::vector<int64_t>& V) {
    for (int64_t v : V) sh.dist[v] = -1;
  }

  int64_t deg_in(int64_t v, int32_t s) const {
    int64_t d = 0;
    for (int64_t e = g.xadj[v]; e < g.xadj[v + 1]; ++e) d += (in(g.adj[e]) == s);
    return d;
  }

  struct Cut {
    bool ok = false;
    std::vector<int64_t> sep;
    int64_t sep_size = 0;
    double ratio = 1e30;
  };

  // Separator from a rooted BFS level structure.
  Cut cut_from(const Levels& L, int32_t s) {
    Cut c;
    const std::vector<int64_t>& ls = L.ls;
    const std::vector<int64_t>& order = L.order;
    const std::vector<int32_t>& dist = *L.dist;
    const int64_t N = L.N;
    int64_t e = (int64_t)ls.size() - 2;  // eccentricity
    if (e < 2) return c;
    int64_t best = -1;
    for (int64_t l = 1; l < e; ++l) {
      int64_t below = ls[l], size = ls[l + 1] - ls[l], above = N - ls[l + 1];
      if (below == 0 || above == 0) continue;
      double r = (double)std::max(below, above) / (double)std::min(below, above);
      if (r > 2.0) continue;
      if (best < 0 || size < c.sep_size || (size == c.sep_size && r < c.ratio)) {
        best = l; c.sep_size = size; c.ratio = r;
      }
    }
    if (best < 0) {  // fall back to the median level
      for (int64_t l = 1; l < e; ++l)
        if (ls[l + 1] > N / 2) { best = l; break; }
      if (best < 0) best = e - 1;
      int64_t below = ls[best], above = N - ls[best + 1];
      c.ratio = (double)std::max(below, above) / (double)std::max<int64_t>(1, std::min(below, above));
    }
    // thin: a level-l vertex without a neighbour at level l+1 joins the lower side
    for (int64_t k = ls[best]; k < ls[best + 1]; ++k) {
      int64_t v = order[k];
      bool up = false;
      for (int64_t a = g.xadj[v]; a < g.xadj[v + 1] && !up; ++a) {
        int64_t u = g.adj[a];
        up = (in(u) == s && dist[u] == best + 1);
      }
      if (up) c.sep.push_back(v);
    }
    c.sep_size = (int64_t)c.sep.size();
    c.ok = c.sep_size > 0;
    return c;
  }

  // Connected components of the set stamped `s` (components in order of their
  // first vertex in V; each keeps V's order, so sorted V gives sorted parts):
  // BFS labels, then one distributing pass over V (no per-part sort).
  std::vector<std::vector<int64_t>> components(const std::vector<int64_t>& V, int32_t s) {
    std::vector<std::vector<int64_t>> parts;
    reset_dist(V);
    std::vector<int64_t> ls, sizes;
    std::vector<int32_t>& lab = sh.dist2;
    for (int64_t v : V) {
      if (in(v) != s || sh.dist[v] >= 0) continue;
      const int64_t N = bfs(v, s, ls);
      const int32_t id = (int32_t)sizes.size();
      for (int64_t k = 0; k < N; ++k) lab[queue[k]] = id;
      sizes.push_back(N);
    }
    parts.resize(sizes.size());
    for (size_t k = 0; k < sizes.size(); ++k) parts[k].reserve(sizes[k]);
    for (int64_t v : V)
      if (in(v) == s) parts[lab[v]].push_back(v);
    return parts;
  }

  static Sub leaf_sub(std::vector<int64_t> V) {
    std::sort(V.begin(), V.end());
    Sub out;
    out.piv.push_back(std::move(V));
    out.kids.emplace_back();
    return out;
  }

  // Dissect V (a connected set). Large independent parts near the top of
  // the tree are dissected by separate threads (each with its own Builder).
  Sub nd(std::vector<int64_t> V, int depth) {
    if ((int64_t)V.size() <= sh.leaf) return leaf_sub(std::move(V));
    auto T0 = std::chrono::steady_clock::now();
    if (queue.size() < V.size()) queue.resize(V.size());
    int32_t s = ++sh.stamp;
    for (int64_t v : V) mark(v, s);
    // pseudo-peripheral pair (a, b); the level structures rooted at both are
    // kept (two slots) and reused by the cuts below instead of recomputed
    int64_t r = V[0];
    int64_t ecc = -1, b = r;
    lv[0].dist = &sh.dist;
    lv[1].dist = &sh.dist2;
    int cur = 0, sa = -1, sb = -1;  // slot of the last BFS; slots rooted at a and at b
    for (int it = 0; it < 4; ++it) {
      levels(r, s, V, lv[cur]);
      const std::vector<int64_t>& ls = lv[cur].ls;
      int64_t e = (int64_t)ls.size() - 2;
      if (e <= ecc) {  // the BFS from b did not go further: it is b's structure
        sb = cur;
        break;
      }
      ecc = e;
      sa = cur;
      int64_t bestv = -1, bestd = 0;
      for (int64_t k = ls[e]; k < lv[cur].N; ++k) {
        int64_t v = lv[cur].order[k];
        int64_t d = deg_in(v, s);
        if (bestv < 0 || d < bestd) { bestv = v; bestd = d; }
      }
      b = bestv;
      r = bestv;
      cur ^= 1;
    }
    if (sb < 0) {  // four improving rounds: b not yet searched
      sb = sa ^ 1;
      levels(b, s, V, lv[sb]);
    }
    Cut ca = cut_from(lv[sa], s);
    Cut cb = cut_from(lv[sb], s);
    Cut* c = nullptr;
    if (ca.ok && cb.ok) {
      bool a_bal = ca.ratio <= 2.0, b_bal = cb.ratio <= 2.0;
      if (a_bal != b_bal) c = a_bal ? &ca : &cb;
      else c = (ca.sep_size <= cb.sep_size) ? &ca : &cb;
    } else if (ca.ok) {
      c = &ca;
    } else if (cb.ok) {
      c = &cb;
    }
    if (c == nullptr || c->sep_size * 2 > (int64_t)V.size()) return leaf_sub(std::move(V));
    std::vector<int64_t> sep = std::move(c->sep);
    int32_t s2 = ++sh.stamp;
    for (int64_t v : V) mark(v, s2);
    for (int64_t v : sep) mark(v, 0);
    auto parts = components(V, s2);
    if (depth < 8) g_sep_ns[depth] += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - T0).count();
    const size_t nV = V.size();
    std::vector<int64_t>().swap(V);
    std::vector<Sub> subs(parts.size());
    const bool par = depth < 6 && nV > 4096 && parts.size() > 1;

    if (par) {
      std::vector<std::thread> th;
      for (size_t k = 1; k < parts.size(); ++k)
        th.emplace_back([this, &subs, &parts, k, depth] {
          Builder sub(sh);
          subs[k] = sub.nd(std::move(parts[k]), depth + 1);
        });
      subs[0] = nd(std::move(parts[0]), depth + 1);
      for (auto& t : th) t.join();
    } else {
      for (size_t k = 0; k < parts.size(); ++k) subs[k] = nd(std::move(parts[k]), depth + 1);
    }
    Sub out;
    std::vector<int32_t> roots;
    for (auto& sb : subs) {
      const int32_t off = (int32_t)out.piv.size();
      for (auto& kk : sb.kids)
        for (auto& x : kk) x += off;
      for (auto& pv : sb.piv) out.piv.push_back(std::move(pv));
      for (auto& kk : sb.kids) out.kids.push_back(std::move(kk));
      roots.push_back((int32_t)out.piv.size() - 1);
    }
    std::sort(sep.begin(), sep.end());
    out.piv.push_back(std::move(sep));
    out.kids.push_back(std::move(roots));
    return out;
  }
};

}  // namespace

std::string analyze(int64_t n, const int64_t* indptr, const int64_t* indices,
                    int32_t leaf_size, Symbolic& S) {
  // KH_ANALYZE_TIMING=1 prints the phase times to stderr (tuning aid)
  const bool timing = std::getenv("KH_ANALYZE_TIMING") != nullptr;
  auto tp = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "kh_analyze %-10s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - tp).count());
    tp = now;
  };
  if (n < 0) return "negative dimension";
  if (leaf_size < 1) leaf_size = 1;
  for (int64_t i = 0; i < n; ++i)
    if (indptr[i + 1] < indptr[i]) return "indptr not monotone";
  for (int64_t e = 0; e < (n ? indptr[n] : 0); ++e)
    if (indices[e] < 0 || indices[e] >= n) return "column index out of range";
  S = Symbolic();
  S.n = n;
  S.leaf_size = leaf_size;
  Graph g = build_graph(n, indptr, indices);
  // canonical analyzed CSR: graph rows (sorted, unique, no self loops) plus
  // the diagonal in place
  S.pat_ptr.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) S.pat_ptr[i + 1] = S.pat_ptr[i] + (g.xadj[i + 1] - g.xadj[i]) + 1;
  S.pat_idx.resize(S.pat_ptr[n]);
  parallel_rows(n, [&](int64_t r0, int64_t r1) {
    for (int64_t i = r0; i < r1; ++i) {
      int64_t w = S.pat_ptr[i];
      bool diag = false;
      for (int64_t e = g.xadj[i]; e < g.xadj[i + 1]; ++e) {
        if (!diag && g.adj[e] > i) { S.pat_idx[w++] = i; diag = true; }
        S.pat_idx[w++] = g.adj[e];
      }
      if (!diag) S.pat_idx[w++] = i;
    }
  });
  S.nnz = S.pat_ptr[n];
  indptr = S.pat_ptr.data();   // the originals below index the analyzed CSR
  indices = S.pat_idx.data();
  lap("graph");
  Shared sh(g, leaf_size);
  Builder B(sh);
  // connected components of the whole graph -> roots; the dissection trees
  // are concatenated in postorder and positions assigned in that order
  std::vector<std::vector<int64_t>> piv;
  std::vector<std::vector<int32_t>> kids;
  {
    int32_t s = ++sh.stamp;
    std::vector<int64_t> all(n);
    std::iota(all.begin(), all.end(), 0);
    for (int64_t v : all) B.mark(v, s);
    B.queue.resize(n);
    auto comps = B.components(all, s);
    for (auto& c : comps) {
      Sub sb = B.nd(std::move(c), 0);
      const int32_t off = (int32_t)piv.size();
      for (auto& kk : sb.kids)
        for (auto& x : kk) x += off;
      for (auto& pv : sb.piv) piv.push_back(std::move(pv));
      for (auto& kk : sb.kids) kids.push_back(std::move(kk));
    }
  }
  if (timing) for (int d = 0; d < 8; ++d) std::fprintf(stderr, "  sep depth %d: %.2f ms (sum over subproblems)\n", d, g_sep_ns[d].exchange(0) * 1e-6);
  lap("dissection");
  const int32_t nf = (int32_t)piv.size();
  S.iperm.assign(n, -1);
  {
    int64_t pos = 0;
    for (auto& pv : piv)
      for (int64_t v : pv) S.iperm[v] = pos++;
  }
  S.perm.assign(n, -1);
  for (int64_t v = 0; v < n; ++v) S.perm[S.iperm[v]] = v;

  S.fronts.resize(nf);
  S.child_ptr.assign(nf + 1, 0);
  for (int32_t f = 0; f < nf; ++f) S.child_ptr[f + 1] = S.child_ptr[f] + (int32_t)kids[f].size();
  S.child_list.resize(S.child_ptr[nf]);
  for (int32_t f = 0; f < nf; ++f) {
    std::copy(kids[f].begin(), kids[f].end(), S.child_list.begin() + S.child_ptr[f]);
    Front& F = S.fronts[f];
    F.p = (int32_t)piv[f].size();
    F.first = F.p ? S.iperm[piv[f][0]] : 0;
    F.parent = -1;
  }
  for (int32_t f = 0; f < nf; ++f)
    for (int32_t k = S.child_ptr[f]; k < S.child_ptr[f + 1]; ++k) S.fronts[S.child_list[k]].parent = f;

  // depth (parents have larger index than children)
  for (int32_t f = nf - 1; f >= 0; --f) {
    Front& F = S.fronts[f];
    F.depth = F.parent < 0 ? 0 : S.fronts[F.parent].depth + 1;
    S.max_depth = std::max(S.max_depth, F.depth);
  }
  S.levels.assign(S.max_depth + 1, {});
  for (int32_t f = 0; f < nf; ++f) S.levels[S.fronts[f].depth].push_back(f);

  // update-row structure, bottom-up level by level: the fronts of a level
  // only read their children's rows, so a level's fronts are split over a
  // few threads (each with its own marker array); results do not depend on
  // the split
  const int nth = (int)std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  std::vector<std::vector<int32_t>> marks(nth);
  std::vector<std::vector<int64_t>> U(nf);
  auto upd_rows = [&](const std::vector<int32_t>& lev, size_t i0, size_t i1, std::vector<int32_t>& mark) {
    if (mark.empty()) mark.assign(n, -1);
    for (size_t i = i0; i < i1; ++i) {
      const int32_t f = lev[i];
      Front& F = S.fronts[f];
      const int64_t last = F.first + F.p - 1;
      std::vector<int64_t>& u = U[f];
      for (int64_t v : piv[f])
        for (int64_t e = g.xadj[v]; e < g.xadj[v + 1]; ++e) {
          int64_t r = S.iperm[g.adj[e]];
          if (r > last && mark[r] != f) { mark[r] = f; u.push_back(r); }
        }
      for (int32_t k = S.child_ptr[f]; k < S.child_ptr[f + 1]; ++k)
        for (int64_t r : U[S.child_list[k]])
          if (r > last && mark[r] != f) { mark[r] = f; u.push_back(r); }
      std::sort(u.begin(), u.end());
      F.q = (int32_t)u.size();
    }
  };
  for (int32_t d = S.max_depth; d >= 0; --d) {
    const std::vector<int32_t>& lev = S.levels[d];
    if (lev.size() < 64 || nth == 1) {
      upd_rows(lev, 0, lev.size(), marks[0]);
      continue;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nth; ++t)
      th.emplace_back(upd_rows, std::cref(lev), lev.size() * t / nth, lev.size() * (t + 1) / nth,
                      std::ref(marks[t]));
    for (auto& x : th) x.join();
  }
  lap("updrows");

  // rows, relind, storage offsets, stats
  int64_t rows_total = 0;
  for (int32_t f = 0; f < nf; ++f) rows_total += S.fronts[f].q;
  S.urows.resize(rows_total);
  S.relind.resize(rows_total);
  int64_t ro = 0, panel = 0;
  for (int32_t f = 0; f < nf; ++f) {
    Front& F = S.fronts[f];
    F.rows_begin = ro;
    F.relind_begin = ro;
    std::copy(U[f].begin(), U[f].end(), S.urows.begin() + ro);
    ro += F.q;
    F.panel_off = panel;
    panel += (int64_t)F.m() * F.p;
    S.max_front = std::max(S.max_front, F.m());
    S.factor_nnz += (int64_t)F.p * (F.p + 1) / 2 + (int64_t)F.q * F.p;
    for (int64_t k = 0; k < F.p; ++k) {
      double r = (double)(F.m() - k - 1);
      S.flops += 8.0 * r * (r + 1.0) / 2.0 + 8.0 * r;
    }
  }
  S.panel_total = panel;
  {
    // relind: fronts are independent (contiguous front ranges per thread);
    // both row lists are sorted, so a merge walk finds each row in the parent
    std::vector<std::string> rerr(nth);
    auto rel = [&](int t) {
      const int32_t f0 = (int32_t)((int64_t)nf * t / nth), f1 = (int32_t)((int64_t)nf * (t + 1) / nth);
      for (int32_t f = f0; f < f1; ++f) {
        const Front& F = S.fronts[f];
        if (F.parent < 0) continue;
        const Front& P = S.fronts[F.parent];
        const int64_t plast = P.first + P.p - 1;
        const int64_t* prow = S.urows.data() + P.rows_begin;
        int32_t j = 0;
        for (int32_t a = 0; a < F.q; ++a) {
          int64_t r = S.urows[F.rows_begin + a];
          int32_t loc;
          if (r <= plast) {
            if (r < P.first) { rerr[t] = "internal: update row below parent pivots"; return; }
            loc = (int32_t)(r - P.first);
          } else {
            while (j < P.q && prow[j] < r) ++j;
            if (j == P.q || prow[j] != r) { rerr[t] = "internal: update row missing in parent"; return; }
            loc = P.p + j;
          }
          S.relind[F.relind_begin + a] = loc;
        }
      }
    };
    if (nf < 256) {
      for (int t = 0; t < nth; ++t) rel(t);
    } else {
      std::vector<std::thread> th;
      for (int t = 1; t < nth; ++t) th.emplace_back(rel, t);
      rel(0);
      for (auto& x : th) x.join();
    }
    for (auto& e : rerr)
      if (!e.empty()) return e;
  }
  lap("relind");
  // pull maps: for child c of P, cmap[c][r] = a with relind_c[a] = r (r < m_P), else -1
  {
    int64_t tot = 0;
    for (int32_t f = 0; f < nf; ++f) {
      Front& F = S.fronts[f];
      F.cmap_begin = tot;
      if (F.parent >= 0) tot += S.fronts[F.parent].m();
    }
    S.cmap.assign(tot, -1);
    for (int32_t f = 0; f < nf; ++f) {
      const Front& F = S.fronts[f];
      if (F.parent < 0) continue;
      for (int32_t a = 0; a < F.q; ++a) S.cmap[F.cmap_begin + S.relind[F.relind_begin + a]] = a;
    }
  }
  for (int32_t d = 0; d <= S.max_depth; ++d) {
    int64_t uo = 0, ru = 0;
    for (int32_t f : S.levels[d]) {
      Front& F = S.fronts[f];
      F.upd_off = uo;
      F.rupd_off = ru;
      uo += (int64_t)F.q * (F.q + 1) / 2;  // packed lower (kh_upk)
      ru += F.q;
    }
    S.upd_size[d & 1] = std::max(S.upd_size[d & 1], uo);
    S.rupd_size[d & 1] = std::max(S.rupd_size[d & 1], ru);
  }

  lap("cmap");
  // original entries: CSR entry (r, c) with iperm[r] >= iperm[c] lands in the
  // front owning pivot iperm[c] at local (row(iperm[r]), iperm[c]-first)
  std::vector<int32_t> front_of(n, -1);
  for (int32_t f = 0; f < nf; ++f)
    for (int64_t k = 0; k < S.fronts[f].p; ++k) front_of[S.fronts[f].first + k] = f;
  // two passes over row ranges, one range per thread: count per (thread,
  // front), then fill at offsets that put thread t's entries of a front
  // after those of threads < t -- the same order as one serial pass
  std::vector<int64_t> cnt(nf + 1, 0);
  std::vector<std::vector<int64_t>> tcnt(nth, std::vector<int64_t>(nf, 0));
  auto row_lo = [&](int t) { return (int64_t)n * t / nth; };
  {
    auto count = [&](int t) {
      std::vector<int64_t>& c = tcnt[t];
      for (int64_t r = row_lo(t); r < row_lo(t + 1); ++r)
        for (int64_t e = indptr[r]; e < indptr[r + 1]; ++e) {
          int64_t i = S.iperm[r], j = S.iperm[indices[e]];
          if (i >= j) ++c[front_of[j]];
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nth; ++t) th.emplace_back(count, t);
    count(0);
    for (auto& x : th) x.join();
  }
  for (int32_t f = 0; f < nf; ++f) {
    int64_t tot = 0;
    for (int t = 0; t < nth; ++t) tot += tcnt[t][f];
    cnt[f + 1] = cnt[f] + tot;
  }
  S.orig_src.resize(cnt[nf]);
  S.orig_dst.resize(cnt[nf]);
  std::vector<std::string> errs(nth);
  {
    auto fill = [&](int t) {
      std::vector<int64_t> pos(nf);
      for (int32_t f = 0; f < nf; ++f) {
        int64_t o = cnt[f];
        for (int u = 0; u < t; ++u) o += tcnt[u][f];
        pos[f] = o;
      }
      for (int64_t r = row_lo(t); r < row_lo(t + 1); ++r)
        for (int64_t e = indptr[r]; e < indptr[r + 1]; ++e) {
          int64_t i = S.iperm[r], j = S.iperm[indices[e]];
          if (i < j) continue;
          int32_t f = front_of[j];
          const Front& F = S.fronts[f];
          int32_t ri;
          if (i < F.first + F.p) {
            ri = (int32_t)(i - F.first);
          } else {
            const int64_t* prow = S.urows.data() + F.rows_begin;
            const int64_t* it = std::lower_bound(prow, prow + F.q, i);
            if (it == prow + F.q || *it != i) { errs[t] = "internal: entry outside front rows"; return; }
            ri = F.p + (int32_t)(it - prow);
          }
          int64_t dst = (int64_t)ri + (j - F.first) * (int64_t)F.m();
          if (dst > INT32_MAX) { errs[t] = "front too large for 32-bit local offsets"; return; }
          S.orig_src[pos[f]] = e;
          S.orig_dst[pos[f]] = (int32_t)dst;
          ++pos[f];
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nth; ++t) th.emplace_back(fill, t);
    fill(0);
    for (auto& x : th) x.join();
  }
  for (auto& e : errs)
    if (!e.empty()) return e;
  // deterministic, write-coalescing order inside each front (fronts are
  // independent: sorted by a few threads over contiguous front ranges)
  auto sort_fronts = [&](int32_t f0, int32_t f1) {
    std::vector<std::pair<int32_t, int64_t>> tmp;
    for (int32_t f = f0; f < f1; ++f) {
      S.fronts[f].orig_begin = cnt[f];
      S.fronts[f].orig_end = cnt[f + 1];
      tmp.clear();
      for (int64_t k = cnt[f]; k < cnt[f + 1]; ++k) tmp.emplace_back(S.orig_dst[k], S.orig_src[k]);
      std::sort(tmp.begin(), tmp.end());
      for (int64_t k = cnt[f]; k < cnt[f + 1]; ++k) {
        S.orig_dst[k] = tmp[k - cnt[f]].first;
        S.orig_src[k] = tmp[k - cnt[f]].second;
      }
    }
  };
  {
    if (nf < 256 || nth == 1) {
      sort_fronts(0, nf);
    } else {
      std::vector<std::thread> th;
      for (int t = 0; t < nth; ++t) {
        const int32_t f0 = (int32_t)((int64_t)nf * t / nth), f1 = (int32_t)((int64_t)nf * (t + 1) / nth);
        th.emplace_back(sort_fronts, f0, f1);
      }
      for (auto& x : th) x.join();
    }
  }
  lap("originals");
  return "";
}

}  // namespace kh
