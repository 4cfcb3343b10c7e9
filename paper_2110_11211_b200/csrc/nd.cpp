// Hybrid nested-dissection ordering: recursive BFS level-set vertex
// separators (George's automatic nested dissection on the graph, no
// coordinates needed) down to small parts, AMD on the parts.
//
// Why: the parallel triangular solves of the local factors are bounded by
// the height of the supernodal elimination tree.  AMD leaves
// a long chain of separator supernodes at the top of every subdomain tree;
// nested dissection makes the top a balanced binary tree of separators
// (height ~ log2 n) for a small change in fill.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "common.h"
#include "host.h"

namespace sfcdd {

namespace {

struct Nd {
  const SymPattern& A;
  int32_t leaf;
  std::vector<int32_t> order;      // output, elimination order
  std::vector<int32_t> part;       // current part id per vertex (-1 = ordered)
  std::vector<int32_t> level;      // BFS scratch
  std::vector<int32_t> local;      // global -> local index scratch
  int32_t next_id = 1;

  Nd(const SymPattern& a, int32_t lf) : A(a), leaf(lf), part(a.n, 0), level(a.n, -1), local(a.n, -1) {}

  // BFS over vertices with part == id starting at root; returns levels in `lv`
  // (vertices per level, in BFS order) and the last vertex reached
  int32_t bfs(int32_t id, int32_t root, std::vector<std::vector<int32_t>>& lv) {
    lv.clear();
    std::vector<int32_t> cur{root}, nxt;
    level[root] = 0;
    int32_t last = root;
    while (!cur.empty()) {
      lv.push_back(cur);
      nxt.clear();
      for (int32_t v : cur) {
        last = v;
        for (int64_t p = A.indptr[v]; p < A.indptr[v + 1]; ++p) {
          const int32_t w = A.indices[p];
          if (w != v && part[w] == id && level[w] < 0) {
            level[w] = (int32_t)lv.size();
            nxt.push_back(w);
          }
        }
      }
      cur.swap(nxt);
    }
    for (const auto& l : lv)
      for (int32_t v : l) level[v] = -1;
    return last;
  }

  void amd_leaf(const std::vector<int32_t>& vs) {
    if (vs.size() <= 2) {
      order.insert(order.end(), vs.begin(), vs.end());
      return;
    }
    SymPattern S;
    S.n = (int64_t)vs.size();
    for (size_t i = 0; i < vs.size(); ++i) local[vs[i]] = (int32_t)i;
    S.indptr.assign(vs.size() + 1, 0);
    for (size_t i = 0; i < vs.size(); ++i) {
      const int32_t v = vs[i];
      for (int64_t p = A.indptr[v]; p < A.indptr[v + 1]; ++p) {
        const int32_t w = A.indices[p];
        if (local[w] >= 0 && part[w] == part[v]) S.indices.push_back(local[w]);
      }
      S.indptr[i + 1] = (int64_t)S.indices.size();
    }
    const std::vector<int32_t> o = amd_order(S);
    for (int32_t i : o) order.push_back(vs[i]);
    for (int32_t v : vs) local[v] = -1;
  }

  // order the vertices `vs` (all with part == id); they may be disconnected
  void dissect(std::vector<int32_t> vs, int32_t id) {
    if ((int32_t)vs.size() <= leaf) {
      amd_leaf(vs);
      for (int32_t v : vs) part[v] = -1;
      return;
    }
    // connected component of vs[0]
    std::vector<std::vector<int32_t>> lv;
    int32_t far = bfs(id, vs[0], lv);
    size_t comp = 0;
    for (const auto& l : lv) comp += l.size();
    if (comp < vs.size()) {  // split off the component, recurse on both
      std::vector<int32_t> a, b;
      const int32_t ida = next_id++, idb = next_id++;
      for (const auto& l : lv)
        for (int32_t v : l) {
          a.push_back(v);
          part[v] = ida;
        }
      for (int32_t v : vs)
        if (part[v] == id) {
          b.push_back(v);
          part[v] = idb;
        }
      dissect(std::move(a), ida);
      dissect(std::move(b), idb);
      return;
    }
    // pseudo-peripheral root: repeat BFS from the farthest vertex
    for (int it = 0; it < 2; ++it) {
      const size_t depth = lv.size();
      const int32_t f2 = bfs(id, far, lv);
      if (lv.size() <= depth) break;
      far = f2;
    }
    if (lv.size() < 3) {  // too shallow to split by levels
      amd_leaf(vs);
      for (int32_t v : vs) part[v] = -1;
      return;
    }
    // separator: the smallest level whose prefix holds 35..65% of the vertices
    const size_t n = vs.size();
    size_t best = 0, pre = 0, best_sz = n + 1;
    std::vector<size_t> prefix(lv.size());
    for (size_t l = 0; l < lv.size(); ++l) {
      prefix[l] = pre;
      pre += lv[l].size();
    }
    for (size_t l = 1; l + 1 < lv.size(); ++l) {
      const double f = (double)prefix[l] / (double)n;
      if (f < 0.35 || f > 0.65) continue;
      if (lv[l].size() < best_sz) {
        best_sz = lv[l].size();
        best = l;
      }
    }
    if (best == 0) {  // no level in the window: take the median level
      for (size_t l = 1; l + 1 < lv.size(); ++l)
        if (prefix[l + 1] * 2 >= n) {
          best = l;
          break;
        }
    }
    std::vector<int32_t> a, b, sep = lv[best];
    const int32_t ida = next_id++, idb = next_id++;
    for (size_t l = 0; l < lv.size(); ++l) {
      if (l == best) continue;
      for (int32_t v : lv[l]) {
        (l < best ? a : b).push_back(v);
        part[v] = l < best ? ida : idb;
      }
    }
    for (int32_t v : sep) part[v] = -2;  // excluded from both halves
    dissect(std::move(a), ida);
    dissect(std::move(b), idb);
    // separator last (its own AMD order keeps its internal fill low)
    for (int32_t v : sep) part[v] = id;
    amd_leaf(sep);
    for (int32_t v : sep) part[v] = -1;
  }
};

}  // namespace

std::vector<int32_t> nd_order(const SymPattern& A, int32_t leaf) {
  const int64_t n = A.n;
  Nd nd(A, std::max<int32_t>(leaf, 8));
  nd.order.reserve(n);
  std::vector<int32_t> all(n);
  for (int64_t i = 0; i < n; ++i) all[i] = (int32_t)i;
  nd.dissect(std::move(all), 0);
  SFCDD_REQUIRE((int64_t)nd.order.size() == n, SFCDD_EINTERNAL, "nested dissection lost vertices");
  return nd.order;
}

}  // namespace sfcdd
