// Supernodal symbolic analysis, relaxed amalgamation and multifrontal numeric
// Cholesky producing the block-inverse factor consumed by the device DAG
// kernel (dag_solve.cu).
//
// Replaces linalg.Factorization (linalg.py:37-72): the reference uses LAPACK
// cho_factor for n <= 512 and SuperLU LU with MMD(A^T+A) above.  Here every
// SPD block is factorized as L L^T (A_i is SPD: linalg.py:62-63 rejects
// non-positive pivots the same way, raised as FactorizationError), and each
// supernode stores M = [L_JJ^{-1}; L_BJ L_JJ^{-1}] so that both triangular
// sweeps become dependency-free GEMVs per supernode.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>

#include "common.h"
#include "host.h"

namespace sfcdd {

FactorOptions::FactorOptions() {
  if (const char* v = std::getenv("SFCDD_RELAX_SMALL")) relax_small = std::atoi(v);
  if (const char* v = std::getenv("SFCDD_RELAX_SMALL_FRAC")) relax_small_frac = std::atof(v);
  if (const char* v = std::getenv("SFCDD_RELAX_FRAC")) relax_frac = std::atof(v);
  if (const char* v = std::getenv("SFCDD_ORDER")) ordering = std::string(v) == "amd" ? 0 : 1;
  if (const char* v = std::getenv("SFCDD_ND_LEAF")) nd_leaf = std::atoi(v);
}

int hardware_threads() {
  unsigned h = std::thread::hardware_concurrency();
  return h == 0 ? 4 : (int)h;
}

namespace {

// ---- elimination tree (Liu) on the permuted pattern -----------------------
void etree(const CsrMatrix& A, const std::vector<int32_t>& order, const std::vector<int32_t>& iperm,
           std::vector<int32_t>& parent) {
  const int64_t n = A.n;
  parent.assign(n, -1);
  std::vector<int32_t> anc(n, -1);
  for (int64_t i = 0; i < n; ++i) {
    const int32_t o = order[i];
    for (int64_t p = A.indptr[o]; p < A.indptr[o + 1]; ++p) {
      int32_t k = iperm[A.indices[p]];
      while (k != -1 && k < i) {
        int32_t kn = anc[k];
        anc[k] = (int32_t)i;
        if (kn == -1) parent[k] = (int32_t)i;
        k = kn;
      }
    }
  }
}

// children lists in ascending order, then iterative DFS postorder
std::vector<int32_t> postorder(const std::vector<int32_t>& parent) {
  const int64_t n = parent.size();
  std::vector<int32_t> head(n, -1), next(n, -1), post;
  post.reserve(n);
  for (int64_t j = n - 1; j >= 0; --j) {
    if (parent[j] < 0) continue;
    next[j] = head[parent[j]];
    head[parent[j]] = (int32_t)j;
  }
  std::vector<int32_t> stack;
  for (int64_t r = 0; r < n; ++r) {
    if (parent[r] != -1) continue;
    stack.push_back((int32_t)r);
    while (!stack.empty()) {
      int32_t v = stack.back();
      int32_t c = head[v];
      if (c == -1) {
        stack.pop_back();
        post.push_back(v);
      } else {
        head[v] = next[c];
        stack.push_back(c);
      }
    }
  }
  return post;
}

struct Node {
  std::vector<int32_t> cols;  // columns in the (post)ordering before renumbering
  int64_t first_col = 0;      // the representative top fundamental supernode's first col
  int32_t s = 0, m = 0;
  int64_t real = 0;
  int32_t parent = -1;
  bool alive = true;
};

}  // namespace

HostFactor analyze_host(const CsrMatrix& A, const FactorOptions& opt) {
  const int64_t n = A.n;
  HostFactor F;
  F.n = n;
  if (n == 0) return F;
  SymPattern P;
  P.n = n;
  P.indptr = A.indptr;
  P.indices = A.indices;
  std::vector<int32_t> order = opt.ordering == 1 ? nd_order(P, opt.nd_leaf) : amd_order(P);
  std::vector<int32_t> iperm(n);
  for (int64_t k = 0; k < n; ++k) iperm[order[k]] = (int32_t)k;
  std::vector<int32_t> parent;
  etree(A, order, iperm, parent);
  // postorder relabel
  std::vector<int32_t> post = postorder(parent);
  std::vector<int32_t> ipost(n);
  for (int64_t k = 0; k < n; ++k) ipost[post[k]] = (int32_t)k;
  std::vector<int32_t> order2(n), iperm2(n), parent2(n);
  for (int64_t k = 0; k < n; ++k) {
    order2[k] = order[post[k]];
    iperm2[order2[k]] = (int32_t)k;
    int32_t pk = parent[post[k]];
    parent2[k] = pk < 0 ? -1 : ipost[pk];
  }
  // column structures (strictly below the diagonal), children before parents
  std::vector<int32_t> chead(n, -1), cnext(n, -1), nchild(n, 0);
  for (int64_t j = n - 1; j >= 0; --j) {
    int32_t p = parent2[j];
    if (p < 0) continue;
    cnext[j] = chead[p];
    chead[p] = (int32_t)j;
    nchild[p]++;
  }
  std::vector<int64_t> sptr(n + 1, 0);
  std::vector<int32_t> sidx;
  sidx.reserve(8 * n);
  std::vector<int32_t> mark(n, -1);
  std::vector<int64_t> cc(n);
  for (int64_t j = 0; j < n; ++j) {
    sptr[j] = sidx.size();
    const int32_t o = order2[j];
    for (int64_t p = A.indptr[o]; p < A.indptr[o + 1]; ++p) {
      int32_t i = iperm2[A.indices[p]];
      if (i > j && mark[i] != j) {
        mark[i] = (int32_t)j;
        sidx.push_back(i);
      }
    }
    for (int32_t c = chead[j]; c != -1; c = cnext[c]) {
      for (int64_t p = sptr[c]; p < sptr[c + 1]; ++p) {
        int32_t i = sidx[p];
        if (i > j && mark[i] != j) {
          mark[i] = (int32_t)j;
          sidx.push_back(i);
        }
      }
    }
    sptr[j + 1] = sidx.size();
    cc[j] = 1 + (sptr[j + 1] - sptr[j]);
  }
  F.nnz_l = 0;
  for (int64_t j = 0; j < n; ++j) F.nnz_l += cc[j];
  // fundamental supernodes
  std::vector<Node> nodes;
  std::vector<int32_t> col2node(n);
  for (int64_t j = 0; j < n; ++j) {
    bool join = j > 0 && parent2[j - 1] == j && nchild[j] == 1 && cc[j - 1] == cc[j] + 1;
    if (!join) {
      Node nd;
      nd.first_col = j;
      nodes.push_back(nd);
    }
    Node& nd = nodes.back();
    nd.cols.push_back((int32_t)j);
    col2node[j] = (int32_t)nodes.size() - 1;
  }
  for (auto& nd : nodes) {
    nd.s = (int32_t)nd.cols.size();
    nd.m = (int32_t)(cc[nd.first_col] - nd.s);
    nd.real = packed_size(nd.s, nd.m);
    int32_t last = nd.cols.back();
    nd.parent = parent2[last] < 0 ? -1 : col2node[parent2[last]];
  }
  // relaxed amalgamation (children before parents in node order)
  const int64_t nn = nodes.size();
  std::vector<std::vector<int32_t>> kids(nn);
  for (int64_t c = 0; c < nn; ++c)
    if (nodes[c].parent >= 0) kids[nodes[c].parent].push_back((int32_t)c);
  for (int64_t c = 0; c < nn; ++c) {
    Node& ch = nodes[c];
    if (!ch.alive || ch.parent < 0) continue;
    Node& pa = nodes[ch.parent];
    int64_t S = (int64_t)ch.s + pa.s;
    int64_t merged = packed_size(S, pa.m);
    int64_t real = ch.real + pa.real;
    int64_t zeros = merged - real;
    bool ok = (S <= opt.relax_small && zeros <= opt.relax_small_frac * merged) ||
              zeros <= opt.relax_frac * merged;
    if (!ok) continue;
    std::vector<int32_t> cols = ch.cols;
    cols.insert(cols.end(), pa.cols.begin(), pa.cols.end());
    pa.cols.swap(cols);
    pa.s = (int32_t)S;
    pa.real = real;
    ch.alive = false;
    ch.cols.clear();
    ch.cols.shrink_to_fit();
    for (int32_t d : kids[c]) {
      if (!nodes[d].alive) continue;
      nodes[d].parent = ch.parent;
      kids[ch.parent].push_back(d);
    }
    kids[c].clear();
  }
  // postorder of the alive supernode tree; children kept in node order
  std::vector<int32_t> alive_ids;
  for (int64_t k = 0; k < nn; ++k)
    if (nodes[k].alive) alive_ids.push_back((int32_t)k);
  std::vector<int32_t> sparent(nn, -1);
  for (int32_t k : alive_ids) sparent[k] = nodes[k].parent;
  std::vector<int32_t> shead(nn, -1), snext(nn, -1);
  for (int64_t t = (int64_t)alive_ids.size() - 1; t >= 0; --t) {
    int32_t k = alive_ids[t];
    int32_t p = sparent[k];
    if (p < 0) continue;
    snext[k] = shead[p];
    shead[p] = k;
  }
  std::vector<int32_t> spost;
  spost.reserve(alive_ids.size());
  {
    std::vector<int32_t> stack;
    for (int32_t r : alive_ids) {
      if (sparent[r] != -1) continue;
      stack.push_back(r);
      while (!stack.empty()) {
        int32_t v = stack.back();
        int32_t c = shead[v];
        if (c == -1) {
          stack.pop_back();
          spost.push_back(v);
        } else {
          shead[v] = snext[c];
          stack.push_back(c);
        }
      }
    }
  }
  // renumber columns
  std::vector<int32_t> newcol(n, -1);
  int32_t next = 0;
  for (int32_t k : spost)
    for (int32_t c : nodes[k].cols) newcol[c] = next++;
  SFCDD_REQUIRE(next == n, SFCDD_EINTERNAL, "amalgamation lost columns");
  F.perm.resize(n);
  for (int64_t c = 0; c < n; ++c) F.perm[newcol[c]] = order2[c];
  std::vector<int32_t> node2sn(nn, -1);
  for (size_t t = 0; t < spost.size(); ++t) node2sn[spost[t]] = (int32_t)t;
  F.sn.resize(spost.size());
  F.rows.clear();
  int64_t val_off = 0;
  for (size_t t = 0; t < spost.size(); ++t) {
    const Node& nd = nodes[spost[t]];
    Supernode& S = F.sn[t];
    S.s = nd.s;
    S.m = nd.m;
    S.col0 = newcol[nd.cols.front()];
    S.parent = nd.parent < 0 ? -1 : node2sn[nd.parent];
    S.rows_off = F.rows.size();
    // below rows = structure of the top fundamental supernode's first col,
    // minus the (original) columns of that fundamental supernode
    int64_t fc = nd.first_col;
    int32_t top_s = 0;
    for (int64_t c = fc; c < n && col2node[c] == col2node[fc]; ++c) ++top_s;
    for (int64_t p = sptr[fc]; p < sptr[fc + 1]; ++p) {
      int32_t i = sidx[p];
      if (i >= fc + top_s) F.rows.push_back(newcol[i]);
    }
    SFCDD_REQUIRE((int64_t)F.rows.size() - S.rows_off == S.m, SFCDD_EINTERNAL, "row count mismatch");
    std::sort(F.rows.begin() + S.rows_off, F.rows.end());
    S.val_off = val_off;
    val_off += packed_size(S.s, S.m);
    F.max_front = std::max<int32_t>(F.max_front, S.s + S.m);
  }
  F.stored = val_off;
  // children lists, levels, relative maps
  const int64_t ns = F.sn.size();
  F.child_ptr.assign(ns + 1, 0);
  for (int64_t k = 0; k < ns; ++k)
    if (F.sn[k].parent >= 0) F.child_ptr[F.sn[k].parent + 1]++;
  for (int64_t k = 0; k < ns; ++k) F.child_ptr[k + 1] += F.child_ptr[k];
  F.child_list.assign(F.child_ptr[ns], 0);
  {
    std::vector<int32_t> fill(F.child_ptr.begin(), F.child_ptr.end() - 1);
    for (int64_t k = 0; k < ns; ++k)
      if (F.sn[k].parent >= 0) F.child_list[fill[F.sn[k].parent]++] = (int32_t)k;
  }
  for (int64_t k = 0; k < ns; ++k) {
    int32_t lv = 0;
    for (int32_t p = F.child_ptr[k]; p < F.child_ptr[k + 1]; ++p)
      lv = std::max(lv, F.sn[F.child_list[p]].level + 1);
    F.sn[k].level = lv;
  }
  std::vector<int32_t> pos(n, -1);
  F.rel.clear();
  for (int64_t k = 0; k < ns; ++k) F.sn[k].rel_off = 0;
  // positions are relative to the parent's frontal [cols ; rows]
  for (int64_t p = 0; p < ns; ++p) {
    const Supernode& P = F.sn[p];
    for (int32_t t = 0; t < P.s; ++t) pos[P.col0 + t] = t;
    for (int32_t a = 0; a < P.m; ++a) pos[F.rows[P.rows_off + a]] = P.s + a;
    for (int32_t q = F.child_ptr[p]; q < F.child_ptr[p + 1]; ++q) {
      Supernode& K = F.sn[F.child_list[q]];
      K.rel_off = F.rel.size();
      for (int32_t a = 0; a < K.m; ++a) {
        int32_t r = F.rows[K.rows_off + a];
        SFCDD_REQUIRE(pos[r] >= 0, SFCDD_EINTERNAL, "child row outside parent front");
        F.rel.push_back(pos[r]);
      }
    }
    for (int32_t t = 0; t < P.s; ++t) pos[P.col0 + t] = -1;
    for (int32_t a = 0; a < P.m; ++a) pos[F.rows[P.rows_off + a]] = -1;
  }
  if (std::getenv("SFCDD_FACTOR_DEBUG")) {
    // critical path of the supernodal tree (supernodes and stored entries)
    std::vector<int64_t> cp_n(ns, 0), cp_b(ns, 0);
    int64_t hmax = 0, bmax = 0;
    for (int64_t k = 0; k < ns; ++k) {
      cp_n[k] += 1;
      cp_b[k] += packed_size(F.sn[k].s, F.sn[k].m);
      hmax = std::max(hmax, cp_n[k]);
      bmax = std::max(bmax, cp_b[k]);
      const int32_t p = F.sn[k].parent;
      if (p >= 0) {
        cp_n[p] = std::max(cp_n[p], cp_n[k]);
        cp_b[p] = std::max(cp_b[p], cp_b[k]);
      }
    }
    std::fprintf(stderr, "[factor] n=%lld supernodes=%lld nnzL=%lld stored=%lld (%.3f) height=%lld critpath=%.1f%%\n",
                 (long long)n, (long long)ns, (long long)F.nnz_l, (long long)F.stored,
                 (double)F.stored / F.nnz_l, (long long)hmax, 100.0 * bmax / F.stored);
    const int edges[] = {1, 2, 4, 8, 16, 32, 64, 128, 1 << 30};
    int64_t cnt[9] = {0}, byt[9] = {0};
    for (int64_t k = 0; k < ns; ++k) {
      int b = 0;
      while (F.sn[k].s > edges[b]) ++b;
      cnt[b]++;
      byt[b] += packed_size(F.sn[k].s, F.sn[k].m);
    }
    for (int b = 0; b < 9; ++b)
      std::fprintf(stderr, "  s<=%d: %lld supernodes, %.1f%% of stored\n", edges[b], (long long)cnt[b],
                   100.0 * byt[b] / F.stored);
  }
  return F;
}

namespace {

// In-place partial Cholesky of the leading s columns of a symmetric front
// (lower, column-major, ld = nf): on exit F11 = L11, F21 = L21 and
// F22 = F22 - L21 L21^T.  Blocked right-looking with 32-column panels.
void partial_cholesky(double* Fm, int64_t nf, int64_t s) {
  const int64_t ld = nf;
  constexpr int64_t NB = 32;
  for (int64_t kb = 0; kb < s; kb += NB) {
    const int64_t ke = std::min(s, kb + NB);
    // panel factorization (columns kb..ke-1, all rows)
    for (int64_t k = kb; k < ke; ++k) {
      double* ck = Fm + k * ld;
      double d = ck[k];
      if (!(d > 0.0))
        throw Error(SFCDD_EFACTOR, "nonpositive pivot, matrix is not SPD");
      d = std::sqrt(d);
      ck[k] = d;
      const double inv = 1.0 / d;
      for (int64_t i = k + 1; i < nf; ++i) ck[i] *= inv;
      for (int64_t j = k + 1; j < ke; ++j) {
        const double c = ck[j];
        double* cj = Fm + j * ld;
        for (int64_t i = j; i < nf; ++i) cj[i] -= ck[i] * c;
      }
    }
    // trailing update with the panel: F[j.., j] -= sum_k F[.., k] F[j, k]
    for (int64_t j = ke; j < nf; ++j) {
      double* cj = Fm + j * ld;
      for (int64_t k = kb; k < ke; ++k) {
        const double* ck = Fm + k * ld;
        const double c = ck[j];
        if (c == 0.0) continue;
        for (int64_t i = j; i < nf; ++i) cj[i] -= ck[i] * c;
      }
    }
  }
}

}  // namespace

void numeric_host(const CsrMatrix& A, HostFactor& F) {
  const int64_t n = F.n;
  F.val.assign(F.stored, 0.0);
  if (n == 0) return;
  std::vector<int32_t> iperm(n);
  for (int64_t k = 0; k < n; ++k) iperm[F.perm[k]] = (int32_t)k;
  std::vector<int32_t> pos(n, -1);
  struct Upd {
    int32_t m;
    std::vector<double> u;
  };
  std::vector<Upd> stack;
  std::vector<double> front, linv;
  const int64_t ns = F.sn.size();
  for (int64_t k = 0; k < ns; ++k) {
    const Supernode& S = F.sn[k];
    const int64_t s = S.s, m = S.m, nf = s + m;
    front.assign(nf * nf, 0.0);
    for (int64_t t = 0; t < s; ++t) pos[S.col0 + t] = (int32_t)t;
    for (int64_t a = 0; a < m; ++a) pos[F.rows[S.rows_off + a]] = (int32_t)(s + a);
    // assemble original entries (lower part)
    for (int64_t t = 0; t < s; ++t) {
      const int64_t c = S.col0 + t;
      const int32_t o = F.perm[c];
      for (int64_t p = A.indptr[o]; p < A.indptr[o + 1]; ++p) {
        int32_t r = iperm[A.indices[p]];
        if (r < c) continue;
        int32_t ps = pos[r];
        SFCDD_REQUIRE(ps >= 0, SFCDD_EINTERNAL, "matrix entry outside front");
        front[t * nf + ps] += A.data[p];
      }
    }
    // extend-add children's update matrices (stack top, in child order)
    const int32_t nch = F.child_ptr[k + 1] - F.child_ptr[k];
    SFCDD_REQUIRE((int64_t)stack.size() >= nch, SFCDD_EINTERNAL, "update stack underflow");
    for (int32_t q = 0; q < nch; ++q) {
      const Supernode& K = F.sn[F.child_list[F.child_ptr[k] + q]];
      const Upd& U = stack[stack.size() - nch + q];
      const int32_t* rel = F.rel.data() + K.rel_off;
      for (int32_t b = 0; b < U.m; ++b) {
        double* col = front.data() + (int64_t)rel[b] * nf;
        const double* ub = U.u.data() + (int64_t)b * U.m;
        for (int32_t a = b; a < U.m; ++a) col[rel[a]] += ub[a];
      }
    }
    stack.resize(stack.size() - nch);
    partial_cholesky(front.data(), nf, s);
    // L11^{-1} (lower) by forward substitution, column by column
    linv.assign(s * s, 0.0);
    for (int64_t j = 0; j < s; ++j) {
      double* xj = linv.data() + j * s;
      xj[j] = 1.0 / front[j * nf + j];
      for (int64_t i = j + 1; i < s; ++i) {
        double acc = 0.0;
        for (int64_t t = j; t < i; ++t) acc += front[t * nf + i] * xj[t];
        xj[i] = -acc / front[i * nf + i];
      }
    }
    // pack M = [Linv ; L21 Linv]
    double* Mv = F.val.data() + S.val_off;
    std::vector<double> wcol(m);
    for (int64_t kc = 0; kc < s; ++kc) {
      double* col = Mv + packed_col_off(s, m, kc);
      for (int64_t i = kc; i < s; ++i) col[i - kc] = linv[kc * s + i];
      std::fill(wcol.begin(), wcol.end(), 0.0);
      for (int64_t t = kc; t < s; ++t) {
        const double c = linv[kc * s + t];
        const double* l21 = front.data() + t * nf + s;
        for (int64_t a = 0; a < m; ++a) wcol[a] += l21[a] * c;
      }
      for (int64_t a = 0; a < m; ++a) col[s - kc + a] = wcol[a];
    }
    // push the Schur complement
    if (S.parent >= 0) {
      Upd U;
      U.m = (int32_t)m;
      U.u.assign(m * m, 0.0);
      for (int64_t b = 0; b < m; ++b)
        for (int64_t a = b; a < m; ++a) U.u[b * m + a] = front[(s + b) * nf + (s + a)];
      stack.push_back(std::move(U));
    }
    for (int64_t t = 0; t < s; ++t) pos[S.col0 + t] = -1;
    for (int64_t a = 0; a < m; ++a) pos[F.rows[S.rows_off + a]] = -1;
  }
}

HostFactor factorize_host(const CsrMatrix& A, const FactorOptions& opt) {
  HostFactor F = analyze_host(A, opt);
  numeric_host(A, F);
  return F;
}

void host_block_solve(const HostFactor& F, const double* b, double* x) {
  const int64_t n = F.n;
  std::vector<double> y(n), xp(n), f, out;
  std::vector<std::vector<double>> upd(F.sn.size());
  for (size_t k = 0; k < F.sn.size(); ++k) {
    const Supernode& S = F.sn[k];
    const int64_t s = S.s, m = S.m;
    f.assign(s + m, 0.0);
    for (int64_t t = 0; t < s; ++t) f[t] = b[F.perm[S.col0 + t]];
    for (int32_t q = F.child_ptr[k]; q < F.child_ptr[k + 1]; ++q) {
      const int32_t c = F.child_list[q];
      const Supernode& K = F.sn[c];
      for (int32_t a = 0; a < K.m; ++a) f[F.rel[K.rel_off + a]] += upd[c][a];
      upd[c].clear();
      upd[c].shrink_to_fit();
    }
    out.assign(s + m, 0.0);
    const double* Mv = F.val.data() + S.val_off;
    for (int64_t kc = 0; kc < s; ++kc) {
      const double* col = Mv + packed_col_off(s, m, kc);
      for (int64_t i = kc; i < s + m; ++i) out[i] += col[i - kc] * f[kc];
    }
    for (int64_t t = 0; t < s; ++t) y[S.col0 + t] = out[t];
    upd[k].resize(m);
    for (int64_t a = 0; a < m; ++a) upd[k][a] = f[s + a] - out[s + a];
  }
  std::vector<double> v;
  for (int64_t k = (int64_t)F.sn.size() - 1; k >= 0; --k) {
    const Supernode& S = F.sn[k];
    const int64_t s = S.s, m = S.m;
    v.resize(s + m);
    for (int64_t t = 0; t < s; ++t) v[t] = y[S.col0 + t];
    for (int64_t a = 0; a < m; ++a) v[s + a] = -xp[F.rows[S.rows_off + a]];
    const double* Mv = F.val.data() + S.val_off;
    for (int64_t kc = 0; kc < s; ++kc) {
      const double* col = Mv + packed_col_off(s, m, kc);
      double acc = 0.0;
      for (int64_t i = kc; i < s + m; ++i) acc += col[i - kc] * v[i];
      xp[S.col0 + kc] = acc;
    }
  }
  for (int64_t j = 0; j < n; ++j) x[F.perm[j]] = xp[j];
}

}  // namespace sfcdd
