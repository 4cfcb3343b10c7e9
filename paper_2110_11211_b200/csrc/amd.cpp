// Approximate minimum degree ordering (Amestoy, Davis & Duff 1996) on the
// quotient graph, written from the published algorithm.
//
// Role on the hot path: the reference factorizes every subdomain block with
// SuperLU using the MMD ordering of A^T + A (linalg.py:55-61).  The factor
// bytes streamed per PCG iteration are set by the fill of that ordering, so
// the builder needs a fill-reducing ordering of the same quality; geometric
// nested dissection on SFC-shaped subdomains measured 1.3-1.5x the MMD fill
// (DESIGN.md), AMD measures within a few percent of it.
//
// Features: element absorption, aggressive absorption, mass elimination,
// supervariable detection by hashing, approximate external degrees.  The
// output lists the pivots in elimination order; a supervariable's members
// (and variables mass-eliminated with it) follow their representative.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "common.h"
#include "host.h"

namespace sfcdd {

namespace {

enum : int8_t { VAR = 0, ELEM = 1, DEAD = 2 };

struct Amd {
  int64_t n;
  std::vector<int64_t> pe;      // list start in iw
  std::vector<int64_t> len;     // list length
  std::vector<int64_t> elen;    // #elements at the head of a variable's list
  std::vector<int64_t> nv;      // supervariable size (negated while in Lk)
  std::vector<int64_t> degree;  // approx external degree / |Le| for elements
  std::vector<int64_t> w;       // |Le \ Lk| workspace and marks
  std::vector<int64_t> head, next, last;  // degree lists
  std::vector<int64_t> hhead, hnext;      // hash buckets
  std::vector<int64_t> member_next, member_tail;  // member chains per principal
  std::vector<int8_t> status;
  std::vector<int64_t> iw;
  int64_t pfree = 0;
  int64_t wflg = 2;

  void deg_remove(int64_t i) {
    int64_t d = degree[i];
    if (last[i] != -1)
      next[last[i]] = next[i];
    else
      head[d] = next[i];
    if (next[i] != -1) last[next[i]] = last[i];
    next[i] = last[i] = -1;
  }
  void deg_insert(int64_t i, int64_t d) {
    degree[i] = d;
    next[i] = head[d];
    last[i] = -1;
    if (head[d] != -1) last[head[d]] = i;
    head[d] = i;
  }
  void append_members(int64_t into, int64_t from) {
    member_next[member_tail[into]] = from;
    member_tail[into] = member_tail[from];
  }
  int64_t clear_flag(int64_t wf, int64_t lemax) {
    if (wf < 2 || wf + lemax < 0 || wf + lemax > (int64_t(1) << 60)) {
      for (int64_t x = 0; x < n; ++x)
        if (w[x] != 0) w[x] = 1;
      wf = 2;
    }
    return wf;
  }
  // compact all live lists to the front of iw
  void garbage_collect() {
    std::vector<std::pair<int64_t, int64_t>> lists;
    lists.reserve(n);
    for (int64_t j = 0; j < n; ++j)
      if (status[j] != DEAD && pe[j] >= 0) lists.emplace_back(pe[j], j);
    std::sort(lists.begin(), lists.end());
    int64_t dst = 0;
    for (auto& pr : lists) {
      int64_t j = pr.second, src = pe[j];
      for (int64_t t = 0; t < len[j]; ++t) iw[dst + t] = iw[src + t];
      pe[j] = dst;
      dst += len[j];
    }
    pfree = dst;
  }
};

}  // namespace

std::vector<int32_t> amd_order(const SymPattern& A) {
  Amd s;
  const int64_t n = A.n;
  s.n = n;
  if (n == 0) return {};
  int64_t nnz = A.indptr[n];
  s.pe.assign(n, -1);
  s.len.assign(n, 0);
  s.elen.assign(n, 0);
  s.nv.assign(n, 1);
  s.degree.assign(n, 0);
  s.w.assign(n, 1);
  s.head.assign(n + 1, -1);
  s.next.assign(n, -1);
  s.last.assign(n, -1);
  s.hhead.assign(n, -1);
  s.hnext.assign(n, -1);
  s.member_next.assign(n, -1);
  s.member_tail.resize(n);
  s.status.assign(n, VAR);
  s.iw.resize(std::max<int64_t>(2 * nnz + 8 * n, 64));
  for (int64_t i = 0; i < n; ++i) {
    s.member_tail[i] = i;
    s.pe[i] = s.pfree;
    for (int64_t p = A.indptr[i]; p < A.indptr[i + 1]; ++p) {
      int64_t j = A.indices[p];
      if (j == i) continue;
      s.iw[s.pfree++] = j;
    }
    s.len[i] = s.pfree - s.pe[i];
  }
  int64_t mindeg = 0;
  for (int64_t i = 0; i < n; ++i) s.deg_insert(i, s.len[i]);

  std::vector<int32_t> order;
  order.reserve(n);
  std::vector<int64_t> lk;  // members of the new element (principal variables)
  std::vector<int64_t> hashed;
  int64_t nel = 0;
  int64_t lemax = 0;

  while (nel < n) {
    // -- select pivot of minimum approximate degree
    int64_t k = -1;
    for (; mindeg <= n; ++mindeg)
      if ((k = s.head[mindeg]) != -1) break;
    SFCDD_REQUIRE(k >= 0, SFCDD_EINTERNAL, "amd: empty degree lists");
    s.deg_remove(k);
    int64_t elenk = s.elen[k];
    int64_t nvk = s.nv[k];
    nel += nvk;

    // -- ensure space for the new element
    int64_t bound = s.len[k] - elenk;
    for (int64_t p = s.pe[k]; p < s.pe[k] + elenk; ++p) bound += s.len[s.iw[p]];
    if (s.pfree + bound > (int64_t)s.iw.size()) {
      s.garbage_collect();
      if (s.pfree + bound > (int64_t)s.iw.size()) s.iw.resize(2 * (s.pfree + bound));
    }

    // -- construct Lk = union of k's variables and of its elements' variables
    s.nv[k] = -nvk;
    int64_t degme = 0;
    int64_t pk_start = s.pfree;
    lk.clear();
    const int64_t pk = s.pe[k], lenk = s.len[k];
    for (int64_t t = 0; t < lenk; ++t) {
      int64_t e = s.iw[pk + t];
      bool is_elem = t < elenk;
      int64_t p0 = is_elem ? s.pe[e] : pk + t;
      int64_t cnt = is_elem ? s.len[e] : 1;
      for (int64_t u = 0; u < cnt; ++u) {
        int64_t i = s.iw[p0 + u];
        int64_t nvi = s.nv[i];
        if (nvi <= 0) continue;  // already in Lk, or non-principal
        degme += nvi;
        s.nv[i] = -nvi;
        s.iw[s.pfree++] = i;
        lk.push_back(i);
        s.deg_remove(i);
      }
      if (is_elem) {  // absorb e into k
        s.pe[e] = -1;
        s.status[e] = DEAD;
        s.w[e] = 0;
      }
    }
    s.status[k] = ELEM;
    s.pe[k] = pk_start;
    s.len[k] = s.pfree - pk_start;
    s.elen[k] = -2;
    lemax = std::max(lemax, degme);
    s.wflg = s.clear_flag(s.wflg, lemax);

    // -- |Le \ Lk| for all elements adjacent to Lk
    for (int64_t i : lk) {
      int64_t eln = s.elen[i];
      if (eln <= 0) continue;
      int64_t nvi = -s.nv[i];
      int64_t wnvi = s.wflg - nvi;
      for (int64_t p = s.pe[i]; p < s.pe[i] + eln; ++p) {
        int64_t e = s.iw[p];
        int64_t we = s.w[e];
        if (we >= s.wflg)
          we -= nvi;
        else if (we != 0)
          we = s.degree[e] + wnvi;
        s.w[e] = we;
      }
    }

    // -- degree update and element pruning for each i in Lk
    hashed.clear();
    for (int64_t i : lk) {
      int64_t p1 = s.pe[i];
      int64_t p2 = p1 + s.elen[i] - 1;
      int64_t pn = p1;
      int64_t deg = 0;
      uint64_t h = 0;
      for (int64_t p = p1; p <= p2; ++p) {
        int64_t e = s.iw[p];
        if (s.w[e] == 0) continue;  // absorbed
        int64_t dext = s.w[e] - s.wflg;
        if (dext > 0) {
          deg += dext;
          s.iw[pn++] = e;
          h += (uint64_t)e;
        } else {  // aggressive absorption: Le is a subset of Lk
          s.pe[e] = -1;
          s.status[e] = DEAD;
          s.w[e] = 0;
        }
      }
      s.elen[i] = pn - p1 + 1;
      int64_t p3 = pn;
      int64_t p4 = p1 + s.len[i];
      for (int64_t p = p2 + 1; p < p4; ++p) {
        int64_t j = s.iw[p];
        int64_t nvj = s.nv[j];
        if (nvj <= 0) continue;  // in Lk or non-principal
        deg += nvj;
        s.iw[pn++] = j;
        h += (uint64_t)j;
      }
      if (s.elen[i] == 1 && p3 == pn) {
        // mass elimination: i is adjacent only to k
        int64_t nvi = -s.nv[i];
        degme -= nvi;
        nvk += nvi;
        nel += nvi;
        s.nv[i] = 0;
        s.elen[i] = -1;
        s.status[i] = DEAD;
        s.pe[i] = -1;
        s.append_members(k, i);
      } else {
        s.degree[i] = std::min(s.degree[i], deg);
        // new element k goes to the front of i's list
        s.iw[pn] = s.iw[p3];
        s.iw[p3] = s.iw[p1];
        s.iw[p1] = k;
        s.len[i] = pn - p1 + 1;
        int64_t hb = (int64_t)(h % (uint64_t)n);
        s.hnext[i] = s.hhead[hb];
        s.hhead[hb] = i;
        s.last[i] = hb;  // remember bucket (i is off the degree lists now)
        hashed.push_back(i);
      }
    }
    s.degree[k] = degme;
    lemax = std::max(lemax, degme);
    s.wflg = s.clear_flag(s.wflg + lemax, lemax);

    // -- supervariable detection
    for (int64_t i : hashed) {
      if (s.nv[i] >= 0) continue;  // already merged (nv=0) or handled
      int64_t hb = s.last[i];
      if (hb < 0) continue;
      int64_t cur = s.hhead[hb];
      s.hhead[hb] = -1;  // take the whole bucket
      for (int64_t a = cur; a != -1; a = s.hnext[a]) {
        if (s.nv[a] >= 0) continue;
        // mark a's list (excluding k at the front)
        for (int64_t p = s.pe[a] + 1; p < s.pe[a] + s.len[a]; ++p) s.w[s.iw[p]] = s.wflg;
        int64_t prev = a;
        for (int64_t b = s.hnext[a]; b != -1; b = s.hnext[b]) {
          bool same = s.nv[b] < 0 && s.len[b] == s.len[a] && s.elen[b] == s.elen[a];
          if (same)
            for (int64_t p = s.pe[b] + 1; p < s.pe[b] + s.len[b]; ++p)
              if (s.w[s.iw[p]] != s.wflg) {
                same = false;
                break;
              }
          if (same) {  // b indistinguishable from a: absorb
            s.nv[a] += s.nv[b];  // both negative
            s.nv[b] = 0;
            s.elen[b] = -1;
            s.status[b] = DEAD;
            s.pe[b] = -1;
            s.append_members(a, b);
            s.hnext[prev] = s.hnext[b];
          } else {
            prev = b;
          }
        }
        ++s.wflg;
      }
      for (int64_t a = cur; a != -1; a = s.hnext[a]) s.last[a] = -1;
    }
    s.wflg = s.clear_flag(s.wflg, lemax);

    // -- finalize: restore nv, compute degrees, reinsert into degree lists
    int64_t p = 0;
    for (int64_t i : lk) {
      int64_t nvi = -s.nv[i];
      if (nvi <= 0) continue;  // merged or mass-eliminated
      s.nv[i] = nvi;
      s.last[i] = -1;
      int64_t d = s.degree[i] + degme - nvi;
      d = std::min(d, n - nel - nvi);
      d = std::max<int64_t>(d, 0);
      s.deg_insert(i, d);
      mindeg = std::min(mindeg, d);
      s.iw[pk_start + p++] = i;
    }
    s.nv[k] = nvk;
    s.len[k] = p;
    if (p == 0) {
      s.pe[k] = -1;
      s.w[k] = 0;
    }
    // -- emit k and everything it represents
    for (int64_t m = k; m != -1; m = s.member_next[m]) order.push_back((int32_t)m);
  }
  SFCDD_REQUIRE((int64_t)order.size() == n, SFCDD_EINTERNAL, "amd: ordering incomplete");
  return order;
}

}  // namespace sfcdd
