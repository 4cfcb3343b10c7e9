// Fragment partition of the supernodal trees and blob layout (see plan.h).
#include "plan.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>

#include "common.h"

namespace sfcdd {

namespace {

struct Frag {
  int32_t factor = 0;
  std::vector<int32_t> sns;  // supernode ids (ascending = postorder)
  int32_t top = -1;
  bool big = false;
  int32_t parent = -1;
  int32_t nchild = 0;
  int32_t height = 0, depth = 0;
  int64_t blob_off = 0;
  int32_t copy_bytes = 0;
};

// running size of an open cluster (upper bounds)
struct Cluster {
  int64_t meta_ints = 0;
  int64_t vals = 0;
  int64_t frontal = 0;    // sum (2s+m): frontal slots + column values
  int64_t ext_u = 0;      // doubles of external child updates
  int64_t ext_u_cnt = 0;  // number of external children
  int64_t nsn = 0;
};

inline int64_t align16(int64_t x) { return (x + 15) & ~int64_t(15); }

void put_pair(std::vector<int32_t>& v, int32_t lo, int32_t hi) {
  v.push_back((int32_t)((uint32_t)lo | ((uint32_t)hi << 16)));
}

}  // namespace

DevicePlan build_plan(const std::vector<const HostFactor*>& factors, const std::vector<int64_t>& gstart,
                      const std::vector<int64_t>& gmod, const PlanOptions& opt) {
  SFCDD_REQUIRE(opt.scratch_max < 65536, SFCDD_EINTERNAL, "scratch positions must fit 16 bits");
  DevicePlan P;
  P.blob_max = opt.blob_max;
  std::vector<Frag> frags;
  std::vector<std::vector<int32_t>> frag_of(factors.size());
  std::vector<std::vector<int32_t>> upd_slot(factors.size());
  int64_t xy_off = 0;
  for (size_t fi = 0; fi < factors.size(); ++fi) {
    const HostFactor& F = *factors[fi];
    P.factors.push_back(FactorDev{gstart[fi], gmod[fi], xy_off, F.n});
    xy_off += F.n;
    P.num_supernodes += F.sn.size();
    P.stored += F.stored;
    P.nnz_l += F.nnz_l;
    const int64_t ns = F.sn.size();
    auto nch = [&](int64_t k) { return (int64_t)(F.child_ptr[k + 1] - F.child_ptr[k]); };
    auto child_m = [&](int64_t k) {
      int64_t v = 0;
      for (int32_t q = F.child_ptr[k]; q < F.child_ptr[k + 1]; ++q) v += F.sn[F.child_list[q]].m;
      return v;
    };
    std::vector<Cluster> cl(ns);
    std::vector<char> open(ns, 0);
    std::vector<std::vector<int32_t>> members(ns);
    frag_of[fi].assign(ns, -1);
    auto blob_bytes = [&](const Cluster& c, int64_t m_top) {
      int64_t ints = H_WORDS + 2 + c.meta_ints + m_top + c.ext_u;
      return align16(4 * ints) + 8 * c.vals;
    };
    auto scratch_of = [&](const Cluster& c, int64_t m_top) { return c.frontal + m_top + c.ext_u; };
    auto close = [&](int32_t root, bool big) {
      Frag fr;
      fr.factor = (int32_t)fi;
      fr.sns = std::move(members[root]);
      std::sort(fr.sns.begin(), fr.sns.end());
      fr.top = root;
      fr.big = big;
      for (int32_t k : fr.sns) frag_of[fi][k] = (int32_t)frags.size();
      frags.push_back(std::move(fr));
      open[root] = 0;
    };
    for (int64_t k = 0; k < ns; ++k) {
      const Supernode& S = F.sn[k];
      Cluster c;
      c.nsn = 1;
      c.meta_ints = R_WORDS + L_WORDS + 2 * S.s + child_m(k) + (S.s + S.m) + S.m +
                    2 * ((S.s + S.m + 31) / 32 + S.s + 1);
      c.vals = packed_size(S.s, S.m);
      c.frontal = 2 * S.s + S.m;
      c.ext_u = child_m(k);
      c.ext_u_cnt = nch(k);
      const bool big = S.s > SMALL_MAX_S || blob_bytes(c, S.m) > opt.blob_max ||
                       scratch_of(c, S.m) > opt.scratch_max;
      if (big) {
        SFCDD_REQUIRE(2 * S.s + S.m <= opt.scratch_max && S.s + S.m <= opt.big_front_max, SFCDD_EINTERNAL,
                      "supernode front exceeds the shared-memory scratch (s+m = " + std::to_string(S.s + S.m) +
                          ")");
        for (int32_t q = F.child_ptr[k]; q < F.child_ptr[k + 1]; ++q)
          if (open[F.child_list[q]]) close(F.child_list[q], false);
        members[k] = {(int32_t)k};
        close((int32_t)k, true);
        continue;
      }
      members[k] = {(int32_t)k};
      std::vector<int32_t> ok;
      for (int32_t q = F.child_ptr[k]; q < F.child_ptr[k + 1]; ++q)
        if (open[F.child_list[q]]) ok.push_back(F.child_list[q]);
      std::sort(ok.begin(), ok.end(), [&](int32_t a, int32_t b) { return cl[a].vals < cl[b].vals; });
      for (int32_t ch : ok) {
        Cluster t = c;
        const Cluster& d = cl[ch];
        t.nsn += d.nsn;
        t.meta_ints += d.meta_ints;
        t.vals += d.vals;
        t.frontal += d.frontal;
        t.ext_u += d.ext_u - F.sn[ch].m;
        t.ext_u_cnt += d.ext_u_cnt - 1;
        if (blob_bytes(t, S.m) <= opt.blob_max && scratch_of(t, S.m) <= opt.scratch_max) {
          c = t;
          auto& mc = members[ch];
          members[k].insert(members[k].end(), mc.begin(), mc.end());
          mc.clear();
          open[ch] = 0;
        } else {
          close(ch, false);
        }
      }
      cl[k] = c;
      open[k] = 1;
    }
    for (int64_t k = 0; k < ns; ++k)
      if (open[k]) close((int32_t)k, false);
    upd_slot[fi].assign(ns, -1);
    for (int64_t k = 0; k < ns; ++k) {
      const int32_t p = F.sn[k].parent;
      if (p >= 0 && frag_of[fi][p] != frag_of[fi][k]) {
        upd_slot[fi][k] = (int32_t)P.upd_doubles;
        P.upd_doubles += F.sn[k].m;
      }
    }
    SFCDD_REQUIRE(P.upd_doubles < (int64_t(1) << 31), SFCDD_EINTERNAL, "update buffer too large");
  }
  P.xy_doubles = xy_off;
  const int32_t nfrag = (int32_t)frags.size();
  P.nfrag = nfrag;
  for (int32_t f = 0; f < nfrag; ++f) {
    Frag& fr = frags[f];
    const HostFactor& F = *factors[fr.factor];
    int32_t p = F.sn[fr.top].parent;
    fr.parent = p < 0 ? -1 : frag_of[fr.factor][p];
    if (fr.parent >= 0) frags[fr.parent].nchild++;
  }
  // creation order is children-before-parents within a factor
  for (int32_t f = 0; f < nfrag; ++f)
    if (frags[f].parent >= 0)
      frags[frags[f].parent].height = std::max(frags[frags[f].parent].height, frags[f].height + 1);
  for (int32_t f = nfrag - 1; f >= 0; --f) frags[f].depth = frags[f].parent < 0 ? 0 : frags[frags[f].parent].depth + 1;

  // ---- blobs
  std::vector<int32_t> ints;
  std::vector<double> vals;
  std::vector<int32_t> loc;
  std::vector<std::vector<int32_t>> col2sn(factors.size());
  for (size_t fi = 0; fi < factors.size(); ++fi) {
    const HostFactor& F = *factors[fi];
    col2sn[fi].assign(F.n, -1);
    for (size_t k = 0; k < F.sn.size(); ++k)
      for (int32_t t = 0; t < F.sn[k].s; ++t) col2sn[fi][F.sn[k].col0 + t] = (int32_t)k;
  }
  for (int32_t f = 0; f < nfrag; ++f) {
    Frag& fr = frags[f];
    const HostFactor& F = *factors[fr.factor];
    const int32_t nsn = (int32_t)fr.sns.size();
    const Supernode& Top = F.sn[fr.top];
    ints.assign(H_WORDS, 0);
    vals.clear();
    ints[H_NSN] = nsn;
    ints[H_BIG] = fr.big ? 1 : 0;
    ints[H_TOP_UPD] = upd_slot[fr.factor][fr.top];
    int32_t scratch_used = 0;
    if (fr.big) {
      const Supernode& S = Top;
      ints[H_NLEV] = 1;
      ints[H_TOP] = 0;
      ints[H_NCOL] = S.s;
      ints[H_COLS] = (int32_t)ints.size();
      for (int32_t c = 0; c < S.s; ++c) ints.push_back(F.perm[S.col0 + c]);
      ints[H_REC] = (int32_t)ints.size();
      ints.resize(ints.size() + R_WORDS, 0);
      const int32_t rec = ints[H_REC];
      ints[rec + R_S] = S.s;
      ints[rec + R_M] = S.m;
      ints[rec + R_VAL] = 0;
      ints[rec + R_ROWS] = (int32_t)ints.size();
      for (int32_t a = 0; a < S.m; ++a) ints.push_back(F.perm[F.rows[S.rows_off + a]]);
      const int32_t k = fr.top;
      const int32_t nc = F.child_ptr[k + 1] - F.child_ptr[k];
      ints[rec + R_NCH] = nc;
      const int32_t chrec = (int32_t)ints.size();
      ints[rec + R_CH] = chrec;
      ints.resize(ints.size() + (size_t)CH_WORDS * nc, 0);
      for (int32_t q = 0; q < nc; ++q) {
        const int32_t c = F.child_list[F.child_ptr[k] + q];
        const Supernode& K = F.sn[c];
        const int32_t rel_off = (int32_t)ints.size();
        ints.insert(ints.end(), F.rel.begin() + K.rel_off, F.rel.begin() + K.rel_off + K.m);
        ints[chrec + CH_WORDS * q] = upd_slot[fr.factor][c];
        ints[chrec + CH_WORDS * q + 1] = K.m;
        ints[chrec + CH_WORDS * q + 2] = rel_off;
        SFCDD_REQUIRE(upd_slot[fr.factor][c] >= 0, SFCDD_EINTERNAL, "big child without update slot");
      }
      const double* v = F.val.data() + S.val_off;
      vals.insert(vals.end(), v, v + packed_size(S.s, S.m));
      scratch_used = 2 * S.s + S.m;  // v/f + backward column accumulators
    } else {
      loc.assign(F.sn.size(), -1);
      for (int32_t t = 0; t < nsn; ++t) loc[fr.sns[t]] = t;
      std::vector<int32_t> lev(nsn, 0);
      int32_t nlev = 0;
      for (int32_t t = 0; t < nsn; ++t) {
        const int32_t k = fr.sns[t];
        for (int32_t q = F.child_ptr[k]; q < F.child_ptr[k + 1]; ++q) {
          const int32_t c = F.child_list[q];
          if (loc[c] >= 0) lev[t] = std::max(lev[t], lev[loc[c]] + 1);
        }
        nlev = std::max(nlev, lev[t] + 1);
      }
      auto front = [&](int32_t t) { return F.sn[fr.sns[t]].s + F.sn[fr.sns[t]].m; };
      // level order (small fronts first within a level: better lane packing)
      std::vector<int32_t> ord(nsn);
      std::iota(ord.begin(), ord.end(), 0);
      std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) {
        if (lev[a] != lev[b]) return lev[a] < lev[b];
        return front(a) < front(b);
      });
      std::vector<int32_t> lid(nsn);  // postorder index -> level-order id
      for (int32_t i = 0; i < nsn; ++i) lid[ord[i]] = i;
      auto sn_of = [&](int32_t id) -> const Supernode& { return F.sn[fr.sns[ord[id]]]; };
      // scratch layout
      std::vector<int32_t> scr(nsn), cpos(nsn);
      int32_t pos = 0;
      for (int32_t i = 0; i < nsn; ++i) {
        scr[i] = pos;
        pos += sn_of(i).s + sn_of(i).m;
      }
      for (int32_t i = 0; i < nsn; ++i) {
        cpos[i] = pos;
        pos += sn_of(i).s;
      }
      std::map<int32_t, int32_t> extx;  // permuted row -> staging position (rows of the top)
      for (int32_t a = 0; a < Top.m; ++a) extx[F.rows[Top.rows_off + a]] = pos + a;
      const int32_t extx_base = pos;
      pos += Top.m;
      std::map<int32_t, int32_t> extu_pos;  // external child -> staging position
      std::vector<int32_t> extu;            // global update index per staged double
      const int32_t extu_base = pos;
      for (int32_t i = 0; i < nsn; ++i) {
        const int32_t k = fr.sns[ord[i]];
        for (int32_t q = F.child_ptr[k]; q < F.child_ptr[k + 1]; ++q) {
          const int32_t c = F.child_list[q];
          if (loc[c] >= 0) continue;
          extu_pos[c] = pos;
          for (int32_t a = 0; a < F.sn[c].m; ++a) extu.push_back(upd_slot[fr.factor][c] + a);
          pos += F.sn[c].m;
        }
      }
      scratch_used = pos;
      ints[H_NLEV] = nlev;
      ints[H_TOP] = lid[loc[fr.top]];
      // columns
      ints[H_NCOL] = 0;
      ints[H_COLS] = (int32_t)ints.size();
      for (int32_t i = 0; i < nsn; ++i)
        for (int32_t c = 0; c < sn_of(i).s; ++c) ints.push_back(F.perm[sn_of(i).col0 + c]);
      ints[H_NCOL] = (int32_t)ints.size() - ints[H_COLS];
      ints[H_COLPOS] = (int32_t)ints.size();
      for (int32_t i = 0; i < nsn; ++i)
        for (int32_t c = 0; c < sn_of(i).s; ++c) put_pair(ints, scr[i] + c, cpos[i] + c);
      ints[H_NEXTX] = Top.m;
      ints[H_EXTX_BASE] = extx_base;
      ints[H_EXTX] = (int32_t)ints.size();
      for (int32_t a = 0; a < Top.m; ++a) ints.push_back(F.perm[F.rows[Top.rows_off + a]]);
      ints[H_NEXTU] = (int32_t)extu.size();
      ints[H_EXTU_BASE] = extu_base;
      ints[H_EXTU] = (int32_t)ints.size();
      ints.insert(ints.end(), extu.begin(), extu.end());
      // records
      ints[H_REC] = (int32_t)ints.size();
      ints.resize(ints.size() + (size_t)R_WORDS * nsn, 0);
      for (int32_t i = 0; i < nsn; ++i) {
        const Supernode& S = sn_of(i);
        int32_t* R = &ints[ints[H_REC] + R_WORDS * i];
        R[R_S] = S.s;
        R[R_M] = S.m;
        R[R_VAL] = (int32_t)vals.size();
        R[R_SCR] = scr[i];
        R[R_CPOS] = cpos[i];
        const double* v = F.val.data() + S.val_off;
        vals.insert(vals.end(), v, v + packed_size(S.s, S.m));
      }
      // per-level tables
      std::vector<int32_t> levtab((size_t)L_WORDS * nlev, 0), runs, gpairs, bpairs, items;
      std::vector<std::pair<int32_t, int32_t>> jp;  // (dst, src) per supernode
      int32_t i = 0;
      for (int32_t l = 0; l < nlev; ++l) {
        int32_t* L = &levtab[(size_t)L_WORDS * l];
        L[L_REC0] = i;
        while (i < nsn && lev[ord[i]] == l) ++i;
        L[L_REC1] = i;
        // forward gather runs
        L[L_RUN0] = (int32_t)runs.size();
        for (int32_t j = L[L_REC0]; j < L[L_REC1]; ++j) {
          const int32_t k = fr.sns[ord[j]];
          jp.clear();
          for (int32_t q = F.child_ptr[k]; q < F.child_ptr[k + 1]; ++q) {
            const int32_t c = F.child_list[q];
            const Supernode& K = F.sn[c];
            const int32_t src = loc[c] >= 0 ? scr[lid[loc[c]]] + K.s : extu_pos[c];
            for (int32_t a = 0; a < K.m; ++a) jp.emplace_back(scr[j] + F.rel[K.rel_off + a], src + a);
          }
          std::stable_sort(jp.begin(), jp.end(),
                           [](const std::pair<int32_t, int32_t>& x, const std::pair<int32_t, int32_t>& y) {
                             return x.first < y.first;
                           });
          for (size_t e = 0; e < jp.size(); ++e) {
            if (e == 0 || jp[e].first != jp[e - 1].first) runs.push_back((int32_t)gpairs.size());
            put_pair(gpairs, jp[e].first, jp[e].second);
          }
        }
        L[L_RUN1] = (int32_t)runs.size();
        // backward row pairs: v_B = -x(rows)
        L[L_BP0] = (int32_t)bpairs.size();
        for (int32_t j = L[L_REC0]; j < L[L_REC1]; ++j) {
          const Supernode& S = sn_of(j);
          for (int32_t a = 0; a < S.m; ++a) {
            const int32_t r = F.rows[S.rows_off + a];
            const int32_t owner = col2sn[fr.factor][r];
            int32_t src;
            if (owner >= 0 && loc[owner] >= 0) {
              src = cpos[lid[loc[owner]]] + (r - (int32_t)F.sn[owner].col0);
            } else {
              auto it = extx.find(r);
              SFCDD_REQUIRE(it != extx.end(), SFCDD_EINTERNAL, "row outside fragment and top rows");
              src = it->second;
            }
            put_pair(bpairs, scr[j] + S.s + a, src);
          }
        }
        L[L_BP1] = (int32_t)bpairs.size();
        // warp items (forward then backward), LPT-assigned to the warps
        for (int pass = 0; pass < 2; ++pass) {
          struct Item {
            int32_t x, y;
            double cost;
          };
          std::vector<Item> lst;
          int32_t j = L[L_REC0];
          while (j < L[L_REC1]) {
            const Supernode& S = sn_of(j);
            if (S.s + S.m <= 32) {
              int32_t j1 = j, rows = 0, smax = 0;
              uint32_t mask = 0;  // lane of each segment start, plus the end lane
              while (j1 < L[L_REC1] && rows + sn_of(j1).s + sn_of(j1).m <= 32) {
                mask |= 1u << rows;
                rows += sn_of(j1).s + sn_of(j1).m;
                smax = std::max<int32_t>(smax, sn_of(j1).s);
                ++j1;
              }
              if (rows < 32) mask |= 1u << rows;
              SFCDD_REQUIRE(j < 65536 && j1 - j < 32768, SFCDD_EINTERNAL, "packed item index overflow");
              lst.push_back({j | ((j1 - j) << 16), (int32_t)mask, 40.0 + (pass == 0 ? 4.0 : 12.0) * smax});
              j = j1;
            } else if (pass == 0) {
              for (int32_t b = 0; b < (S.s + S.m + 31) / 32; ++b)
                lst.push_back({j, b, 20.0 + 4.0 * std::min(S.s, 32 * b + 32)});
              ++j;
            } else {
              for (int32_t k = 0; k < S.s; ++k) lst.push_back({j, k, 30.0 + 4.0 * ((S.s + S.m - k + 31) / 32)});
              ++j;
            }
          }
          std::stable_sort(lst.begin(), lst.end(), [](const Item& a, const Item& b) { return a.cost > b.cost; });
          std::vector<std::vector<Item>> per(NWARP_PLAN);
          std::vector<double> load(NWARP_PLAN, 0.0);
          for (const Item& it : lst) {
            const int w = (int)(std::min_element(load.begin(), load.end()) - load.begin());
            per[w].push_back(it);
            load[w] += it.cost;
          }
          int32_t* W = L + (pass == 0 ? L_FW : L_BW);
          for (int w = 0; w < NWARP_PLAN; ++w) {
            W[w] = (int32_t)items.size() / 2;
            for (const Item& it : per[w]) items.insert(items.end(), {it.x, it.y});
          }
          W[NWARP_PLAN] = (int32_t)items.size() / 2;
        }
      }
      runs.push_back((int32_t)gpairs.size());
      ints[H_LEVELS] = (int32_t)ints.size();
      ints.insert(ints.end(), levtab.begin(), levtab.end());
      ints[H_RUNS] = (int32_t)ints.size();
      ints.insert(ints.end(), runs.begin(), runs.end());
      ints[H_GPAIRS] = (int32_t)ints.size();
      ints.insert(ints.end(), gpairs.begin(), gpairs.end());
      ints[H_BPAIRS] = (int32_t)ints.size();
      ints.insert(ints.end(), bpairs.begin(), bpairs.end());
      if (ints.size() & 1) ints.push_back(0);  // int2 alignment of the items
      ints[H_ITEMS] = (int32_t)ints.size();
      ints.insert(ints.end(), items.begin(), items.end());
    }
    ints[H_SCRATCH] = scratch_used;
    const int64_t meta_bytes = align16(4 * (int64_t)ints.size());
    ints[H_VAL_OFF] = (int32_t)meta_bytes;
    const int64_t val_bytes = align16(8 * (int64_t)vals.size());
    fr.blob_off = P.blobs.size();
    fr.copy_bytes = fr.big ? 0 : (int32_t)(meta_bytes + val_bytes);
    SFCDD_REQUIRE(fr.copy_bytes <= opt.blob_max, SFCDD_EINTERNAL, "fragment blob exceeds shared-memory budget");
    SFCDD_REQUIRE(scratch_used <= opt.scratch_max, SFCDD_EINTERNAL, "fragment scratch exceeds budget");
    P.blobs.resize(P.blobs.size() + meta_bytes + val_bytes, 0);
    std::memcpy(P.blobs.data() + fr.blob_off, ints.data(), 4 * ints.size());
    std::memcpy(P.blobs.data() + fr.blob_off + meta_bytes, vals.data(), 8 * vals.size());
    P.max_scratch = std::max<int32_t>(P.max_scratch, scratch_used);
    P.max_copy = std::max(P.max_copy, fr.copy_bytes);
    if (fr.big) ++P.nbig;
  }
  // ---- task order: decreasing critical-path rank over the combined
  // forward/backward DAG (HLFET list scheduling).  Weights are a rough
  // per-task time model in microseconds (fixed cost + streamed bytes).
  std::vector<double> wt(nfrag), rank_f(nfrag, 0.0), rank_b(nfrag, 0.0);
  std::vector<std::vector<int32_t>> fkids(nfrag);
  for (int32_t f = 0; f < nfrag; ++f) {
    const Frag& fr = frags[f];
    const HostFactor& F = *factors[fr.factor];
    int64_t v = 0;
    for (int32_t k : fr.sns) v += packed_size(F.sn[k].s, F.sn[k].m);
    wt[f] = fr.big ? 3.0 + 8.0 * v / 40e3 : 3.0 + 8.0 * v / 15e3;
    if (fr.parent >= 0) fkids[fr.parent].push_back(f);
  }
  for (int32_t f = 0; f < nfrag; ++f) {  // children before parents
    double mx = 0.0;
    for (int32_t c : fkids[f]) mx = std::max(mx, rank_b[c]);
    rank_b[f] = wt[f] + mx;
  }
  for (int32_t f = nfrag - 1; f >= 0; --f)  // parents before children
    rank_f[f] = wt[f] + (frags[f].parent >= 0 ? rank_f[frags[f].parent] : rank_b[f]);
  std::vector<int32_t> order(2 * (size_t)nfrag);
  std::iota(order.begin(), order.end(), 0);  // id < nfrag: forward of id; else backward of id - nfrag
  auto rank_of = [&](int32_t id) { return id < nfrag ? rank_f[id] : rank_b[id - nfrag]; };
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return rank_of(a) > rank_of(b); });
  P.tasks.resize(2 * (size_t)nfrag);
  for (size_t t = 0; t < order.size(); ++t) {
    const bool bwd = order[t] >= nfrag;
    const int32_t f = bwd ? order[t] - nfrag : order[t];
    const Frag& fr = frags[f];
    TaskDev& T = P.tasks[t];
    T.blob_off = fr.blob_off;
    T.copy_bytes = fr.copy_bytes;
    T.frag = f;
    T.factor = fr.factor;
    T.wait_on = bwd ? fr.parent : fr.nchild;  // bwd: -1 = wait for own forward
    T.signal = bwd ? -1 : fr.parent;
    T.flags = (fr.big ? TASK_BIG : 0) | (bwd ? TASK_BWD : 0);
  }
  if (std::getenv("SFCDD_PLAN_DEBUG")) {
    int64_t big_vals = 0, small_vals = 0, lev_sum = 0, sn_sum = 0, maxh = 0;
    for (const Frag& fr : frags) {
      const HostFactor& F = *factors[fr.factor];
      int64_t v = 0;
      for (int32_t k : fr.sns) v += packed_size(F.sn[k].s, F.sn[k].m);
      const int32_t* h = reinterpret_cast<const int32_t*>(P.blobs.data() + fr.blob_off);
      if (fr.big) {
        big_vals += v;
      } else {
        small_vals += v;
        lev_sum += h[H_NLEV];
        sn_sum += fr.sns.size();
      }
      maxh = std::max<int64_t>(maxh, fr.height);
    }
    const int64_t ns = nfrag - P.nbig;
    std::fprintf(stderr,
                 "[plan] frags=%d big=%d (%.1f%% of values) small: avg %.1f supernodes, %.1f levels, "
                 "avg blob %.1f KB; max frag height %lld; blob total %.1f MB (values %.1f MB)\n",
                 nfrag, P.nbig, 100.0 * big_vals / std::max<int64_t>(1, big_vals + small_vals),
                 (double)sn_sum / std::max<int64_t>(1, ns), (double)lev_sum / std::max<int64_t>(1, ns),
                 P.blobs.size() / 1024.0 / std::max(1, nfrag), (long long)maxh, P.blobs.size() / 1e6,
                 8e-6 * (big_vals + small_vals));
  }
  return P;
}

}  // namespace sfcdd
