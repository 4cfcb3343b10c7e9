// Fragment partition of the supernodal trees and blob layout (see plan.h).
#include "plan.h"

#include <algorithm>
#include <cstring>
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

inline int64_t align16(int64_t x) { return (x + 15) & ~int64_t(15); }

}  // namespace

DevicePlan build_plan(const std::vector<const HostFactor*>& factors, const std::vector<int64_t>& gstart,
                      const std::vector<int64_t>& gmod, const PlanOptions& opt) {
  DevicePlan P;
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
    auto nch = [&](int64_t k) { return F.child_ptr[k + 1] - F.child_ptr[k]; };
    auto meta_ints = [&](int64_t k) {
      int64_t v = 1 + R_WORDS + F.sn[k].s + F.sn[k].m + CH_WORDS * nch(k);
      for (int32_t q = F.child_ptr[k]; q < F.child_ptr[k + 1]; ++q) v += F.sn[F.child_list[q]].m;
      return v;
    };
    auto cost = [&](int64_t k) { return 4 * meta_ints(k) + 8 * packed_size(F.sn[k].s, F.sn[k].m) + 8; };
    const int64_t budget = opt.blob_max - 4 * H_WORDS - 64;
    std::vector<int64_t> w(ns, 0), sc(ns, 0);
    std::vector<char> open(ns, 0);
    std::vector<std::vector<int32_t>> members(ns);
    frag_of[fi].assign(ns, -1);
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
    std::vector<int32_t> kids;
    for (int64_t k = 0; k < ns; ++k) {
      kids.assign(F.child_list.begin() + F.child_ptr[k], F.child_list.begin() + F.child_ptr[k + 1]);
      const int64_t sk = F.sn[k].s + F.sn[k].m;
      const bool big = cost(k) > budget || sk > opt.scratch_max;
      if (big) {
        for (int32_t c : kids)
          if (open[c]) close(c, false);
        members[k] = {(int32_t)k};
        close((int32_t)k, true);
        continue;
      }
      w[k] = cost(k);
      sc[k] = sk;
      members[k] = {(int32_t)k};
      std::vector<int32_t> ok;
      for (int32_t c : kids)
        if (open[c]) ok.push_back(c);
      std::sort(ok.begin(), ok.end(), [&](int32_t a, int32_t b) { return w[a] < w[b]; });
      for (int32_t c : ok) {
        if (w[k] + w[c] <= budget && sc[k] + sc[c] <= opt.scratch_max) {
          w[k] += w[c];
          sc[k] += sc[c];
          auto& mc = members[c];
          members[k].insert(members[k].end(), mc.begin(), mc.end());
          mc.clear();
          open[c] = 0;
        } else {
          close(c, false);
        }
      }
      open[k] = 1;
    }
    for (int64_t k = 0; k < ns; ++k)
      if (open[k]) close((int32_t)k, false);
    // update slots for fragment tops with a parent
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
  // fragment tree
  for (int32_t f = 0; f < nfrag; ++f) {
    Frag& fr = frags[f];
    const HostFactor& F = *factors[fr.factor];
    int32_t p = F.sn[fr.top].parent;
    fr.parent = p < 0 ? -1 : frag_of[fr.factor][p];
    if (fr.parent >= 0) frags[fr.parent].nchild++;
  }
  // creation order is children-before-parents within a factor
  for (int32_t f = 0; f < nfrag; ++f)
    if (frags[f].parent >= 0) frags[frags[f].parent].height = std::max(frags[frags[f].parent].height, frags[f].height + 1);
  for (int32_t f = nfrag - 1; f >= 0; --f)
    frags[f].depth = frags[f].parent < 0 ? 0 : frags[frags[f].parent].depth + 1;

  // ---- blobs
  std::vector<int32_t> ints;
  std::vector<double> vals;
  std::vector<int32_t> loc;
  for (int32_t f = 0; f < nfrag; ++f) {
    Frag& fr = frags[f];
    const HostFactor& F = *factors[fr.factor];
    const int32_t nsn = (int32_t)fr.sns.size();
    loc.assign(F.sn.size(), -1);  // O(ns) per fragment; fine for setup
    for (int32_t t = 0; t < nsn; ++t) loc[fr.sns[t]] = t;
    // in-fragment levels
    std::vector<int32_t> lev(nsn, 0);
    int32_t nlev = 0;
    for (int32_t t = 0; t < nsn; ++t) {
      int32_t k = fr.sns[t];
      for (int32_t q = F.child_ptr[k]; q < F.child_ptr[k + 1]; ++q) {
        int32_t c = F.child_list[q];
        if (loc[c] >= 0) lev[t] = std::max(lev[t], lev[loc[c]] + 1);
      }
      nlev = std::max(nlev, lev[t] + 1);
    }
    std::vector<int32_t> lev_list(nsn);
    std::iota(lev_list.begin(), lev_list.end(), 0);
    std::stable_sort(lev_list.begin(), lev_list.end(), [&](int32_t a, int32_t b) { return lev[a] < lev[b]; });
    std::vector<int32_t> lev_ptr(nlev + 1, 0);
    for (int32_t t = 0; t < nsn; ++t) lev_ptr[lev[t] + 1]++;
    for (int32_t l = 0; l < nlev; ++l) lev_ptr[l + 1] += lev_ptr[l];

    ints.assign(H_WORDS, 0);
    ints[H_NSN] = nsn;
    ints[H_NLEV] = nlev;
    ints[H_LEV_PTR] = (int32_t)ints.size();
    ints.insert(ints.end(), lev_ptr.begin(), lev_ptr.end());
    ints[H_LEV_LIST] = (int32_t)ints.size();
    ints.insert(ints.end(), lev_list.begin(), lev_list.end());
    ints[H_REC] = (int32_t)ints.size();
    ints.resize(ints.size() + (size_t)R_WORDS * nsn, 0);
    vals.clear();
    int32_t scratch = 0;
    for (int32_t t = 0; t < nsn; ++t) {
      const int32_t k = fr.sns[t];
      const Supernode& S = F.sn[k];
      const int32_t rec = ints[H_REC] + R_WORDS * t;
      ints[rec + R_S] = S.s;
      ints[rec + R_M] = S.m;
      ints[rec + R_VAL] = (int32_t)vals.size();
      ints[rec + R_SCR] = scratch;
      scratch += S.s + S.m;
      ints[rec + R_PARENT] = (S.parent >= 0 && loc[S.parent] >= 0) ? loc[S.parent] : -1;
      ints[rec + R_IDX] = (int32_t)ints.size();
      for (int32_t c = 0; c < S.s; ++c) ints.push_back(F.perm[S.col0 + c]);
      for (int32_t a = 0; a < S.m; ++a) ints.push_back(F.perm[F.rows[S.rows_off + a]]);
      const int32_t nc = F.child_ptr[k + 1] - F.child_ptr[k];
      ints[rec + R_NCH] = nc;
      const int32_t chrec = (int32_t)ints.size();
      ints[rec + R_CH] = chrec;
      ints.resize(ints.size() + (size_t)CH_WORDS * nc, 0);
      for (int32_t q = 0; q < nc; ++q) {
        const int32_t c = F.child_list[F.child_ptr[k] + q];
        const Supernode& K = F.sn[c];
        int32_t* cr = &ints[chrec + CH_WORDS * q];
        cr[0] = loc[c];  // -1 if external
        cr[1] = K.m;
        cr[3] = loc[c] >= 0 ? -1 : upd_slot[fr.factor][c];
        SFCDD_REQUIRE(loc[c] >= 0 || cr[3] >= 0, SFCDD_EINTERNAL, "external child without update slot");
        int32_t rel_off = (int32_t)ints.size();
        ints.insert(ints.end(), F.rel.begin() + K.rel_off, F.rel.begin() + K.rel_off + K.m);
        ints[chrec + CH_WORDS * q + 2] = rel_off;
      }
      if (!fr.big || true) {
        const double* v = F.val.data() + S.val_off;
        vals.insert(vals.end(), v, v + packed_size(S.s, S.m));
      }
    }
    ints[H_SCRATCH] = scratch;
    ints[H_TOP] = loc[fr.top];
    ints[H_TOP_UPD] = upd_slot[fr.factor][fr.top];
    const int64_t meta_bytes = align16(4 * (int64_t)ints.size());
    ints[H_VAL_OFF] = (int32_t)meta_bytes;
    const int64_t val_bytes = align16(8 * (int64_t)vals.size());
    fr.blob_off = P.blobs.size();
    fr.copy_bytes = (int32_t)(fr.big ? meta_bytes : meta_bytes + val_bytes);
    SFCDD_REQUIRE(fr.copy_bytes <= opt.blob_max, SFCDD_EINTERNAL, "fragment blob exceeds shared-memory budget");
    P.blobs.resize(P.blobs.size() + meta_bytes + val_bytes, 0);
    std::memcpy(P.blobs.data() + fr.blob_off, ints.data(), 4 * ints.size());
    std::memcpy(P.blobs.data() + fr.blob_off + meta_bytes, vals.data(), 8 * vals.size());
    P.max_scratch = std::max(P.max_scratch, scratch);
    P.max_copy = std::max(P.max_copy, fr.copy_bytes);
  }
  // ---- task order
  std::vector<int32_t> fwd(nfrag), bwd(nfrag);
  std::iota(fwd.begin(), fwd.end(), 0);
  std::iota(bwd.begin(), bwd.end(), 0);
  std::stable_sort(fwd.begin(), fwd.end(), [&](int32_t a, int32_t b) { return frags[a].height < frags[b].height; });
  std::stable_sort(bwd.begin(), bwd.end(), [&](int32_t a, int32_t b) { return frags[a].depth < frags[b].depth; });
  P.tasks.resize(2 * (size_t)nfrag);
  for (int32_t t = 0; t < nfrag; ++t) {
    const Frag& fr = frags[fwd[t]];
    TaskDev& T = P.tasks[t];
    T.blob_off = fr.blob_off;
    T.copy_bytes = fr.copy_bytes;
    T.frag = fwd[t];
    T.factor = fr.factor;
    T.wait_on = fr.nchild;
    T.signal = fr.parent;
    T.big = fr.big ? 1 : 0;
  }
  for (int32_t t = 0; t < nfrag; ++t) {
    const Frag& fr = frags[bwd[t]];
    TaskDev& T = P.tasks[nfrag + t];
    T.blob_off = fr.blob_off;
    T.copy_bytes = fr.copy_bytes;
    T.frag = bwd[t];
    T.factor = fr.factor;
    T.wait_on = fr.parent;  // -1: wait for own forward
    T.signal = -1;
    T.big = fr.big ? 1 : 0;
  }
  return P;
}

}  // namespace sfcdd
