// Group partition of the supernodal trees, blob layouts and the task queue
// of the warp-task dataflow solve (see plan.h).
#include "plan.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <string>
#include <thread>
#include <mutex>

#include "common.h"

namespace sfcdd {

namespace {

struct Group {
  int32_t factor = 0;
  bool big = false;
  std::vector<int32_t> sns;  // supernode ids, ascending (= postorder)
  int32_t top = -1;           // BIG: the supernode; FRAG: the first top
  std::vector<int32_t> tops;  // FRAG: the roots of the group's subtrees (siblings: one parent supernode)
  int32_t parent = -1;  // parent group
  std::vector<int32_t> kids;
  std::vector<int32_t> ftask, btask;  // indices into the unordered task list
  std::vector<int32_t> atask, xtask;  // BIG: assembly / -x_B gather tasks
  int64_t y_off = -1;                 // BIG: global y slot
  int64_t f_off = -1;                 // BIG: assembled front [f_J ; f_B] (s + m)
  int64_t xb_off = -1;                // BIG: -x_B (m)
  int32_t height = 0;
};

// alignment padding and the run-table sentinel of a FRAG blob (ints)
constexpr int64_t FRAG_PAD = 8;

// running size of an open FRAG cluster (upper bounds)
struct Cluster {
  int64_t meta_ints = 0;
  int64_t vals = 0;
  int64_t frontal = 0;    // sum (2s+m): frontal slots + column values
  int64_t ext_u = 0;      // doubles of external child updates
  int64_t nsn = 0;
  int64_t height = 1;     // tree levels of the cluster (one level-table row each)
};

inline int64_t align16(int64_t x) { return (x + 15) & ~int64_t(15); }

void put_pair(std::vector<int32_t>& v, int32_t lo, int32_t hi) {
  v.push_back((int32_t)((uint32_t)lo | ((uint32_t)hi << 16)));
}

// Blob output of one factor (factor-local offsets; merged in factor order).
struct FactorEmit {
  bool defer = false;
  int32_t factor = 0;
  int64_t size = 0;                  // device bytes emitted (local offsets)
  std::vector<uint8_t> image;        // all bytes, or metadata only (defer)
  std::vector<MetaSeg> segs;         // defer: local dev_off / image host_off
  std::vector<ValDesc> vdesc;        // dst = local device byte offset
  std::vector<int64_t> asm_patches;  // image byte offsets of asm16 words to rebase
  std::vector<TaskDev> tasks;
  std::vector<double> tw;
  int32_t max_scratch = 0, max_copy = 0;
  int64_t max_slot = 0;  // max over tasks of align128(blob bytes) + 8 * scratch doubles
  void need_slot(int32_t bytes, int64_t scratch_doubles) {
    max_slot = std::max<int64_t>(max_slot, ((int64_t)bytes + 127) / 128 * 128 + 8 * scratch_doubles);
  }
  bool has_direct = false;
  bool has_mrow = false;

  int64_t put_meta(const std::vector<int32_t>& ints, int64_t meta_bytes) {
    const int64_t off = size;
    const int64_t h = (int64_t)image.size();
    if (defer) segs.push_back(MetaSeg{off, h, meta_bytes});
    image.resize(h + meta_bytes, 0);
    std::memcpy(image.data() + h, ints.data(), 4 * ints.size());
    size += meta_bytes;
    return h;
  }
  // metadata-only record (global assembly record of a huge supernode)
  int64_t raw(const std::vector<int32_t>& ints) {
    const int64_t off = size;
    put_meta(ints, align16(4 * (int64_t)ints.size()));
    return off;
  }
  // one blob: metadata + nvals values placed by descriptors (their dst is
  // relative to the value area); asm_word >= 0: that int holds asm16
  int64_t emit_descs(std::vector<int32_t>& ints, int32_t val_off_word, int64_t nvals, const ValDesc* vd, size_t nvd,
                     int32_t& copy_bytes, const HostFactor* F, int32_t asm_word = -1, bool meta_only = false) {
    const int64_t meta_bytes = align16(4 * (int64_t)ints.size());
    if (val_off_word >= 0) ints[val_off_word] = (int32_t)meta_bytes;
    const int64_t val_bytes = align16(8 * nvals);
    const int64_t off = size;
    const int64_t h = put_meta(ints, meta_bytes);
    if (asm_word >= 0) asm_patches.push_back(h + 4 * (int64_t)asm_word);
    if (!defer) image.resize(image.size() + val_bytes, 0);
    size += val_bytes;
    for (size_t i = 0; i < nvd; ++i) {
      ValDesc d = vd[i];
      d.dst += off + meta_bytes;
      d.factor = factor;
      vdesc.push_back(d);
      if (!defer) {
        SFCDD_REQUIRE(F && !F->val.empty(), SFCDD_EINTERNAL, "plan without values needs defer_values");
        ValDesc hd = d;
        hd.dst -= off;  // into this blob's bytes of the image (image offset == off here)
        place_values(hd, F->val.data() + d.src, image.data() + h);
      }
    }
    // ROW / COL tasks copy their metadata only; the values stay in HBM
    copy_bytes = (int32_t)(meta_only ? meta_bytes : meta_bytes + val_bytes);
    max_copy = std::max(max_copy, copy_bytes);
    return off;
  }
  int64_t emit(std::vector<int32_t>& ints, int32_t val_off_word, int64_t nvals, const ValDesc* vd,
               int32_t& copy_bytes, const HostFactor& F, int32_t asm_word = -1, bool meta_only = false) {
    return emit_descs(ints, val_off_word, nvals, vd, vd ? 1 : 0, copy_bytes, &F, asm_word, meta_only);
  }
  int64_t emit(std::vector<int32_t>& ints, int32_t val_off_word, int64_t nvals, const ValDesc* vd,
               int32_t& copy_bytes) {
    return emit_descs(ints, val_off_word, nvals, vd, vd ? 1 : 0, copy_bytes, nullptr);
  }
  int64_t emit_frag(std::vector<int32_t>& ints, int32_t val_off_word, int64_t nvals, const std::vector<ValDesc>& vd,
                    int32_t& copy_bytes, const HostFactor& F) {
    return emit_descs(ints, val_off_word, nvals, vd.data(), vd.size(), copy_bytes, &F);
  }
};

template <class Fn>
void parallel_range(int64_t n, int threads, Fn fn) {
  if (threads <= 0) threads = hardware_threads();
  threads = (int)std::max<int64_t>(1, std::min<int64_t>(threads, n));
  if (threads == 1) {
    for (int64_t i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<int64_t> next{0};
  std::vector<std::thread> pool;
  std::exception_ptr err;
  std::mutex mu;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&]() {
      for (;;) {
        const int64_t i = next.fetch_add(1);
        if (i >= n) return;
        try {
          fn(i);
        } catch (...) {
          std::lock_guard<std::mutex> g(mu);
          if (!err) err = std::current_exception();
          next = n;
          return;
        }
      }
    });
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

inline int64_t blob_size(int64_t ints, int64_t vals) { return align16(4 * ints) + align16(8 * vals); }

}  // namespace

PlanOptions::PlanOptions() {
  if (const char* e = std::getenv("SFCDD_BLOB_MAX")) blob_max = std::atoi(e);
  if (const char* e = std::getenv("SFCDD_SCRATCH_MAX")) scratch_max = std::atoi(e);
  if (const char* e = std::getenv("SFCDD_WORKERS")) workers = std::atoi(e);
  if (const char* e = std::getenv("SFCDD_ROW_MAX")) row_max = std::min(128, std::max(1, std::atoi(e)));
  if (const char* e = std::getenv("SFCDD_COL_MAX")) col_max = std::min(32, std::max(1, std::atoi(e)));
  if (const char* e = std::getenv("SFCDD_SLACK_US")) slack_us = std::atof(e);
  if (const char* e = std::getenv("SFCDD_ASM_MAX")) asm_max = std::max(32, std::atoi(e));
  if (const char* e = std::getenv("SFCDD_ASM_RED")) asm_redundancy = std::atof(e);
  if (const char* e = std::getenv("SFCDD_XB_MIN")) xb_min_tasks = std::atoi(e);
  if (const char* e = std::getenv("SFCDD_DIRECT_ROWS")) direct_min_rows = std::atoi(e);
  if (const char* e = std::getenv("SFCDD_DIRECT_COLS")) direct_min_cols = std::atoi(e);
  if (const char* e = std::getenv("SFCDD_SPLIT_MIN")) split_min_factors = std::atoi(e);
  if (const char* e = std::getenv("SFCDD_MROW_ROWS")) mrow_rows = std::min(RING_CHUNK, std::max(0, std::atoi(e)));
  if (const char* e = std::getenv("SFCDD_MROW_MIN")) mrow_min_bytes = std::atoi(e);
  if (const char* e = std::getenv("SFCDD_PACK")) pack_siblings = std::atoi(e) != 0;
  if (const char* e = std::getenv("SFCDD_PACK_MAX")) pack_max = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("SFCDD_WPB")) wpb = std::atoi(e);
  if (const char* e = std::getenv("SFCDD_SLOT_MAX")) slot_max = std::max(-1, std::atoi(e));
  tuned = std::getenv("SFCDD_BLOB_MAX") || std::getenv("SFCDD_WPB");
}

void choose_blob_shape(const std::vector<const HostFactor*>& factors, PlanOptions& opt) {
  if (opt.tuned) return;
  double big = 0.0, tot = 0.0;
  for (const HostFactor* F : factors)
    for (const Supernode& S : F->sn) {
      const double v = (double)S.s * (S.s + S.m) - 0.5 * (double)S.s * (S.s - 1);
      tot += v;
      if (8.0 * v > opt.blob_max) big += v;  // cannot sit in a FRAG blob
    }
  if (std::getenv("SFCDD_PLAN_DEBUG"))
    std::fprintf(stderr, "[plan] values in supernodes above one blob: %.1f%%\n", tot > 0.0 ? 100.0 * big / tot : 0.0);
  // measured with the shared blob + scratch slot budget (profiles/r02/s5): C2 34 % -> 8 KB / 4 workers wins by
  // 7 %, C4 47 % -> by 5 %; C3 79 % needs 16 KB (a row of its widest BLOB supernode does not fit 8 KB)
  if (tot > 0.0 && big > 0.60 * tot) {
    opt.blob_max = 16 * 1024;
    opt.wpb = 2;
  }
  // one budget for blob + scratch (the scratch follows the task's own blob):
  // the largest slot that keeps 5 CTAs per SM resident (228 KB of shared
  // memory, 1 KB reserved and < 256 B static per CTA)
  if (opt.slot_max == 0) opt.slot_max = (int32_t)(((233472 / 5 - 1024 - 256) / opt.wpb) / 128 * 128);
}

void place_values(const ValDesc& d, const double* M, uint8_t* buf) {
  double* out = reinterpret_cast<double*>(buf + d.dst);
  switch (d.kind) {
    case VD_COPY:
      std::memcpy(out, M, 8 * (size_t)d.len);
      break;
    case VD_ROW:  // out[k R + i] = M[r0 + i, k]
      for (int32_t k = 0; k < d.len; ++k) {
        const double* col = M + packed_col_off(d.s, d.m, k);
        const int32_t nr = d.rows > 0 ? d.rows : d.w;
        for (int32_t i = std::max(0, k - d.p0); i < nr; ++i) out[(int64_t)k * d.w + i] = col[d.p0 + i - k];
      }
      break;
    case VD_COL:  // out[r c + j] = M[k0 + r, k0 + j]
      for (int32_t j = 0; j < d.w; ++j) {
        const double* col = M + packed_col_off(d.s, d.m, d.p0 + j);
        for (int32_t r = j; r < d.len; ++r) out[(int64_t)r * d.w + j] = col[r - j];
      }
      break;
    default:
      throw Error(SFCDD_EINTERNAL, "unknown value descriptor");
  }
}

DevicePlan build_plan(const std::vector<const HostFactor*>& factors, const std::vector<int64_t>& gstart,
                      const std::vector<int64_t>& gmod, const PlanOptions& opt_in) {
  PlanOptions opt = opt_in;
  {
    // DIRECT blocks only where the plan needs them: a supernode so wide that
    // not even one row / one column of its dense block fits a blob (BASELINE
    // C5: s ~ 2300).  Such plans stream every wide supernode; the others keep
    // the smaller kernel without the streaming path.
    bool need = false;
    for (const HostFactor* F : factors)
      for (const Supernode& S : F->sn)
        need = need || blob_size(RW_WORDS, (int64_t)S.s) > opt.blob_max ||
               blob_size(CL_WORDS + 1, (int64_t)S.s + S.m) > opt.blob_max;
    if (opt.direct_min_rows < 0) opt.direct_min_rows = need ? 8 : 0;
    if (opt.direct_min_cols < 0) opt.direct_min_cols = need ? 4 : 0;
  }
  SFCDD_REQUIRE(opt.scratch_max < 65536 && opt.big_scratch_max < 65536, SFCDD_EINTERNAL,
                "scratch positions must fit 16 bits");
  SFCDD_REQUIRE(opt.blob_max >= 2048 && opt.blob_max % 16 == 0, SFCDD_EVALUE, "blob_max must be >= 2048, 16-aligned");
  SFCDD_REQUIRE(opt.wpb == 2 || opt.wpb == 4 || opt.wpb == 8, SFCDD_EVALUE, "SFCDD_WPB must be 2, 4 or 8");
  DevicePlan P;
  P.blob_max = opt.blob_max;
  // Slot budget (opt.slot_max > 0): a task's scratch starts right after its
  // own blob (dag_solve.cu), so blob and scratch share one budget -- a task
  // with little scratch may carry a blob larger than blob_max.  Otherwise the
  // two areas have separate budgets (explicit blob_max / scratch_max).
  const bool slot_budget = opt.slot_max > 0;
  auto fits_frag = [&](int64_t bytes, int64_t scratch) {
    if (!slot_budget) return bytes <= opt.blob_max && scratch <= opt.scratch_max;
    return (bytes + 127) / 128 * 128 + 8 * scratch <= opt.slot_max && scratch < 65536;
  };
  auto blob_cap = [&](int64_t scratch) -> int64_t {  // largest blob next to `scratch` doubles
    if (!slot_budget) return opt.blob_max;
    // (a task whose scratch leaves less than half a blob falls back to the
    // separate budgets: the slot then grows to blob_max + its scratch, as
    // without the slot budget -- few-subdomain plans with wide separators,
    // whose COL tasks gather a whole front column into the scratch)
    const int64_t room = (opt.slot_max - 8 * scratch) / 128 * 128;
    return room >= opt.blob_max / 2 ? room : opt.blob_max;
  };
  P.wpb = opt.wpb;
  std::vector<Group> groups;
  std::vector<std::vector<int32_t>> group_of(factors.size());
  std::vector<std::vector<int32_t>> upd_slot(factors.size());
  int64_t xy_off = 0;

  double pt_[4] = {0, 0, 0, 0};
  auto pt_t0 = std::chrono::steady_clock::now();
  auto ptime = [&]() { auto t = std::chrono::steady_clock::now(); double d = std::chrono::duration<double>(t - pt_t0).count(); pt_t0 = t; return d; };
  // ---- 1. groups: greedy bottom-up clustering of small supernodes
  for (size_t fi = 0; fi < factors.size(); ++fi) {
    const HostFactor& F = *factors[fi];
    P.factors.push_back(FactorDev{gstart[fi], gmod[fi], xy_off, F.n});
    xy_off += F.n;
    P.num_supernodes += F.sn.size();
    P.stored += F.stored;
    P.nnz_l += F.nnz_l;
    const int64_t ns = F.sn.size();
    auto child_m = [&](int64_t k) {
      int64_t v = 0;
      for (int32_t q = F.child_ptr[k]; q < F.child_ptr[k + 1]; ++q) v += F.sn[F.child_list[q]].m;
      return v;
    };
    std::vector<Cluster> cl(ns);
    std::vector<char> open(ns, 0);
    std::vector<std::vector<int32_t>> members(ns);
    group_of[fi].assign(ns, -1);
    auto frag_bytes = [&](const Cluster& c, int64_t m_top) {
      return blob_size(H_WORDS + 2 + FRAG_PAD + c.meta_ints + L_WORDS * c.height + m_top + c.ext_u, c.vals);
    };
    auto frag_scratch = [&](const Cluster& c, int64_t m_top) { return c.frontal + m_top + c.ext_u; };
    auto close_roots = [&](const std::vector<int32_t>& roots, bool big) {
      Group g;
      g.factor = (int32_t)fi;
      for (int32_t r : roots) {
        g.sns.insert(g.sns.end(), members[r].begin(), members[r].end());
        members[r].clear();
        open[r] = 0;
      }
      std::sort(g.sns.begin(), g.sns.end());
      g.tops = roots;
      std::sort(g.tops.begin(), g.tops.end());
      g.top = g.tops[0];
      g.big = big;
      for (int32_t k : g.sns) group_of[fi][k] = (int32_t)groups.size();
      groups.push_back(std::move(g));
    };
    auto close = [&](int32_t root, bool big) { close_roots({root}, big); };
    // Sibling packing: the closed subtrees below one parent supernode (3-D
    // subdomains: dozens of tiny leaf subtrees hang off every wide front) share
    // fragments -- first-fit decreasing into bins that respect the blob and
    // scratch budgets (upper bounds: nothing is shared between the subtrees)
    auto pack_siblings = [&](std::vector<int32_t>& roots) {
      if (roots.empty()) return;
      if (!opt.pack_siblings || roots.size() == 1) {
        for (int32_t r : roots) close(r, false);
        roots.clear();
        return;
      }
      struct Bin {
        int64_t ints = 0, vals = 0, scratch = 0;
        std::vector<int32_t> roots;
      };
      auto r_ints = [&](int32_t r) {  // (one level table per root: an upper bound, the levels are shared)
        return cl[r].meta_ints + L_WORDS * cl[r].height + F.sn[r].m + cl[r].ext_u + 2;
      };
      auto r_scr = [&](int32_t r) { return cl[r].frontal + F.sn[r].m + cl[r].ext_u; };
      std::stable_sort(roots.begin(), roots.end(), [&](int32_t a, int32_t b) {
        return 4 * r_ints(a) + 8 * cl[a].vals > 4 * r_ints(b) + 8 * cl[b].vals;
      });
      std::vector<Bin> bins;
      for (int32_t r : roots) {
        Bin* dst = nullptr;
        for (Bin& b : bins)
          if (fits_frag(blob_size(H_WORDS + 2 + FRAG_PAD + b.ints + r_ints(r), b.vals + cl[r].vals),
                        b.scratch + r_scr(r)) &&
              (int32_t)b.roots.size() < opt.pack_max) {
            dst = &b;
            break;
          }
        if (!dst) {
          bins.emplace_back();
          dst = &bins.back();
        }
        dst->ints += r_ints(r);
        dst->vals += cl[r].vals;
        dst->scratch += r_scr(r);
        dst->roots.push_back(r);
      }
      for (Bin& b : bins) close_roots(b.roots, false);
      roots.clear();
    };
    for (int64_t k = 0; k < ns; ++k) {
      const Supernode& S = F.sn[k];
      Cluster c;
      c.nsn = 1;
      // record, cols + colpos, gather pairs, runs (distinct front positions
      // the children touch), v_B pairs, forward + backward items (packed items
      // are shared between supernodes: at most one each)
      c.meta_ints = R_WORDS + 2 * S.s + child_m(k) + std::min<int64_t>(S.s + S.m, child_m(k)) + S.m +
                    2 * ((S.s + S.m + 31) / 32 + (S.s + 31) / 32);
      c.vals = packed_size(S.s, S.m);
      c.frontal = 2 * S.s + S.m;
      c.ext_u = child_m(k);
      const bool big = S.s > SMALL_MAX_S || !fits_frag(frag_bytes(c, S.m), frag_scratch(c, S.m));
      std::vector<int32_t> shut;  // children closed below k
      if (big) {
        for (int32_t q = F.child_ptr[k]; q < F.child_ptr[k + 1]; ++q)
          if (open[F.child_list[q]]) shut.push_back(F.child_list[q]);
        pack_siblings(shut);
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
        t.height = std::max(t.height, d.height + 1);
        if (fits_frag(frag_bytes(t, S.m), frag_scratch(t, S.m))) {
          c = t;
          auto& mc = members[ch];
          members[k].insert(members[k].end(), mc.begin(), mc.end());
          mc.clear();
          open[ch] = 0;
        } else {
          shut.push_back(ch);
        }
      }
      pack_siblings(shut);
      cl[k] = c;
      open[k] = 1;
    }
    for (int64_t k = 0; k < ns; ++k)
      if (open[k]) close((int32_t)k, false);
    // update slots: every supernode whose parent lives in another group
    upd_slot[fi].assign(ns, -1);
    for (int64_t k = 0; k < ns; ++k) {
      const int32_t p = F.sn[k].parent;
      if (p >= 0 && group_of[fi][p] != group_of[fi][k]) {
        upd_slot[fi][k] = (int32_t)P.upd_doubles;
        P.upd_doubles += F.sn[k].m;
      }
    }
  }
  P.xy_doubles = xy_off;
  const int32_t G = (int32_t)groups.size();
  P.ngroups = G;
  for (int32_t g = 0; g < G; ++g) {
    Group& gr = groups[g];
    const HostFactor& F = *factors[gr.factor];
    const int32_t p = F.sn[gr.top].parent;
    gr.parent = p < 0 ? -1 : group_of[gr.factor][p];
    if (gr.parent >= 0) groups[gr.parent].kids.push_back(g);
    if (gr.big) {
      // update-buffer slots of a BIG group, allocated up front so that the
      // blob emission below can run per factor in parallel: y_J (s), the
      // assembled front [f_J ; f_B] (s + m, used in ASM mode) and -x_B (m,
      // used in XB mode)
      // (16-byte aligned, -x_B right after y_J: a COL task's whole input
      // v = [y_J[k0:s) ; -x_B] is ONE contiguous range it bulk-copies, and an
      // ROW task bulk-copies its front pieces; dag_solve.cu run_row / run_col)
      const Supernode& J = F.sn[gr.top];
      P.upd_doubles += P.upd_doubles & 1;
      gr.y_off = P.upd_doubles;
      P.upd_doubles += J.s;
      gr.xb_off = P.upd_doubles;
      P.upd_doubles += J.m;
      P.upd_doubles += P.upd_doubles & 1;
      gr.f_off = P.upd_doubles;
      P.upd_doubles += J.s + J.m;
      ++P.nbig;
    } else {
      ++P.nfrag;
    }
  }
  for (int32_t g = 0; g < G; ++g)  // children have smaller ids than parents
    if (groups[g].parent >= 0)
      groups[groups[g].parent].height = std::max(groups[groups[g].parent].height, groups[g].height + 1);

  pt_[0] = ptime();
  // ---- 2. blobs + tasks (unordered), emitted per factor in parallel into
  // factor-local buffers (offsets relative to the factor), then merged in
  // factor order (deterministic for any thread count)
  std::vector<TaskDev> tl;
  std::vector<double> tw;  // task weight (us, rough model used for the queue order)
  std::vector<int32_t> gbegin(factors.size() + 1, G);
  for (int32_t g = G - 1; g >= 0; --g) gbegin[groups[g].factor] = g;
  for (int64_t fi = (int64_t)factors.size() - 1; fi >= 0; --fi)
    if (gbegin[fi] == G) gbegin[fi] = gbegin[fi + 1];
  const bool defer = opt.defer_values;
  std::vector<FactorEmit> emits(factors.size());
  if (!defer)
    for (const HostFactor* F : factors)
      SFCDD_REQUIRE(F->val.size() == (size_t)F->stored, SFCDD_EINTERNAL, "plan without values needs defer_values");
  auto emit_factor = [&](int64_t fi_) {
  const size_t fi = (size_t)fi_;
  FactorEmit& E = emits[fi];
  E.defer = defer;
  E.factor = (int32_t)fi;
  std::vector<int32_t> ints;
  std::vector<int32_t> loc;
  std::vector<int32_t> col2sn_f;
  {
    const HostFactor& F = *factors[fi];
    col2sn_f.assign(F.n, -1);
    for (size_t k = 0; k < F.sn.size(); ++k)
      for (int32_t t = 0; t < F.sn[k].s; ++t) col2sn_f[F.sn[k].col0 + t] = (int32_t)k;
  }
  auto add_task = [&](int32_t g, int32_t kind, int64_t off, int32_t bytes, int64_t nvals, double w) {
    TaskDev T{};
    T.blob_off = off;
    T.copy_bytes = bytes;
    T.kind = kind;
    T.factor = groups[g].factor;
    T.group = g;
    T.values = (int32_t)nvals;
    E.tasks.push_back(T);
    E.tw.push_back(w);
  };
  for (int32_t g = gbegin[fi]; g < gbegin[fi + 1]; ++g) {
    const Group& gr = groups[g];
    const HostFactor& F = *factors[gr.factor];
    const Supernode& Top = F.sn[gr.top];
    if (gr.big) {
      // ---------------------------------------------------------- BIG
      const Supernode& S = Top;
      const int32_t s = S.s, m = S.m;
      // child update indices summed into each front position (fixed order:
      // children, then rows)
      std::vector<std::vector<int32_t>> contrib(s + m);
      for (int32_t q = F.child_ptr[gr.top]; q < F.child_ptr[gr.top + 1]; ++q) {
        const int32_t c = F.child_list[q];
        const Supernode& K = F.sn[c];
        SFCDD_REQUIRE(upd_slot[gr.factor][c] >= 0, SFCDD_EINTERNAL, "big child without update slot");
        for (int32_t a = 0; a < K.m; ++a) contrib[F.rel[K.rel_off + a]].push_back(upd_slot[gr.factor][c] + a);
      }
      // forward row blocks that never straddle s (rows [0, s): y rows; rows
      // [s, s+m): update rows).  BLOB blocks: as many rows as fit the blob
      // next to the metadata -- values and metadata arrive in ONE bulk copy,
      // the lowest-latency form for the many small dense blocks.  A supernode
      // too wide for that (fewer than direct_min_rows rows per blob at full
      // width) is cut into balanced blocks of <= row_max rows whose values
      // stay in HBM and are streamed into registers (DIRECT; dag_solve.cu).
      auto row_nnz = [&](int32_t r0, int32_t C, int32_t NB) {
        int64_t nnz = 0;
        for (int32_t q = 0; q < C + NB; ++q) nnz += (int64_t)contrib[q < C ? q : r0 + (q - C)].size();
        return nnz;
      };
      auto balanced = [&](int32_t lo, int32_t hi, int32_t wmax, std::vector<std::pair<int32_t, int32_t>>& out) {
        const int32_t n = hi - lo;
        if (n <= 0) return;
        const int32_t nt = (n + wmax - 1) / wmax, w = (n + nt - 1) / nt;
        for (int32_t r0 = lo; r0 < hi; r0 += w) out.emplace_back(r0, std::min(w, hi - r0));
      };
      const bool split_ok = (int64_t)factors.size() >= opt.split_min_factors;
      const bool direct_rows =
          (opt.blob_max - align16(4 * (int64_t)RW_WORDS)) / (8 * (int64_t)s) < opt.direct_min_rows;
      auto row_split = [&](bool inl, std::vector<std::pair<int32_t, int32_t>>& out) {
        out.clear();
        if (direct_rows) {
          balanced(0, s, std::min(opt.row_max, 32), out);  // DIRECT: one lane per row
          balanced(s, s + m, std::min(opt.row_max, 32), out);
          if (inl)  // the task's own assembly CSR must fit the blob, its front piece the scratch
            for (const auto& rb : out) {
              const int32_t r0 = rb.first, R = rb.second;
              const int32_t C = r0 < s ? r0 + R : s, NB = r0 < s ? 0 : R;
              if (blob_size(RW_WORDS + C + (C + NB + 1) + row_nnz(r0, C, NB), 0) > blob_cap(C + NB + 6) ||
                  C + NB + 2 > opt.big_scratch_max)
                return false;
            }
          return true;
        }
        // (any row count runs: lanes = rows, blocks of > 32 rows in passes; the
        // finer steps fill the blob where a power of two would leave it half empty)
        static const int32_t cand[] = {128, 112, 96, 80, 64, 56, 48, 40, 32, 28, 24, 20, 16, 14, 12, 10, 8, 6, 4, 3, 2, 1};
        for (int32_t r0 = 0; r0 < s + m;) {
          const int32_t lim = r0 < s ? s : s + m;
          int32_t R = 0;
          for (int32_t cnd : cand) {
            if (cnd > opt.row_max && cnd > 1) continue;
            const int32_t Re = std::min(cnd, lim - r0);
            const int32_t C = r0 < s ? r0 + Re : s, NB = r0 < s ? 0 : Re;
            const int64_t meta = inl ? RW_WORDS + C + (C + NB + 1) + row_nnz(r0, C, NB) : RW_WORDS;
            if (blob_size(meta, (int64_t)Re * C) <= blob_cap(C + NB + 6) && C + NB + 2 <= opt.big_scratch_max) {
              R = Re;
              break;
            }
          }
          // not even one row next to its scratch: the separate budgets (the slot grows past slot_max)
          if (R == 0 && slot_budget) {
            const int32_t C = r0 < s ? r0 + 1 : s, NB = r0 < s ? 0 : 1;
            const int64_t meta = inl ? RW_WORDS + C + (C + NB + 1) + row_nnz(r0, C, NB) : RW_WORDS;
            if (blob_size(meta, (int64_t)C) <= opt.blob_max && C + NB + 2 <= opt.big_scratch_max) R = 1;
          }
          if (R == 0) return false;
          out.emplace_back(r0, R);
          r0 += R;
        }
        return true;
      };
      std::vector<std::pair<int32_t, int32_t>> split_a, split_i;
      SFCDD_REQUIRE(row_split(false, split_a), SFCDD_EINTERNAL,
                    "big supernode row does not fit a task blob (s = " + std::to_string(s) + ")");
      double gathered = 0.0;
      for (const auto& rb : split_a) gathered += rb.first < s ? rb.first + rb.second : s + rb.second;
      // three ways to assemble the front for the ROW tasks: ASM tasks (once per
      // supernode, one extra dependency hop; the ROW tasks then read f through
      // the vector ring), a global assembly record shared by the ROW tasks
      // (the metadata would crowd the values out of the blobs, or not fit), or
      // inline metadata in every ROW blob
      int64_t fj_nnz = 0;
      for (int32_t q = 0; q < s; ++q) fj_nnz += (int64_t)contrib[q].size();
      const bool huge = !direct_rows && 4 * (RW_WORDS + 2 * s + 1 + fj_nnz) > opt.blob_max / 2;
      const bool scratch_ok = s + opt.row_max + 2 <= opt.big_scratch_max;  // inline / record modes hold f_J in the slot
      const bool use_asm =
          !scratch_ok || (split_ok && (direct_rows || gathered >= opt.asm_redundancy * (s + m)));
      const bool global_asm = !use_asm && (huge || !row_split(true, split_i));
      const auto& split = (use_asm || global_asm) ? split_a : split_i;
      int64_t asm16 = -1;
      if (global_asm) {
        ints.assign({s, m});
        for (int32_t c = 0; c < s; ++c) ints.push_back(F.perm[S.col0 + c]);
        int32_t nnz = 0;
        for (int32_t p = 0; p <= s + m; ++p) {
          ints.push_back(nnz);
          if (p < s + m) nnz += (int32_t)contrib[p].size();
        }
        for (int32_t p = 0; p < s + m; ++p) ints.insert(ints.end(), contrib[p].begin(), contrib[p].end());
        const int64_t asm_off = E.raw(ints);  // factor-local; rebased (asm16 patches) at the merge
        asm16 = asm_off / 16;
      }
      if (use_asm) {  // the assembled front [f_J ; f_B] at gr.f_off
        // forward assembly: f = [f_J ; f_B] in chunks of front positions
        for (int32_t q0 = 0; q0 < s + m;) {
          int32_t nq = 0;
          int64_t nnz = 0, ncol = 0;
          while (q0 + nq < s + m && nq < opt.asm_max) {
            const int32_t q = q0 + nq;
            const int64_t nnz2 = nnz + (int64_t)contrib[q].size(), ncol2 = ncol + (q < s);
            if (blob_size(AS_WORDS + ncol2 + (nq + 2) + nnz2, 0) > opt.blob_max) break;
            nnz = nnz2;
            ncol = ncol2;
            ++nq;
          }
          SFCDD_REQUIRE(nq > 0, SFCDD_EINTERNAL, "assembly position does not fit a task blob");
          ints.assign(AS_WORDS, 0);
          ints[AS_S] = s;
          ints[AS_Q0] = q0;
          ints[AS_NQ] = nq;
          ints[AS_FOFF] = (int32_t)gr.f_off;
          ints[AS_COLS] = (int32_t)ints.size();
          for (int32_t q = q0; q < q0 + nq && q < s; ++q) ints.push_back(F.perm[S.col0 + q]);
          ints[AS_PTR] = (int32_t)ints.size();
          int32_t e = 0;
          for (int32_t q = q0; q <= q0 + nq; ++q) {
            ints.push_back(e);
            if (q < q0 + nq) e += (int32_t)contrib[q].size();
          }
          ints[AS_SRC] = (int32_t)ints.size();
          for (int32_t q = q0; q < q0 + nq; ++q) ints.insert(ints.end(), contrib[q].begin(), contrib[q].end());
          while (ints.size() % 4) ints.push_back(0);
          int32_t bytes = 0;
          const int64_t off = E.emit(ints, -1, 0, nullptr, bytes);  // metadata only
          ints.clear();
          E.need_slot(bytes, 0);
          add_task(g, TK_ASM_FWD, off, bytes, 0, 1.2 + 0.004 * (nq + (double)e));
          q0 += nq;
        }
      }
      // MROW: in ASM mode the update rows of a narrow supernode become a few
      // long DIRECT tasks (plan.h) instead of m / R row blocks
      const bool mrow = use_asm && opt.mrow_rows > 0 && opt.direct_min_rows > 0 && m > 0 && s <= RING_CHUNK &&
                        8 * (int64_t)m * s >= opt.mrow_min_bytes;
      if (mrow) {
        std::vector<std::pair<int32_t, int32_t>> tasks_rows;
        balanced(s, s + m, opt.mrow_rows, tasks_rows);
        for (const auto& tr : tasks_rows) {
          const int32_t r0 = tr.first, rows = tr.second;
          const int32_t nb = (rows + 31) / 32, Rb = (rows + nb - 1) / nb;
          ints.assign(RW_WORDS, 0);
          ints[RW_S] = s;
          ints[RW_R] = Rb;
          ints[RW_C] = s;
          ints[RW_R0] = r0;
          ints[RW_NB] = rows;
          ints[RW_YOFF] = (int32_t)gr.y_off;
          ints[RW_UOFF] = upd_slot[gr.factor][gr.top];
          ints[RW_FOFF] = (int32_t)gr.f_off;
          ints[RW_ASM16] = 0;
          ints[RW_ASM_HI] = -1;
          ints[RW_SCRATCH] = 2 * RING_STRIDE;
          ints[RW_INBLOB] = 0;
          ints[RW_NBLK] = nb;
          std::vector<ValDesc> vds;
          for (int32_t b = 0; b < nb; ++b) {
            ValDesc vd{};
            vd.dst = 8 * (int64_t)b * Rb * s;
            vd.src = S.val_off;
            vd.kind = VD_ROW;
            vd.s = s;
            vd.m = m;
            vd.p0 = r0 + b * Rb;
            vd.w = Rb;
            vd.len = s;
            vd.rows = std::min(Rb, rows - b * Rb);
            vds.push_back(vd);
          }
          int32_t bytes = 0;
          const int64_t off = E.emit_descs(ints, RW_VAL_OFF, (int64_t)nb * Rb * s, vds.data(), vds.size(), bytes, &F, -1, true);
          E.has_direct = true;
          E.has_mrow = true;
          E.max_scratch = std::max<int32_t>(E.max_scratch, 2 * RING_STRIDE);
          E.need_slot(bytes, 2 * RING_STRIDE);
          add_task(g, TK_ROW_FWD, off, bytes, (int64_t)rows * s, 1.8 + 0.0004 * rows * s);
        }
      }
      for (const auto& rb : split) {
        const int32_t r0 = rb.first, R = rb.second;
        if (mrow && r0 >= s) continue;  // covered by the MROW tasks
        const int32_t C = r0 < s ? r0 + R : s;
        const int32_t NB = r0 < s ? 0 : R;
        ints.assign(RW_WORDS, 0);
        ints[RW_S] = s;
        ints[RW_R] = R;
        ints[RW_C] = C;
        ints[RW_R0] = r0;
        ints[RW_NB] = NB;
        ints[RW_YOFF] = (int32_t)gr.y_off;
        ints[RW_UOFF] = upd_slot[gr.factor][gr.top];
        ints[RW_FOFF] = use_asm ? (int32_t)gr.f_off : -1;
        ints[RW_ASM16] = (int32_t)(uint32_t)(asm16 & 0xffffffffLL);
        ints[RW_ASM_HI] = asm16 >= 0 ? (int32_t)(asm16 >> 32) : -1;
        if (!use_asm && !global_asm) {
          ints[RW_COLS] = (int32_t)ints.size();
          for (int32_t c = 0; c < C; ++c) ints.push_back(F.perm[S.col0 + c]);
          ints[RW_PTR] = (int32_t)ints.size();
          int32_t e = 0;
          for (int32_t q = 0; q <= C + NB; ++q) {
            ints.push_back(e);
            if (q < C + NB) e += (int32_t)contrib[q < C ? q : r0 + (q - C)].size();
          }
          ints[RW_SRC] = (int32_t)ints.size();
          for (int32_t q = 0; q < C + NB; ++q) {
            const auto& cl = contrib[q < C ? q : r0 + (q - C)];
            ints.insert(ints.end(), cl.begin(), cl.end());
          }
        }
        // scratch: the vector ring (ASM mode) or the task's own front piece
        const int32_t scr = direct_rows && use_asm ? 2 * RING_STRIDE : C + NB + 6;  // (+ padding of bulk-copied pieces)
        ints[RW_SCRATCH] = scr;
        ints[RW_INBLOB] = direct_rows ? 0 : 1;
        ints[RW_NBLK] = 1;
        // values: R x C column-major, (i, k) = M[r0 + i, k] for k <= r0 + i;
        // DIRECT blocks leave them in HBM (the task copies its metadata only)
        ValDesc vd{};
        vd.src = S.val_off;
        vd.kind = VD_ROW;
        vd.s = s;
        vd.m = m;
        vd.p0 = r0;
        vd.w = R;
        vd.len = C;
        const int32_t asm_word = asm16 >= 0 ? RW_ASM16 : -1;
        int32_t bytes = 0;
        const int64_t off = E.emit(ints, RW_VAL_OFF, (int64_t)R * C, &vd, bytes, F, asm_word, direct_rows);
        SFCDD_REQUIRE(bytes <= std::max<int64_t>(blob_cap(scr), opt.blob_max), SFCDD_EINTERNAL,
                      "ROW blob exceeds the slot (bytes " + std::to_string(bytes) + ", scratch " + std::to_string(scr) +
                          ", s " + std::to_string(s) + ", R " + std::to_string(R) + ", C " + std::to_string(C) +
                          (use_asm ? ", asm" : global_asm ? ", record" : ", inline") + (direct_rows ? ", direct)" : ", blob)"));
        E.need_slot(bytes, scr);
        E.has_direct = E.has_direct || direct_rows;
        E.max_scratch = std::max<int32_t>(E.max_scratch, scr);
        add_task(g, TK_ROW_FWD, off, bytes, (int64_t)R * C, (use_asm ? 1.8 : 2.36) + 0.0013 * R * C);
      }
      // backward column blocks, dense row-major L x c (L = s+m-k0): BLOB blocks
      // (as many columns as fit the blob) or, when fewer than direct_min_cols
      // columns of the full height would fit, DIRECT blocks of <= col_max
      // columns streamed from HBM.  -x_B is gathered once per supernode by XB
      // tasks where many COL tasks would repeat the gather (the COL tasks then
      // read v = [y_J[k0:s) ; -x_B] through the vector ring) or where the
      // inline row list / gathered v would not fit the slot
      const bool direct_cols =
          (opt.blob_max - align16(4 * (int64_t)(CL_WORDS + opt.col_max))) / (8 * (int64_t)(s + m)) < opt.direct_min_cols;
      auto col_width = [&](int32_t k0, bool inl) {
        const int32_t L = s + m - k0;
        int32_t c = std::min<int32_t>(opt.col_max, s - k0);
        while (c > 1 && blob_size(CL_WORDS + c + (inl ? m : 0), (int64_t)L * c) > blob_cap(L + 2)) --c;
        // (c == 1 may exceed the slot cap and still fit blob_max: the slot then grows past slot_max,
        // the separate-budget behaviour for a column whose gathered vector fills most of a slot)
        if (std::getenv("SFCDD_EVEN_COLS") && c > 1 && (c & 1) && k0 + c < s) --c;
        return c;
      };
      std::vector<std::pair<int32_t, int32_t>> csplit;
      bool ring_col, use_xb;
      if (direct_cols) {
        balanced(0, s, opt.col_max, csplit);
        const bool inline_fits =
            blob_size(CL_WORDS + opt.col_max + m, 0) <= blob_cap(s + m + 2) && s + m + 2 <= opt.big_scratch_max;
        ring_col = split_ok || !inline_fits;  // v is contiguous in upd: y_J then -x_B
        use_xb = m > 0 && ring_col;
      } else {
        int32_t ncol_tasks = 0;
        for (int32_t k0 = 0; k0 < s; k0 += col_width(k0, false)) ++ncol_tasks;
        // XB also when a column block with its inline row list cannot fit a blob
        const bool inline_fits =
            blob_size(CL_WORDS + 1 + m, (int64_t)(s + m)) <= blob_cap(s + m + 2) && s + m + 2 <= opt.big_scratch_max;
        use_xb = m > 0 && ((split_ok && ncol_tasks >= opt.xb_min_tasks) || !inline_fits);
        ring_col = use_xb || (m == 0 && !inline_fits);
        for (int32_t k0 = 0; k0 < s;) {
          const int32_t c = col_width(k0, !ring_col);
          csplit.emplace_back(k0, c);
          k0 += c;
        }
      }
      if (use_xb) {  // -x_B at gr.xb_off
        for (int32_t a0 = 0; a0 < m;) {
          int32_t na = std::min<int32_t>(m - a0, opt.asm_max);
          while (na > 1 && blob_size(XB_WORDS + na, 0) > opt.blob_max) --na;
          ints.assign(XB_WORDS, 0);
          ints[XB_A0] = a0;
          ints[XB_NA] = na;
          ints[XB_XOFF] = (int32_t)gr.xb_off;
          ints[XB_ROWS] = (int32_t)ints.size();
          for (int32_t a = a0; a < a0 + na; ++a) ints.push_back(F.perm[F.rows[S.rows_off + a]]);
          while (ints.size() % 4) ints.push_back(0);
          int32_t bytes = 0;
          const int64_t off = E.emit(ints, -1, 0, nullptr, bytes);  // metadata only
          ints.clear();
          E.need_slot(bytes, 0);
          add_task(g, TK_XB_BWD, off, bytes, 0, 1.2 + 0.003 * na);
          a0 += na;
        }
      }
      for (const auto& cb : csplit) {
        const int32_t k0 = cb.first, c = cb.second;
        const int32_t L = s + m - k0;
        ints.assign(CL_WORDS, 0);
        ints[CL_S] = s;
        ints[CL_M] = m;
        ints[CL_K0] = k0;
        ints[CL_C] = c;
        ints[CL_YOFF] = (int32_t)gr.y_off;
        ints[CL_XOFF] = ring_col ? (int32_t)gr.xb_off : -1;
        ints[CL_COLS] = (int32_t)ints.size();
        for (int32_t j = 0; j < c; ++j) ints.push_back(F.perm[S.col0 + k0 + j]);
        if (!ring_col) {
          ints[CL_ROWS] = (int32_t)ints.size();
          for (int32_t a = 0; a < m; ++a) ints.push_back(F.perm[F.rows[S.rows_off + a]]);
        }
        const int32_t scr = direct_cols && ring_col ? 2 * RING_STRIDE : L + 2;
        ints[CL_SCRATCH] = scr;
        ints[CL_INBLOB] = direct_cols ? 0 : 1;
        // values: L x c row-major, (r, j) = M[k0 + r, k0 + j] for j <= r (DIRECT: left in HBM)
        const int64_t nv = (int64_t)L * c - (int64_t)c * (c - 1) / 2;
        ValDesc vd{};
        vd.src = S.val_off;
        vd.kind = VD_COL;
        vd.s = s;
        vd.m = m;
        vd.p0 = k0;
        vd.w = c;
        vd.len = L;
        int32_t bytes = 0;
        const int64_t off = E.emit(ints, CL_VAL_OFF, (int64_t)L * c, &vd, bytes, F, -1, direct_cols);
        SFCDD_REQUIRE(bytes <= std::max<int64_t>(blob_cap(scr), opt.blob_max), SFCDD_EINTERNAL,
                      "big supernode column does not fit a task blob (s+m = " + std::to_string(s + m) + ")");
        E.need_slot(bytes, scr);
        E.has_direct = E.has_direct || direct_cols;
        E.max_scratch = std::max<int32_t>(E.max_scratch, scr);
        add_task(g, TK_COL_BWD, off, bytes, nv, (use_xb ? 1.8 : 2.24) + 0.0013 * nv);
      }
      continue;
    }
    // ------------------------------------------------------------ FRAG
    const int32_t nsn = (int32_t)gr.sns.size();
    ints.assign(H_WORDS, 0);
    std::vector<ValDesc> fvd;
    int64_t fvals = 0;
    ints[H_NSN] = nsn;
    loc.assign(F.sn.size(), -1);
    for (int32_t t = 0; t < nsn; ++t) loc[gr.sns[t]] = t;
    std::vector<int32_t> lev(nsn, 0);
    int32_t nlev = 0;
    for (int32_t t = 0; t < nsn; ++t) {
      const int32_t k = gr.sns[t];
      for (int32_t q = F.child_ptr[k]; q < F.child_ptr[k + 1]; ++q) {
        const int32_t c = F.child_list[q];
        if (loc[c] >= 0) lev[t] = std::max(lev[t], lev[loc[c]] + 1);
      }
      nlev = std::max(nlev, lev[t] + 1);
    }
    auto front = [&](int32_t t) { return F.sn[gr.sns[t]].s + F.sn[gr.sns[t]].m; };
    // level order (small fronts first within a level: better lane packing)
    std::vector<int32_t> ord(nsn);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) {
      if (lev[a] != lev[b]) return lev[a] < lev[b];
      return front(a) < front(b);
    });
    std::vector<int32_t> lid(nsn);  // postorder index -> level-order id
    for (int32_t i = 0; i < nsn; ++i) lid[ord[i]] = i;
    auto sn_of = [&](int32_t id) -> const Supernode& { return F.sn[gr.sns[ord[id]]]; };
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
    std::map<int32_t, int32_t> extx;  // row -> staging position (rows of the tops: one parent front)
    std::vector<int32_t> extx_rows;
    const int32_t extx_base = pos;
    for (int32_t tp : gr.tops) {
      const Supernode& T = F.sn[tp];
      for (int32_t a = 0; a < T.m; ++a) {
        const int32_t r = F.rows[T.rows_off + a];
        if (extx.emplace(r, pos).second) {
          extx_rows.push_back(r);
          ++pos;
        }
      }
    }
    std::map<int32_t, int32_t> extu_pos;  // external child -> staging position
    std::vector<int32_t> extu;            // global update index per staged double
    const int32_t extu_base = pos;
    for (int32_t i = 0; i < nsn; ++i) {
      const int32_t k = gr.sns[ord[i]];
      for (int32_t q = F.child_ptr[k]; q < F.child_ptr[k + 1]; ++q) {
        const int32_t c = F.child_list[q];
        if (loc[c] >= 0) continue;
        extu_pos[c] = pos;
        SFCDD_REQUIRE(upd_slot[gr.factor][c] >= 0, SFCDD_EINTERNAL, "external child without update slot");
        for (int32_t a = 0; a < F.sn[c].m; ++a) extu.push_back(upd_slot[gr.factor][c] + a);
        pos += F.sn[c].m;
      }
    }
    const int32_t scratch_used = pos;
    ints[H_NLEV] = nlev;
    ints[H_NTOP] = (int32_t)gr.tops.size();
    ints[H_TOPS] = (int32_t)ints.size();
    for (int32_t tp : gr.tops) {
      ints.push_back(lid[loc[tp]]);
      ints.push_back(upd_slot[gr.factor][tp]);
    }
    ints[H_COLS] = (int32_t)ints.size();
    for (int32_t i = 0; i < nsn; ++i)
      for (int32_t c = 0; c < sn_of(i).s; ++c) ints.push_back(F.perm[sn_of(i).col0 + c]);
    ints[H_NCOL] = (int32_t)ints.size() - ints[H_COLS];
    ints[H_COLPOS] = (int32_t)ints.size();
    for (int32_t i = 0; i < nsn; ++i)
      for (int32_t c = 0; c < sn_of(i).s; ++c) put_pair(ints, scr[i] + c, cpos[i] + c);
    ints[H_NEXTX] = (int32_t)extx_rows.size();
    ints[H_EXTX_BASE] = extx_base;
    ints[H_EXTX] = (int32_t)ints.size();
    for (int32_t r : extx_rows) ints.push_back(F.perm[r]);
    ints[H_NEXTU] = (int32_t)extu.size();
    ints[H_EXTU_BASE] = extu_base;
    ints[H_EXTU] = (int32_t)ints.size();
    ints.insert(ints.end(), extu.begin(), extu.end());
    while (ints.size() % 4) ints.push_back(0);  // int4 records
    ints[H_REC] = (int32_t)ints.size();
    ints.resize(ints.size() + (size_t)R_WORDS * nsn, 0);
    int64_t nvals = 0;
    for (int32_t i = 0; i < nsn; ++i) {
      const Supernode& S = sn_of(i);
      int32_t* R = &ints[ints[H_REC] + R_WORDS * i];
      SFCDD_REQUIRE(S.s < 4096 && S.m < 32768, SFCDD_EINTERNAL, "supernode too large for a FRAG record");
      R[R_SM] = S.s | (S.m << 16);
      R[R_VAL] = (int32_t)fvals;
      R[R_SCR] = scr[i];
      R[R_CPOS] = cpos[i];
      ValDesc vd{};
      vd.dst = 8 * fvals;  // within the value area (emit() rebases)
      vd.src = S.val_off;
      vd.kind = VD_COPY;
      vd.s = S.s;
      vd.m = S.m;
      vd.len = (int32_t)packed_size(S.s, S.m);
      fvd.push_back(vd);
      fvals += packed_size(S.s, S.m);
      nvals += packed_size(S.s, S.m);
    }
    // Backward items of one level.  Supernodes with s <= 32 are packed into
    // column-lane items: lanes = (supernode, column k, row phase) with 2^lp
    // phases per column (lp in bits 12-14 of the record's s|m word), each
    // lane summing every 2^lp-th row of column k, then a shuffle reduction
    // over the phases.  Lane order is DESCENDING record order (larger fronts,
    // hence more phases, first, so segment starts stay aligned to their phase
    // count); the item is {lo | cnt << 16, mask of segment start lanes (+ the
    // end lane)} over records [lo, lo + cnt).  Wider supernodes: blocks of up
    // to 32 columns, lanes = (column, row phase) (bwd_cols).
    auto emit_bwd_items = [&](int32_t* L, std::vector<int32_t>& its) {
      L[L_BI0] = (int32_t)its.size() / 2;
      int32_t j = L[L_REC1] - 1;
      while (j >= L[L_REC0]) {
        const Supernode& S = sn_of(j);
        if (S.s > 32) {
          for (int32_t k0 = 0; k0 < S.s; k0 += 32)
            its.insert(its.end(), {j, k0 | (std::min<int32_t>(32, S.s - k0) << 16)});
          --j;
          continue;
        }
        const int32_t hi = j;
        int32_t lo = j, lanes = 0;
        while (lo >= L[L_REC0] && sn_of(lo).s <= 32 && lanes + sn_of(lo).s <= 32 && hi - lo < 31) {
          lanes += sn_of(lo).s;
          --lo;
        }
        ++lo;
        const int32_t cnt = hi - lo + 1;
        std::vector<int32_t> lp(cnt, 0);
        std::vector<char> frozen(cnt, 0);
        auto layout = [&](uint32_t* mask_out) -> int32_t {
          int32_t off = 0;
          uint32_t mask = 0;
          for (int32_t q = 0; q < cnt; ++q) {
            const int32_t Pq = 1 << lp[q];
            off = (off + Pq - 1) / Pq * Pq;
            if (off >= 32) return 33;
            mask |= 1u << off;
            off += sn_of(hi - q).s * Pq;
          }
          if (off < 32) mask |= 1u << off;
          if (mask_out) *mask_out = mask;
          return off;
        };
        for (;;) {  // give more row phases to the longest columns while the lanes last
          int32_t best = -1;
          double bw = 0.0;
          for (int32_t q = 0; q < cnt; ++q) {
            const Supernode& T = sn_of(hi - q);
            const double w = (double)(T.s + T.m) / (1 << lp[q]);
            if (!frozen[q] && w > bw) {
              bw = w;
              best = q;
            }
          }
          if (best < 0 || bw <= 2.0) break;
          ++lp[best];
          if (lp[best] > 5 || layout(nullptr) > 32) {
            --lp[best];
            frozen[best] = 1;
          }
        }
        uint32_t mask = 0;
        SFCDD_REQUIRE(layout(&mask) <= 32, SFCDD_EINTERNAL, "backward item lane overflow");
        for (int32_t q = 0; q < cnt; ++q) ints[ints[H_REC] + R_WORDS * (hi - q) + R_SM] |= lp[q] << 12;
        its.insert(its.end(), {(int32_t)((uint32_t)lo | ((uint32_t)cnt << 16)), (int32_t)mask});
        j = lo - 1;
      }
      L[L_BI1] = (int32_t)its.size() / 2;
    };
    std::vector<int32_t> levtab((size_t)L_WORDS * nlev, 0), runs, gpairs, bpairs, items;
    std::vector<std::pair<int32_t, int32_t>> jp;
    int32_t i = 0;
    for (int32_t l = 0; l < nlev; ++l) {
      int32_t* L = &levtab[(size_t)L_WORDS * l];
      L[L_REC0] = i;
      while (i < nsn && lev[ord[i]] == l) ++i;
      L[L_REC1] = i;
      // forward gather runs
      L[L_RUN0] = (int32_t)runs.size();
      for (int32_t j = L[L_REC0]; j < L[L_REC1]; ++j) {
        const int32_t k = gr.sns[ord[j]];
        jp.clear();
        for (int32_t q = F.child_ptr[k]; q < F.child_ptr[k + 1]; ++q) {
          const int32_t c = F.child_list[q];
          const Supernode& K = F.sn[c];
          const int32_t src = loc[c] >= 0 ? scr[lid[loc[c]]] + K.s : extu_pos[c];
          for (int32_t a = 0; a < K.m; ++a) jp.emplace_back(scr[j] + F.rel[K.rel_off + a], src + a);
        }
        std::stable_sort(jp.begin(), jp.end(), [](const std::pair<int32_t, int32_t>& x,
                                                  const std::pair<int32_t, int32_t>& y) { return x.first < y.first; });
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
          const int32_t owner = col2sn_f[r];
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
      // warp items: forward (row blocks / packed) then backward (columns / packed)
      for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) {
          emit_bwd_items(L, items);
          continue;
        }
        L[pass == 0 ? L_FI0 : L_BI0] = (int32_t)items.size() / 2;
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
            const uint32_t tiny = smax <= 4 ? 0x80000000u : 0u;
            items.insert(items.end(), {(int32_t)((uint32_t)(j | ((j1 - j) << 16)) | tiny), (int32_t)mask});
            j = j1;
          } else if (pass == 0) {
            for (int32_t b = 0; b < (S.s + S.m + 31) / 32; ++b) items.insert(items.end(), {j, b});
            ++j;
          } else {
            // backward: blocks of up to 32 columns; lanes = (column, row-phase)
            for (int32_t k0 = 0; k0 < S.s; k0 += 32)
              items.insert(items.end(), {j, k0 | (std::min<int32_t>(32, S.s - k0) << 16)});
            ++j;
          }
        }
        L[pass == 0 ? L_FI1 : L_BI1] = (int32_t)items.size() / 2;
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
    ints[H_SCRATCH] = scratch_used;
    ints[H_ZERO] = nsn > 0 ? cpos[0] : 0;  // frontal slots [0, cpos[0])
    SFCDD_REQUIRE(slot_budget || scratch_used <= opt.scratch_max, SFCDD_EINTERNAL, "fragment scratch exceeds budget");
    int32_t bytes = 0;
    const int64_t off = E.emit_frag(ints, H_VAL_OFF, fvals, fvd, bytes, F);
    SFCDD_REQUIRE(fits_frag(bytes, scratch_used), SFCDD_EINTERNAL, "fragment blob exceeds the slot budget");
    E.need_slot(bytes, scratch_used);
    E.max_scratch = std::max(E.max_scratch, scratch_used);
    // task time model (us), fitted to traced C2 launches (tools/trace_dag.py)
    add_task(g, TK_FRAG_FWD, off, bytes, nvals, 2.13 + 0.0041 * nvals + 0.57 * nlev);
    add_task(g, TK_FRAG_BWD, off, bytes, nvals, 1.11 + 0.0021 * nvals + 0.68 * nlev);
  }

  };  // emit_factor
  parallel_range((int64_t)factors.size(), opt.threads, emit_factor);
  // merge in factor order: rebase blob offsets, value descriptors and the
  // global assembly-record references (asm16)
  P.deferred = defer;
  {
    int64_t tot = 0, meta_tot = 0;
    for (const FactorEmit& E : emits) {
      tot += E.size;
      meta_tot += (int64_t)E.image.size();
    }
    P.blob_bytes = tot;
    P.blobs.reserve(defer ? meta_tot : tot);
  }
  int64_t cursor = 0;
  for (FactorEmit& E : emits) {
    const int64_t dbase = cursor;
    for (const auto& pa : E.asm_patches) {  // (lo, hi) int32 words at image byte offset pa
      uint32_t lo;
      int32_t hi;
      std::memcpy(&lo, E.image.data() + pa, 4);
      std::memcpy(&hi, E.image.data() + pa + 4, 4);
      const int64_t v = ((int64_t)hi << 32 | lo) + dbase / 16;
      lo = (uint32_t)(v & 0xffffffffLL);
      hi = (int32_t)(v >> 32);
      std::memcpy(E.image.data() + pa, &lo, 4);
      std::memcpy(E.image.data() + pa + 4, &hi, 4);
    }
    if (defer) {
      const int64_t hbase = (int64_t)P.blobs.size();
      for (MetaSeg sg : E.segs) {
        sg.dev_off += dbase;
        sg.host_off += hbase;
        P.segs.push_back(sg);
      }
    }
    P.blobs.insert(P.blobs.end(), E.image.begin(), E.image.end());
    E.image.clear();
    E.image.shrink_to_fit();
    for (ValDesc vd : E.vdesc) {
      vd.dst += dbase;
      P.vdesc.push_back(vd);
    }
    E.vdesc.clear();
    E.vdesc.shrink_to_fit();
    for (size_t t = 0; t < E.tasks.size(); ++t) {
      TaskDev T = E.tasks[t];
      T.blob_off += dbase;
      tl.push_back(T);
      tw.push_back(E.tw[t]);
      Group& G_ = groups[T.group];
      std::vector<int32_t>& lst = T.kind == TK_ASM_FWD ? G_.atask
                                  : T.kind == TK_XB_BWD ? G_.xtask
                                  : (T.kind == TK_FRAG_FWD || T.kind == TK_ROW_FWD) ? G_.ftask
                                                                                      : G_.btask;
      lst.push_back((int32_t)tl.size() - 1);
    }
    cursor += E.size;
    P.max_scratch = std::max(P.max_scratch, E.max_scratch);
    P.slot_need = std::max(P.slot_need, E.max_slot);
    P.max_copy = std::max(P.max_copy, E.max_copy);
    P.has_direct = P.has_direct || E.has_direct;
    P.has_mrow = P.has_mrow || E.has_mrow;
  }
  SFCDD_REQUIRE(P.upd_doubles < (int64_t(1) << 31), SFCDD_EINTERNAL, "update buffer too large");

  pt_[1] = ptime();
  // ---- 3. dependencies (counters: plan.h)
  auto FIN = [&](int32_t g) { return 1 + g; };
  auto BDONE = [&](int32_t g) { return 1 + G + g; };
  auto RDONE = [&](int32_t g) { return 1 + 2 * G + g; };
  auto ADONE = [&](int32_t g) { return 1 + 3 * G + g; };
  auto XDONE = [&](int32_t g) { return 1 + 4 * G + g; };
  for (int32_t g = 0; g < G; ++g) {
    const Group& gr = groups[g];
    int32_t kids_f = 0;
    for (int32_t c : gr.kids) kids_f += (int32_t)groups[c].ftask.size();
    // children's forward -> (BIG: assembly ->) forward rows
    for (int32_t t : gr.atask) {
      tl[t].wait_idx = kids_f > 0 ? FIN(g) : -1;
      tl[t].wait_target = kids_f;
      tl[t].signal_idx = ADONE(g);
    }
    for (int32_t t : gr.ftask) {
      if (!gr.atask.empty()) {
        tl[t].wait_idx = ADONE(g);
        tl[t].wait_target = (int32_t)gr.atask.size();
      } else {
        tl[t].wait_idx = kids_f > 0 ? FIN(g) : -1;
        tl[t].wait_target = kids_f;
      }
      tl[t].signal_idx = gr.parent >= 0 ? FIN(gr.parent) : RDONE(g);
    }
    // parent's backward (root: own forward) -> (BIG: -x_B gather ->) backward
    for (int32_t t : gr.xtask) {
      SFCDD_REQUIRE(gr.parent >= 0, SFCDD_EINTERNAL, "root supernode with below rows");
      tl[t].wait_idx = BDONE(gr.parent);
      tl[t].wait_target = (int32_t)groups[gr.parent].btask.size();
      tl[t].signal_idx = XDONE(g);
    }
    for (int32_t t : gr.btask) {
      if (!gr.xtask.empty()) {
        tl[t].wait_idx = XDONE(g);
        tl[t].wait_target = (int32_t)gr.xtask.size();
      } else if (gr.parent >= 0) {
        tl[t].wait_idx = BDONE(gr.parent);
        tl[t].wait_target = (int32_t)groups[gr.parent].btask.size();
      } else {
        tl[t].wait_idx = RDONE(g);
        tl[t].wait_target = (int32_t)gr.ftask.size();
      }
      tl[t].signal_idx = BDONE(g);
    }
  }

  pt_[2] = ptime();
  // ---- 4. queue order: decreasing critical-path rank (HLFET) over the
  // combined forward/backward DAG -- a topological order (weights > 0)
  std::vector<double> wf(G, 0.0), wb(G, 0.0), wa(G, 0.0), wx(G, 0.0), rank_f(G, 0.0), rank_b(G, 0.0),
      succ_f(G, 0.0), succ_b(G, 0.0);
  for (int32_t g = 0; g < G; ++g) {
    for (int32_t t : groups[g].ftask) wf[g] = std::max(wf[g], tw[t]);
    for (int32_t t : groups[g].btask) wb[g] = std::max(wb[g], tw[t]);
    for (int32_t t : groups[g].atask) wa[g] = std::max(wa[g], tw[t]);
    for (int32_t t : groups[g].xtask) wx[g] = std::max(wx[g], tw[t]);
  }
  for (int32_t g = 0; g < G; ++g) {  // children before parents
    double mx = 0.0;
    for (int32_t c : groups[g].kids) mx = std::max(mx, rank_b[c]);
    succ_b[g] = mx;
    rank_b[g] = wx[g] + wb[g] + mx;
  }
  for (int32_t g = G - 1; g >= 0; --g) {  // parents before children
    succ_f[g] = groups[g].parent >= 0 ? rank_f[groups[g].parent] : rank_b[g];
    rank_f[g] = wa[g] + wf[g] + succ_f[g];
  }
  std::vector<double> rank(tl.size());
  for (size_t t = 0; t < tl.size(); ++t) {
    const int32_t g = tl[t].group;
    switch (tl[t].kind) {
      case TK_ASM_FWD: rank[t] = tw[t] + wf[g] + succ_f[g]; break;
      case TK_XB_BWD: rank[t] = tw[t] + wb[g] + succ_b[g]; break;
      case TK_FRAG_FWD:
      case TK_ROW_FWD: rank[t] = tw[t] + succ_f[g]; break;
      default: rank[t] = tw[t] + succ_b[g]; break;
    }
  }
  // queue = start order of a simulated list schedule on opt.workers warps:
  // whenever a warp is free it takes the highest-rank READY task.  At run
  // time warps dequeue in this order, so a task is (nearly) ready when it is
  // dequeued instead of pinning a warp while it waits.
  std::vector<int32_t> order;
  order.reserve(tl.size());
  {
    const int32_t nctr = 1 + CTR_PER_GROUP * G;
    std::vector<int32_t> ctr(nctr, 0);
    std::vector<std::vector<int32_t>> waiters(nctr);
    auto cmp_rank = [&](int32_t a, int32_t b) { return rank[a] < rank[b] || (rank[a] == rank[b] && a > b); };
    std::vector<int32_t> ready;  // max-heap by rank
    for (size_t t = 0; t < tl.size(); ++t) {
      if (tl[t].wait_idx < 0) {
        ready.push_back((int32_t)t);
      } else {
        waiters[tl[t].wait_idx].push_back((int32_t)t);
      }
    }
    std::make_heap(ready.begin(), ready.end(), cmp_rank);
    using Ev = std::pair<double, int32_t>;
    std::vector<Ev> ev;  // min-heap of (end time, task)
    auto ev_cmp = [](const Ev& a, const Ev& b) { return a.first > b.first; };
    // resident warps of the kernel: slots of blob_max + scratch, wpb-warp
    // CTAs, <= 20 worker warps/SM by registers (dag_solve.cu)
    int64_t workers = opt.workers;
    if (workers <= 0) {
      const int64_t slot = std::max<int64_t>(P.slot_need, 256);
      const int64_t ctas = std::max<int64_t>(1, (227 * 1024) / (opt.wpb * slot));
      workers = (int64_t)opt.sms * std::min<int64_t>(20, opt.wpb * ctas);
    }
    P.workers = (int32_t)workers;
    int64_t free_w = std::max<int64_t>(1, workers);
    double now = 0.0;
    while (order.size() < tl.size()) {
      while (free_w > 0 && !ready.empty()) {
        std::pop_heap(ready.begin(), ready.end(), cmp_rank);
        const int32_t t = ready.back();
        ready.pop_back();
        order.push_back(t);
        --free_w;
        ev.emplace_back(now + tw[t], t);
        std::push_heap(ev.begin(), ev.end(), ev_cmp);
      }
      if (order.size() == tl.size()) break;
      SFCDD_REQUIRE(!ev.empty(), SFCDD_EINTERNAL, "task graph has a cycle");
      std::pop_heap(ev.begin(), ev.end(), ev_cmp);
      const Ev e = ev.back();
      ev.pop_back();
      now = e.first;
      if (e.second < 0) {  // a waiter's release delay has passed: it is ready
        ready.push_back(-e.second - 1);
        std::push_heap(ready.begin(), ready.end(), cmp_rank);
        continue;
      }
      ++free_w;
      const int32_t c = tl[e.second].signal_idx;
      ++ctr[c];
      for (int32_t w : waiters[c])
        if (ctr[c] == tl[w].wait_target) {
          // modelled durations are means: a dependent task enters the queue
          // opt.slack_us after its last predecessor's modelled end, so at run
          // time its warp rarely finds the dependency still unfinished
          if (opt.slack_us > 0.0) {
            ev.emplace_back(now + opt.slack_us, -w - 1);
            std::push_heap(ev.begin(), ev.end(), ev_cmp);
          } else {
            ready.push_back(w);
            std::push_heap(ready.begin(), ready.end(), cmp_rank);
          }
        }
    }
    P.sim_us = now;
    P.crit_us = 0.0;
    int32_t cur = -1;
    for (size_t t = 0; t < tl.size(); ++t)
      if (rank[t] > P.crit_us) {
        P.crit_us = rank[t];
        cur = (int32_t)t;
      }
    if (std::getenv("SFCDD_PLAN_DEBUG") && cur >= 0) {
      // walk the critical path: successor with the largest rank
      std::vector<std::vector<int32_t>> succ(nctr);
      std::string path;
      int hops[TK_KINDS] = {0};
      double wsum[TK_KINDS] = {0};
      while (cur >= 0) {
        if (tl[cur].kind == TK_ROW_FWD) {
          const Group& gr = groups[tl[cur].group];
          const Supernode& S = factors[gr.factor]->sn[gr.top];
          path += " " + std::to_string(S.s) + "/" + std::to_string(S.m) + "(" +
                  std::to_string(groups[tl[cur].group].ftask.size()) + ")";
        }
        hops[tl[cur].kind]++;
        wsum[tl[cur].kind] += tw[cur];
        int32_t best = -1;
        for (int32_t w : waiters[tl[cur].signal_idx])
          if (best < 0 || rank[w] > rank[best]) best = w;
        cur = best;
      }
      std::fprintf(stderr, "[plan] critical big chain s/m(row tasks):%s\n", path.c_str());
      std::fprintf(stderr,
                   "[plan] critical path: frag_f %d (%.0f us) frag_b %d (%.0f us) row %d (%.0f us) col %d (%.0f us) "
                   "asm %d (%.0f us) xb %d (%.0f us)\n",
                   hops[0], wsum[0], hops[1], wsum[1], hops[2], wsum[2], hops[3], wsum[3], hops[4], wsum[4], hops[5],
                   wsum[5]);
    }
  }
  pt_[3] = ptime();
  P.tasks.resize(tl.size());
  for (size_t t = 0; t < order.size(); ++t) P.tasks[t] = tl[order[t]];

  if (std::getenv("SFCDD_PLAN_DEBUG") && !P.deferred) {  // (parses the host blob image)
    int64_t big_vals = 0, small_vals = 0, lev_sum = 0, sn_sum = 0, nrow = 0, ncol = 0;
    int32_t maxh = 0;
    for (const TaskDev& T : P.tasks) {
      if (T.kind == TK_FRAG_FWD) {
        small_vals += T.values;
        const int32_t* h = reinterpret_cast<const int32_t*>(P.blobs.data() + T.blob_off);
        lev_sum += h[H_NLEV];
        sn_sum += h[H_NSN];
      } else if (T.kind == TK_ROW_FWD) {
        ++nrow;
      } else if (T.kind == TK_COL_BWD) {
        big_vals += T.values;
        ++ncol;
      }
    }
    for (const Group& gr : groups) maxh = std::max(maxh, gr.height);
    {  // copied bytes vs factor value bytes per task kind
      double cb[TK_KINDS] = {0}, vb[TK_KINDS] = {0}, nt[TK_KINDS] = {0};
      for (const TaskDev& T : P.tasks) {
        cb[T.kind] += T.copy_bytes;
        vb[T.kind] += 8.0 * T.values;
        nt[T.kind] += 1;
      }
      double dense = 0, sparse = 0, hist[8] = {0};
      for (const TaskDev& T : P.tasks) {
        if (T.kind != TK_FRAG_FWD) continue;
        const int32_t* h = reinterpret_cast<const int32_t*>(P.blobs.data() + T.blob_off);
        const int32_t* rec = h + h[H_REC] + 4 * h[h[H_TOPS]];
        const double sc = h[H_NCOL], mt = (double)((unsigned)rec[0] >> 16);
        const double dv = sc * (sc + 1) / 2 + sc * mt;
        dense += dv;
        sparse += T.values;
        const double r = dv / std::max(1, T.values);
        hist[r < 1.25 ? 0 : r < 1.5 ? 1 : r < 2 ? 2 : r < 3 ? 3 : 4] += 1;
      }
      {
        double sp_sum = 0, nc_sum = 0, runs_sum = 0, nfr = 0, spx = 0, nx = 0;
        for (const TaskDev& T : P.tasks) {
          if (T.kind != TK_FRAG_FWD) continue;
          const int32_t* h = reinterpret_cast<const int32_t*>(P.blobs.data() + T.blob_off);
          const int32_t* cl = h + h[H_COLS];
          std::vector<int32_t> c(cl, cl + h[H_NCOL]);
          std::sort(c.begin(), c.end());
          int runs = c.empty() ? 0 : 1;
          for (size_t i = 1; i < c.size(); ++i) runs += c[i] != c[i - 1] + 1;
          if (!c.empty()) sp_sum += c.back() - c.front() + 1;
          nc_sum += c.size();
          runs_sum += runs;
          nfr += 1;
          const int32_t* ex = h + h[H_EXTX];
          std::vector<int32_t> e(ex, ex + h[H_NEXTX]);
          std::sort(e.begin(), e.end());
          if (!e.empty()) spx += e.back() - e.front() + 1;
          nx += e.size();
        }
        std::fprintf(stderr, "[plan] FRAG cols: avg %.1f, ro span %.1f (%.2fx), %.1f runs; ext rows %.1f span %.1f\n",
                     nc_sum / nfr, sp_sum / nfr, sp_sum / nc_sum, runs_sum / nfr, nx / nfr, spx / nfr);
      }
      {  // backward item mix
        double n_tiny = 0, n_pack = 0, n_cols = 0, w_tiny = 0, w_pack = 0, w_cols = 0, smax_pack = 0;
        for (const TaskDev& T : P.tasks) {
          if (T.kind != TK_FRAG_BWD) continue;
          const int32_t* h = reinterpret_cast<const int32_t*>(P.blobs.data() + T.blob_off);
          const int32_t* lv = h + h[H_LEVELS];
          const int32_t* it = h + h[H_ITEMS];
          const int32_t* rc = h + h[H_REC];
          for (int l = 0; l < h[H_NLEV]; ++l)
            for (int q = lv[L_WORDS * l + L_BI0]; q < lv[L_WORDS * l + L_BI1]; ++q) {
              const uint32_t ix = (uint32_t)it[2 * q];
              const int cnt = (int)((ix >> 16) & 0x7fffu);
              auto work = [&](int j) {
                const int s_ = rc[4 * j] & 0xfff, m_ = (int)((unsigned)rc[4 * j] >> 16);
                return (double)s_ * (s_ + m_) - 0.5 * s_ * (s_ - 1);
              };
              if (cnt == 0) {
                n_cols += 1;
                w_cols += work(ix);
              } else {
                double w = 0, sm = 0;
                for (int j = 0; j < cnt; ++j) {
                  w += work((ix & 0xffff) + j);
                  sm = std::max<double>(sm, rc[4 * ((ix & 0xffff) + j)] & 0xfff);
                }
                if (ix & 0x80000000u) {
                  n_tiny += 1;
                  w_tiny += w;
                } else {
                  n_pack += 1;
                  w_pack += w;
                  smax_pack += sm;
                }
              }
            }
        }
        std::fprintf(stderr, "[plan] FRAG bwd items: tiny %.0f (%.0f fma each), packed %.0f (%.0f fma, smax %.1f), cols %.0f (%.0f fma)\n",
                     n_tiny, w_tiny / std::max(1.0, n_tiny), n_pack, w_pack / std::max(1.0, n_pack),
                     smax_pack / std::max(1.0, n_pack), n_cols, w_cols / std::max(1.0, n_cols));
      }
      std::fprintf(stderr, "[plan] flattened FRAG values %.1f MB vs sparse %.1f MB (%.2fx); ratio hist <1.25 %.0f <1.5 %.0f <2 %.0f <3 %.0f >=3 %.0f\n",
                   8 * dense / 1e6, 8 * sparse / 1e6, dense / sparse, hist[0], hist[1], hist[2], hist[3], hist[4]);
      const char* nm[TK_KINDS] = {"frag_f", "frag_b", "row", "col", "asm", "xb"};
      for (int k = 0; k < TK_KINDS; ++k)
        std::fprintf(stderr, "[plan] %s: %.0f tasks, copied %.1f MB, values %.1f MB (%.2fx), %.0f B/task\n", nm[k],
                     nt[k], cb[k] / 1e6, vb[k] / 1e6, cb[k] / std::max(1.0, vb[k]), cb[k] / std::max(1.0, nt[k]));
    }
    {  // FRAG blob-size histogram, and the fragments hanging off BIG parents (sibling packing potential)
      double hb[6] = {0, 0, 0, 0, 0, 0}, nbp = 0, bbp = 0, nroot = 0;
      std::map<int32_t, std::pair<double, double>> per_parent;  // BIG parent group -> (fragments, bytes)
      for (const TaskDev& T : P.tasks) {
        if (T.kind != TK_FRAG_FWD) continue;
        const int b = T.copy_bytes < 512 ? 0 : T.copy_bytes < 1024 ? 1 : T.copy_bytes < 2048 ? 2 : T.copy_bytes < 4096 ? 3
                      : T.copy_bytes < 8192 ? 4 : 5;
        hb[b] += 1;
        const int32_t pg = groups[T.group].parent;
        if (pg < 0) nroot += 1;
        else if (groups[pg].big) {
          nbp += 1;
          bbp += T.copy_bytes;
          per_parent[pg].first += 1;
          per_parent[pg].second += T.copy_bytes;
        }
      }
      double bins = 0;
      for (const auto& kv : per_parent) bins += std::ceil(kv.second.second / (0.85 * opt.blob_max));
      std::fprintf(stderr,
                   "[plan] FRAG blob bytes: <512 %.0f <1K %.0f <2K %.0f <4K %.0f <8K %.0f >=8K %.0f; children of BIG "
                   "parents %.0f (%.0f B avg, %zu parents -> ~%.0f packed bins), roots %.0f\n",
                   hb[0], hb[1], hb[2], hb[3], hb[4], hb[5], nbp, bbp / std::max(1.0, nbp), per_parent.size(), bins, nroot);
    }
    {  // per-level FRAG work profile
      double nl = 0, runs = 0, pairs = 0, fi = 0, bi = 0, bpr = 0, ncol = 0, nxu = 0, nxx = 0, nf = 0, maxr = 0;
      for (const TaskDev& T : P.tasks) {
        if (T.kind != TK_FRAG_FWD) continue;
        const int32_t* h = reinterpret_cast<const int32_t*>(P.blobs.data() + T.blob_off);
        const int32_t* runs_a = h + h[H_RUNS];
        nf += 1;
        ncol += h[H_NCOL];
        nxu += h[H_NEXTU];
        nxx += h[H_NEXTX];
        for (int32_t l = 0; l < h[H_NLEV]; ++l) {
          const int32_t* L = h + h[H_LEVELS] + L_WORDS * l;
          nl += 1;
          runs += L[L_RUN1] - L[L_RUN0];
          maxr = std::max<double>(maxr, L[L_RUN1] - L[L_RUN0]);
          pairs += runs_a[L[L_RUN1]] - runs_a[L[L_RUN0]];
          fi += L[L_FI1] - L[L_FI0];
          bi += L[L_BI1] - L[L_BI0];
          bpr += L[L_BP1] - L[L_BP0];
        }
      }
      std::fprintf(stderr,
                   "[plan] FRAG per level: %.1f runs (%.1f pairs, max %.0f), %.1f fwd items, %.1f bwd items, %.1f "
                   "bwd pairs; per task: %.1f cols, %.1f ext updates, %.1f ext rows\n",
                   runs / nl, pairs / nl, maxr, fi / nl, bi / nl, bpr / nl, ncol / nf, nxu / nf, nxx / nf);
    }
    std::fprintf(stderr,
                 "[plan] groups=%d frag=%d big=%d (%.1f%% of values; %lld row + %lld col tasks) frag avg: %.1f "
                 "supernodes, %.1f levels, %.1f values; max group height %d; blobs %.1f MB; max scratch %d; "
                 "simulated schedule %.1f us on %d warps (critical path %.1f us)\n",
                 G, P.nfrag, P.nbig, 100.0 * big_vals / std::max<int64_t>(1, big_vals + small_vals),
                 (long long)nrow, (long long)ncol, (double)sn_sum / std::max(1, P.nfrag),
                 (double)lev_sum / std::max(1, P.nfrag), (double)small_vals / std::max(1, P.nfrag), maxh,
                 P.blobs.size() / 1e6, P.max_scratch, P.sim_us, P.workers, P.crit_us);
  }
  if (std::getenv("SFCDD_PLAN_DEBUG")) std::fprintf(stderr, "[plan] phase seconds: groups %.2f blobs %.2f deps %.2f queue %.2f\n", pt_[0], pt_[1], pt_[2], pt_[3]);
  return P;
}

}  // namespace sfcdd
