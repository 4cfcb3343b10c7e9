// Host interpreter of a DevicePlan: executes the warp tasks in queue order
// with exactly the blob semantics of the device kernel (dag_solve.cu) --
// FRAG level tables, gather runs, row pairs and warp items; ROW blocks with
// their gather runs; COL blocks -- and checks every task's dependency counter
// is satisfied when the queue reaches it.  Test hook only (lets the CPU test
// suite validate plan layouts without a GPU); not on the product path.
#include <algorithm>
#include <cstring>
#include <limits>
#include <vector>

#include "common.h"
#include "plan.h"

namespace sfcdd {

namespace {
inline int32_t lo16(int32_t v) { return (int32_t)((uint32_t)v & 0xffffu); }
inline int32_t hi16(int32_t v) { return (int32_t)((uint32_t)v >> 16); }
}  // namespace

void plan_exec_host(const DevicePlan& P, const double* rhs, double* xy) {
  std::vector<double> upd(P.upd_doubles, 0.0);
  std::vector<double> scratch;
  std::vector<int64_t> ctr(1 + CTR_PER_GROUP * (size_t)P.ngroups, 0);
  for (size_t t = 0; t < P.tasks.size(); ++t) {
    const TaskDev& T = P.tasks[t];
    SFCDD_REQUIRE(T.wait_idx < 0 || ctr[T.wait_idx] >= T.wait_target, SFCDD_EINTERNAL,
                  "task queue is not a topological order");
    const uint8_t* blob = P.blobs.data() + T.blob_off;
    const int32_t* h = reinterpret_cast<const int32_t*>(blob);
    const FactorDev& Fd = P.factors[T.factor];
    auto gidx = [&](int32_t ro) {
      int64_t g = Fd.gstart + ro;
      if (g >= Fd.gmod) g -= Fd.gmod;
      return g;
    };
    double* x = xy + Fd.xy_off;
    if (T.kind == TK_ASM_FWD) {
      const int32_t s = h[AS_S], q0 = h[AS_Q0], nq = h[AS_NQ];
      const int32_t* cols = h + h[AS_COLS];
      const int32_t* ptr = h + h[AS_PTR];
      const int32_t* src = h + h[AS_SRC];
      for (int32_t i = 0; i < nq; ++i) {
        const int32_t q = q0 + i;
        double acc = q < s ? rhs[gidx(cols[i])] : 0.0;
        for (int32_t e = ptr[i]; e < ptr[i + 1]; ++e) acc += upd[src[e]];
        upd[h[AS_FOFF] + q] = acc;
      }
    } else if (T.kind == TK_XB_BWD) {
      const int32_t* rows = h + h[XB_ROWS];
      for (int32_t i = 0; i < h[XB_NA]; ++i) upd[h[XB_XOFF] + h[XB_A0] + i] = -x[rows[i]];
    } else if (T.kind == TK_ROW_FWD) {
      const double* V = reinterpret_cast<const double*>(blob + h[RW_VAL_OFF]);
      const int32_t s = h[RW_S], R = h[RW_R], C = h[RW_C], r0 = h[RW_R0], NB = h[RW_NB];
      if (h[RW_NBLK] > 1) {  // MROW: blocks of R update rows, leading dimension R, C = s
        const double* f = upd.data() + h[RW_FOFF];
        for (int32_t b = 0; b < h[RW_NBLK]; ++b)
          for (int32_t i = 0; i < R && b * R + i < NB; ++i) {
            double acc = 0.0;
            for (int32_t k = 0; k < C; ++k) acc += V[((size_t)b * C + k) * R + i] * f[k];
            const int32_t rw = r0 + b * R + i;
            upd[h[RW_UOFF] + rw - s] = f[rw] - acc;
          }
        ctr[T.signal_idx] += 1;
        continue;
      }
      scratch.assign(C + NB, 0.0);
      double* S = scratch.data();
      if (h[RW_FOFF] >= 0) {
        const double* f = upd.data() + h[RW_FOFF];
        for (int32_t q = 0; q < C; ++q) S[q] = f[q];
        for (int32_t i = 0; i < NB; ++i) S[C + i] = f[r0 + i];
      } else {
        const bool ga = h[RW_ASM_HI] >= 0;  // global assembly record (huge s)
        const int64_t o16 = ga ? ((int64_t)(uint32_t)h[RW_ASM16] | ((int64_t)h[RW_ASM_HI] << 32)) : 0;
        const int32_t* am = reinterpret_cast<const int32_t*>(P.blobs.data() + 16 * o16);
        const int32_t* cols = ga ? am + 2 : h + h[RW_COLS];
        const int32_t* ptr = ga ? am + 2 + am[0] : h + h[RW_PTR];
        const int32_t* src = ga ? ptr + am[0] + am[1] + 1 : h + h[RW_SRC];
        for (int32_t q = 0; q < C + NB; ++q) {
          const int32_t p = ga ? (q < C ? q : r0 + (q - C)) : q;
          double acc = q < C ? rhs[gidx(cols[q])] : 0.0;
          for (int32_t e = ptr[p]; e < ptr[p + 1]; ++e) acc += upd[src[e]];
          S[q] = acc;
        }
      }
      for (int32_t i = 0; i < R; ++i) {
        double acc = 0.0;
        for (int32_t k = 0; k < C; ++k) acc += V[(size_t)k * R + i] * S[k];
        const int32_t rw = r0 + i;
        if (rw < s)
          upd[h[RW_YOFF] + rw] = acc;
        else
          upd[h[RW_UOFF] + rw - s] = S[C + i] - acc;
      }
    } else if (T.kind == TK_COL_BWD) {
      const double* V = reinterpret_cast<const double*>(blob + h[CL_VAL_OFF]);
      const int32_t s = h[CL_S], m = h[CL_M], k0 = h[CL_K0], c = h[CL_C];
      const int32_t* cols = h + h[CL_COLS];
      const int32_t L = s + m - k0;
      scratch.assign(L, 0.0);
      double* v = scratch.data();
      for (int32_t i = k0; i < s; ++i) v[i - k0] = upd[h[CL_YOFF] + i];
      for (int32_t a = 0; a < m; ++a)
        v[s - k0 + a] = h[CL_XOFF] >= 0 ? upd[h[CL_XOFF] + a] : -x[h[h[CL_ROWS] + a]];
      for (int32_t j = 0; j < c; ++j) {
        double acc = 0.0;
        for (int32_t r = j; r < L; ++r) acc += V[(size_t)r * c + j] * v[r];
        x[cols[j]] = acc;
      }
    } else {
      const bool fwd = T.kind == TK_FRAG_FWD;
      const double* vals = reinterpret_cast<const double*>(blob + h[H_VAL_OFF]);
      const int32_t* recs = h + h[H_REC];
      const int32_t* cols = h + h[H_COLS];
      // like the kernel: only the frontal slots are zeroed; everything else
      // must be written before it is read (NaN poison catches a miss)
      scratch.assign(h[H_SCRATCH], std::numeric_limits<double>::quiet_NaN());
      if (fwd) std::fill(scratch.begin(), scratch.begin() + h[H_ZERO], 0.0);
      double* S = scratch.data();
      const int32_t ncol = h[H_NCOL];
      const int32_t* colpos = h + h[H_COLPOS];
      const int32_t nlev = h[H_NLEV];
      const int32_t* levtab = h + h[H_LEVELS];
      const int32_t* runs = h + h[H_RUNS];
      const int32_t* gp = h + h[H_GPAIRS];
      const int32_t* bp = h + h[H_BPAIRS];
      const int32_t* items = h + h[H_ITEMS];
      auto rs = [&](const int32_t* R) { return R[R_SM] & 0xfff; };
      auto rlp = [&](const int32_t* R) { return (R[R_SM] >> 12) & 7; };
      auto rm = [&](const int32_t* R) { return (int32_t)((uint32_t)R[R_SM] >> 16); };
      // rows handled by a warp item, in lane order (also checks the lane masks)
      auto item_rows = [&](int32_t x0, int32_t y, bool forward, auto&& fn) {
        x0 &= 0x7fffffff;  // forward "tiny" flag
        const int32_t cnt = x0 >> 16;
        if (cnt > 0 && !forward) {  // column lanes, descending records, segments aligned to 2^lp
          x0 &= 0xffff;
          uint32_t mask = 0;
          int32_t off = 0;
          for (int32_t q = 0; q < cnt; ++q) {
            const int32_t* R = recs + R_WORDS * (x0 + cnt - 1 - q);
            const int32_t Pq = 1 << rlp(R);
            off = (off + Pq - 1) / Pq * Pq;
            mask |= 1u << off;
            off += rs(R) * Pq;
          }
          if (off < 32) mask |= 1u << off;
          SFCDD_REQUIRE(off <= 32 && mask == (uint32_t)y, SFCDD_EINTERNAL, "backward item lane mask mismatch");
          for (int32_t j = x0; j < x0 + cnt; ++j)
            for (int32_t k = 0; k < rs(recs + R_WORDS * j); ++k) fn(recs + R_WORDS * j, k);
        } else if (cnt > 0) {
          x0 &= 0xffff;
          uint32_t mask = 0;
          int32_t rows = 0;
          for (int32_t j = x0; j < x0 + cnt; ++j) {
            mask |= 1u << rows;
            rows += rs(recs + R_WORDS * j) + rm(recs + R_WORDS * j);
          }
          if (rows < 32) mask |= 1u << rows;
          SFCDD_REQUIRE(rows <= 32 && mask == (uint32_t)y, SFCDD_EINTERNAL, "packed item lane mask mismatch");
          for (int32_t j = x0; j < x0 + cnt; ++j) {
            const int32_t* R = recs + R_WORDS * j;
            if (forward)
              for (int32_t i = 0; i < rs(R) + rm(R); ++i) fn(R, i);
            else
              for (int32_t k = 0; k < rs(R); ++k) fn(R, k);
          }
        } else {
          const int32_t* R = recs + R_WORDS * x0;
          if (forward)
            for (int32_t i = 32 * y; i < std::min(32 * y + 32, rs(R) + rm(R)); ++i) fn(R, i);
          else
            for (int32_t k = y & 0xffff; k < (y & 0xffff) + (y >> 16); ++k) fn(R, k);
        }
      };
      if (fwd) {
        for (int32_t c = 0; c < ncol; ++c) S[lo16(colpos[c])] = rhs[gidx(cols[c])];
        const int32_t* eu = h + h[H_EXTU];
        for (int32_t e = 0; e < h[H_NEXTU]; ++e) S[h[H_EXTU_BASE] + e] = upd[eu[e]];
        for (int32_t l = 0; l < nlev; ++l) {
          const int32_t* L = levtab + L_WORDS * l;
          for (int32_t r = L[L_RUN0]; r < L[L_RUN1]; ++r) {
            const int32_t dst = lo16(gp[runs[r]]);
            double acc = S[dst];
            for (int32_t p = runs[r]; p < runs[r + 1]; ++p) acc += S[hi16(gp[p])];
            S[dst] = acc;
          }
          for (int32_t it = L[L_FI0]; it < L[L_FI1]; ++it)
            item_rows(items[2 * it], items[2 * it + 1], true, [&](const int32_t* R, int32_t i) {
              const int32_t s = rs(R), m = rm(R);
              const double* M = vals + R[R_VAL];
              double* f = S + R[R_SCR];
              double acc = 0.0;
              const int32_t kmax = i < s ? i : s - 1;
              for (int32_t k = 0; k <= kmax; ++k) acc += M[packed_col_off(s, m, k) + (i - k)] * f[k];
              if (i < s)
                S[R[R_CPOS] + i] = acc;
              else
                f[i] -= acc;
            });
        }
        for (int32_t c = 0; c < ncol; ++c) x[cols[c]] = S[hi16(colpos[c])];
        for (int32_t tp = 0; tp < h[H_NTOP]; ++tp) {
          const int32_t* tops = h + h[H_TOPS] + 2 * tp;
          if (tops[1] < 0) continue;
          const int32_t* R = recs + R_WORDS * tops[0];
          for (int32_t a = 0; a < rm(R); ++a) upd[tops[1] + a] = S[R[R_SCR] + rs(R) + a];
        }
      } else {
        for (int32_t c = 0; c < ncol; ++c) S[lo16(colpos[c])] = x[cols[c]];
        const int32_t* ex = h + h[H_EXTX];
        for (int32_t e = 0; e < h[H_NEXTX]; ++e) S[h[H_EXTX_BASE] + e] = x[ex[e]];
        for (int32_t l = nlev - 1; l >= 0; --l) {
          const int32_t* L = levtab + L_WORDS * l;
          for (int32_t p = L[L_BP0]; p < L[L_BP1]; ++p) S[lo16(bp[p])] = -S[hi16(bp[p])];
          for (int32_t it = L[L_BI0]; it < L[L_BI1]; ++it)
            item_rows(items[2 * it], items[2 * it + 1], false, [&](const int32_t* R, int32_t k) {
              const int32_t s = rs(R), m = rm(R);
              const double* col = vals + R[R_VAL] + packed_col_off(s, m, k);
              const double* v = S + R[R_SCR];
              double acc = 0.0;
              for (int32_t i = k; i < s + m; ++i) acc += col[i - k] * v[i];
              S[R[R_CPOS] + k] = acc;
            });
        }
        for (int32_t c = 0; c < ncol; ++c) x[cols[c]] = S[hi16(colpos[c])];
      }
    }
    ctr[T.signal_idx] += 1;
  }
}

}  // namespace sfcdd
