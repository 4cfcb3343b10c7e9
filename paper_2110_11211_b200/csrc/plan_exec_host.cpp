// Host interpreter of a DevicePlan: executes the forward/backward tasks in
// queue order with exactly the blob semantics of the device kernel
// (dag_solve.cu).  Test hook only -- lets the CPU test suite check the plan
// layout (fragments, child records, relative maps, update slots) without a
// GPU.  Not used by the product path.
#include <cstring>
#include <vector>

#include "common.h"
#include "plan.h"

namespace sfcdd {

void plan_exec_host(const DevicePlan& P, const double* rhs, double* xy) {
  std::vector<double> upd(P.upd_doubles, 0.0);
  std::vector<double> scratch;
  const int32_t nf = P.nfrag;
  for (int32_t t = 0; t < 2 * nf; ++t) {
    const TaskDev& T = P.tasks[t];
    const bool fwd = t < nf;
    const uint8_t* blob = P.blobs.data() + T.blob_off;
    const int32_t* h = reinterpret_cast<const int32_t*>(blob);
    const double* vals = reinterpret_cast<const double*>(blob + h[H_VAL_OFF]);
    const FactorDev& Fd = P.factors[T.factor];
    const int32_t nlev = h[H_NLEV];
    const int32_t* lev_ptr = h + h[H_LEV_PTR];
    const int32_t* lev_list = h + h[H_LEV_LIST];
    const int32_t* recs = h + h[H_REC];
    scratch.assign(h[H_SCRATCH], 0.0);
    auto gidx = [&](int32_t ro) {
      int64_t g = Fd.gstart + ro;
      if (g >= Fd.gmod) g -= Fd.gmod;
      return g;
    };
    if (fwd) {
      for (int32_t lv = 0; lv < nlev; ++lv) {
        for (int32_t j = lev_ptr[lv]; j < lev_ptr[lv + 1]; ++j) {
          const int32_t l = lev_list[j];
          const int32_t* R = recs + R_WORDS * l;
          const int32_t s = R[R_S], m = R[R_M];
          double* f = scratch.data() + R[R_SCR];
          const int32_t* ro = h + R[R_IDX];
          for (int32_t i = 0; i < s; ++i) f[i] = rhs[gidx(ro[i])];
          for (int32_t i = s; i < s + m; ++i) f[i] = 0.0;
          for (int32_t q = 0; q < R[R_NCH]; ++q) {
            const int32_t* cr = h + R[R_CH] + CH_WORDS * q;
            const double* src;
            if (cr[0] >= 0) {
              const int32_t* RC = recs + R_WORDS * cr[0];
              src = scratch.data() + RC[R_SCR] + RC[R_S];
            } else {
              src = upd.data() + cr[3];
            }
            const int32_t* rel = h + cr[2];
            for (int32_t a = 0; a < cr[1]; ++a) f[rel[a]] += src[a];
          }
          const double* M = vals + R[R_VAL];
          for (int32_t i = 0; i < s + m; ++i) {
            double acc = 0.0;
            const int32_t kmax = i < s ? i : s - 1;
            for (int32_t k = 0; k <= kmax; ++k) acc += M[packed_col_off(s, m, k) + (i - k)] * f[k];
            if (i < s)
              xy[Fd.xy_off + ro[i]] = acc;
            else
              f[i] -= acc;
          }
          if (R[R_PARENT] < 0 && h[H_TOP_UPD] >= 0)
            for (int32_t a = 0; a < m; ++a) upd[h[H_TOP_UPD] + a] = f[s + a];
        }
      }
    } else {
      std::vector<double> v;
      for (int32_t lv = nlev - 1; lv >= 0; --lv) {
        for (int32_t j = lev_ptr[lv]; j < lev_ptr[lv + 1]; ++j) {
          const int32_t l = lev_list[j];
          const int32_t* R = recs + R_WORDS * l;
          const int32_t s = R[R_S], m = R[R_M];
          const int32_t* ro = h + R[R_IDX];
          v.resize(s + m);
          for (int32_t i = 0; i < s; ++i) v[i] = xy[Fd.xy_off + ro[i]];
          for (int32_t a = 0; a < m; ++a) v[s + a] = -xy[Fd.xy_off + ro[s + a]];
          const double* M = vals + R[R_VAL];
          for (int32_t k = 0; k < s; ++k) {
            double acc = 0.0;
            const double* col = M + packed_col_off(s, m, k);
            for (int32_t i = k; i < s + m; ++i) acc += col[i - k] * v[i];
            xy[Fd.xy_off + ro[k]] = acc;
          }
        }
      }
    }
  }
}

}  // namespace sfcdd
