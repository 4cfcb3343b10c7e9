// C-ABI plumbing shared by all entry points, plus the host-only test hooks.
#include <chrono>
#include <cstring>
#include <string>

#include "common.h"
#include "host.h"
#include "plan.h"

namespace sfcdd {
static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace sfcdd

using namespace sfcdd;

extern "C" const char* sfcdd_last_error(void) { return g_last_error.c_str(); }

extern "C" int sfcdd_version(void) { return 1; }

static CsrMatrix csr_from(int64_t n, const int64_t* indptr, const int32_t* indices, const double* data) {
  CsrMatrix A;
  A.n = n;
  A.indptr.assign(indptr, indptr + n + 1);
  int64_t nnz = indptr[n];
  A.indices.assign(indices, indices + nnz);
  if (data)
    A.data.assign(data, data + nnz);
  else
    A.data.assign(nnz, 1.0);
  for (int64_t i = 0; i < nnz; ++i)
    SFCDD_REQUIRE(A.indices[i] >= 0 && A.indices[i] < n, SFCDD_EVALUE, "column index out of range");
  return A;
}

extern "C" int sfcdd_host_amd(int64_t n, const int64_t* indptr, const int32_t* indices, int32_t* perm_out) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(n >= 0, SFCDD_EVALUE, "negative dimension");
  CsrMatrix A = csr_from(n, indptr, indices, nullptr);
  SymPattern P;
  P.n = n;
  P.indptr = A.indptr;
  P.indices = A.indices;
  std::vector<int32_t> o = amd_order(P);
  std::memcpy(perm_out, o.data(), n * sizeof(int32_t));
  SFCDD_API_END
}

extern "C" int sfcdd_host_factor_solve(int64_t n, const int64_t* indptr, const int32_t* indices,
                                       const double* data, const double* b, double* x, int64_t* nnz_l,
                                       int64_t* stored) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(n >= 0, SFCDD_EVALUE, "negative dimension");
  CsrMatrix A = csr_from(n, indptr, indices, data);
  FactorOptions opt;
  HostFactor F = factorize_host(A, opt);
  host_block_solve(F, b, x);
  if (nnz_l) *nnz_l = F.nnz_l;
  if (stored) *stored = F.stored;
  SFCDD_API_END
}

namespace sfcdd {
// principal sub-block of a global CSR matrix on a cyclic range
CsrMatrix extract_block(const CsrMatrix& A, int64_t start, int64_t len) {
  const int64_t n = A.n;
  CsrMatrix B;
  B.n = len;
  B.indptr.assign(len + 1, 0);
  for (int64_t r = 0; r < len; ++r) {
    int64_t g = start + r;
    if (g >= n) g -= n;
    for (int64_t p = A.indptr[g]; p < A.indptr[g + 1]; ++p) {
      int64_t c = A.indices[p] - start;
      if (c < 0) c += n;
      if (c < len) {
        B.indices.push_back((int32_t)c);
        B.data.push_back(A.data[p]);
      }
    }
    B.indptr[r + 1] = B.indices.size();
  }
  return B;
}
}  // namespace sfcdd

extern "C" int sfcdd_host_plan_solve(int64_t n, const int64_t* indptr, const int32_t* indices,
                                     const double* data, int32_t p, const int64_t* start,
                                     const int64_t* len, const double* rhs, double* xy,
                                     int32_t blob_max, int32_t scratch_max, int64_t* nfrag) {
  SFCDD_API_BEGIN
  CsrMatrix A = csr_from(n, indptr, indices, data);
  std::vector<HostFactor> fs(p);
  FactorOptions fo;
  for (int32_t i = 0; i < p; ++i) fs[i] = factorize_host(extract_block(A, start[i], len[i]), fo);
  std::vector<const HostFactor*> ptrs;
  std::vector<int64_t> gs, gm;
  for (int32_t i = 0; i < p; ++i) {
    ptrs.push_back(&fs[i]);
    gs.push_back(start[i]);
    gm.push_back(n);
  }
  PlanOptions po;
  if (blob_max > 0) po.blob_max = blob_max;
  if (scratch_max > 0) po.scratch_max = scratch_max;
  if (blob_max <= 0) choose_blob_shape(ptrs, po);
  DevicePlan plan = build_plan(ptrs, gs, gm, po);
  plan_exec_host(plan, rhs, xy);
  if (nfrag) *nfrag = plan.ngroups;
  SFCDD_API_END
}

// Diagnostics (host only): wall seconds of the setup phases for one SPD block:
// times[0] ordering + symbolic analysis, times[1] host numeric factorization,
// times[2] device-plan build; sizes[0] nnz(L), sizes[1] stored, sizes[2]
// supernodes, sizes[3] sum over supernodes of m(m+1)/2 (update-matrix doubles),
// sizes[4] largest front, sizes[5] sum of s^3/3 + s^2 m + s m^2 (factor flops).
extern "C" int sfcdd_host_setup_timing(int64_t n, const int64_t* indptr, const int32_t* indices,
                                       const double* data, int32_t numeric, double* times, int64_t* sizes) {
  SFCDD_API_BEGIN
  CsrMatrix A = csr_from(n, indptr, indices, data);
  FactorOptions fo;
  auto t0 = std::chrono::steady_clock::now();
  HostFactor F = analyze_host(A, fo);
  auto t1 = std::chrono::steady_clock::now();
  if (numeric) numeric_host(A, F);
  auto t2 = std::chrono::steady_clock::now();
  if (numeric) {
    PlanOptions po;
    std::vector<const HostFactor*> ptrs{&F};
    choose_blob_shape(ptrs, po);
    DevicePlan plan = build_plan(ptrs, {0}, {n}, po);
  }
  auto t3 = std::chrono::steady_clock::now();
  times[0] = std::chrono::duration<double>(t1 - t0).count();
  times[1] = std::chrono::duration<double>(t2 - t1).count();
  times[2] = std::chrono::duration<double>(t3 - t2).count();
  int64_t upd = 0, fl = 0;
  for (const Supernode& S : F.sn) {
    upd += (int64_t)S.m * (S.m + 1) / 2;
    fl += (int64_t)S.s * S.s * S.s / 3 + (int64_t)S.s * S.s * S.m + (int64_t)S.s * S.m * S.m;
  }
  sizes[0] = F.nnz_l;
  sizes[1] = F.stored;
  sizes[2] = (int64_t)F.sn.size();
  sizes[3] = upd;
  sizes[4] = F.max_front;
  sizes[5] = fl;
  SFCDD_API_END
}

// Test hook (host only): the deferred-value plan (metadata segments + value
// descriptors, the path of device-side factor values) rebuilds exactly the
// blob image of the plan built with host values.  *mismatch = number of
// differing bytes (0 expected); *nseg / *nvd = segment / descriptor counts.
extern "C" int sfcdd_host_plan_deferred_check(int64_t n, const int64_t* indptr, const int32_t* indices,
                                              const double* data, int32_t p, const int64_t* start,
                                              const int64_t* len, int64_t* mismatch, int64_t* nseg,
                                              int64_t* nvd) {
  SFCDD_API_BEGIN
  CsrMatrix A = csr_from(n, indptr, indices, data);
  std::vector<HostFactor> fs(p), sym(p);
  FactorOptions fo;
  for (int32_t i = 0; i < p; ++i) {
    CsrMatrix B = extract_block(A, start[i], len[i]);
    fs[i] = factorize_host(B, fo);
    sym[i] = analyze_host(B, fo);
  }
  std::vector<const HostFactor*> pv, ps;
  std::vector<int64_t> gs, gm;
  for (int32_t i = 0; i < p; ++i) {
    pv.push_back(&fs[i]);
    ps.push_back(&sym[i]);
    gs.push_back(start[i]);
    gm.push_back(n);
  }
  PlanOptions po;
  choose_blob_shape(pv, po);
  DevicePlan full = build_plan(pv, gs, gm, po);
  po.defer_values = true;
  DevicePlan def = build_plan(ps, gs, gm, po);
  SFCDD_REQUIRE(def.blob_bytes == full.blob_bytes, SFCDD_EINTERNAL, "deferred plan size differs");
  std::vector<uint8_t> img((size_t)def.blob_bytes, 0);
  for (const MetaSeg& s : def.segs) std::memcpy(img.data() + s.dev_off, def.blobs.data() + s.host_off, s.bytes);
  for (const ValDesc& d : def.vdesc) place_values(d, fs[d.factor].val.data() + d.src, img.data());
  int64_t bad = 0;
  for (int64_t i = 0; i < def.blob_bytes; ++i) bad += img[i] != full.blobs[i];
  *mismatch = bad;
  *nseg = (int64_t)def.segs.size();
  *nvd = (int64_t)def.vdesc.size();
  SFCDD_REQUIRE(def.tasks.size() == full.tasks.size(), SFCDD_EINTERNAL, "task count differs");
  for (size_t t = 0; t < def.tasks.size(); ++t)
    SFCDD_REQUIRE(std::memcmp(&def.tasks[t], &full.tasks[t], sizeof(TaskDev)) == 0, SFCDD_EINTERNAL,
                  "task lists differ");
  SFCDD_API_END
}
