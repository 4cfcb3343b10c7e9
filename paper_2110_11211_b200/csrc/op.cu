// The two-level Schwarz operator: matrix-free stencil, coarse space, local
// solves (DagSolver), weighting/combination, and a device-resident PCG.
//
// Reference composition replaced here (paths relative to
// /root/reference/pkg/src/sfcdd/):
//   grid.assemble_laplacian + symmetrize_diag   grid.py:91-130   -> Stencil
//   partition.compute_weights                   partition.py:151 -> cover/weights
//   coarse.build_coarse / DeflationOperators    coarse.py:38-88  -> R0 chunks, A0^{-1}
//   schwarz.SchwarzOperator.apply               schwarz.py:103   -> apply()
//   krylov.pcg                                  krylov.py:257    -> pcg()
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>

#include "gpu_factor.h"
#include "op.h"
#include "plan.h"
#include "tiles.h"

namespace sfcdd {

CsrMatrix extract_block(const CsrMatrix& A, int64_t start, int64_t len);

namespace {

inline unsigned nblocks(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

template <typename F>
void parallel_for(int64_t n, int threads, F fn) {
  threads = std::max(1, std::min<int>(threads, (int)n));
  if (threads == 1) {
    for (int64_t i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<int64_t> next{0};
  std::vector<std::thread> pool;
  std::exception_ptr err;
  std::mutex mu;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      for (;;) {
        int64_t i = next.fetch_add(1);
        if (i >= n) break;
        try {
          fn(i);
        } catch (...) {
          std::lock_guard<std::mutex> g(mu);
          if (!err) err = std::current_exception();
          next = n;
        }
      }
    });
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

// ------------------------------------------------------------ device side
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// deterministic block-wide sum (fixed tree), result valid in every thread
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double red[VEC_THREADS / 32];
  __shared__ double total;
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < VEC_THREADS / 32 ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) total = t;
  }
  __syncthreads();
  return total;
}

// two deterministic block-wide sums at once (one set of barriers)
__device__ __forceinline__ double2 block_sum2(double a, double b) {
  __shared__ double2 red2[VEC_THREADS / 32];
  __shared__ double2 total2;
  a = warp_sum(a);
  b = warp_sum(b);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red2[warp] = make_double2(a, b);
  __syncthreads();
  if (warp == 0) {
    double2 t = lane < VEC_THREADS / 32 ? red2[lane] : make_double2(0.0, 0.0);
    t.x = warp_sum(t.x);
    t.y = warp_sum(t.y);
    if (lane == 0) total2 = t;
  }
  __syncthreads();
  return total2;
}

// points of a reduction chunk are processed PT per thread per round, every
// load of a round issued before any use (memory-level parallelism)
constexpr int PT = 4;

// last-block election; the last block must reset *ticket
__device__ __forceinline__ bool last_block(uint32_t* ticket) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) am_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  return am_last;
}

__device__ __forceinline__ double reduce_partials(const double* part, int n) {
  double v = 0.0;
#pragma unroll 4
  for (int i = threadIdx.x; i < n; i += VEC_THREADS) v += __ldcg(part + i);
  return block_sum(v);
}

__device__ __forceinline__ double stencil_at(const Stencil& S, const double* __restrict__ x, int64_t g) {
  double acc = S.dhat * x[g];
  for (int a = 0; a < 2 * S.d; ++a) {
    const int32_t nb = __ldg(S.nbr + (int64_t)a * S.n + g);
    if (nb >= 0) acc = fma(S.off[a >> 1], x[nb], acc);
  }
  return acc;
}

__device__ __forceinline__ bool skip(const DevState* st) { return st != nullptr && st->done; }

// neighbour table from perm/rank (grid.py:91-114 assembles the same couplings)
__global__ void k_nbr(GridGeom g, const int64_t* __restrict__ perm, const int64_t* __restrict__ rank,
                      int32_t* __restrict__ nbr) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= g.n) return;
  int64_t lex = perm[s];
  int64_t c[MAX_GRID_DIM];
  int64_t stride[MAX_GRID_DIM];
  int64_t rem = lex, st = 1;
  for (int j = g.d - 1; j >= 0; --j) {
    c[j] = rem % g.shape[j];
    rem /= g.shape[j];
    stride[j] = st;
    st *= g.shape[j];
  }
  for (int j = 0; j < g.d; ++j) {
    nbr[(int64_t)(2 * j) * g.n + s] = c[j] > 0 ? (int32_t)rank[lex - stride[j]] : -1;
    nbr[(int64_t)(2 * j + 1) * g.n + s] = c[j] + 1 < g.shape[j] ? (int32_t)rank[lex + stride[j]] : -1;
  }
}

__global__ void k_fill_agg(const int64_t* __restrict__ agg_start, int32_t n0, int32_t* __restrict__ agg) {
  const int32_t a = blockIdx.x;
  if (a >= n0) return;
  for (int64_t g = agg_start[a] + threadIdx.x; g < agg_start[a + 1]; g += blockDim.x) agg[g] = a;
}

// per-chunk sums of v (R0 v partials) -- coarse.py:78 restriction
__global__ void k_chunk_sum(const double* __restrict__ v, Chunks C, double* __restrict__ part) {
  const int ch = blockIdx.x;
  double s = 0.0;
  const int64_t c_end = C.start[ch + 1];
  for (int64_t g = C.start[ch] + threadIdx.x; g < c_end; g += VEC_THREADS) s += v[g];
  s = block_sum(s);
  if (threadIdx.x == 0) part[ch] = s;
}

// y0 = A0^{-1} c with c[a] = sum of the chunk partials of aggregate a.
// Dense GEMV over the redundant coarse inverse (Bank-Holst copy):
// GEMV_WPR warps per row, 8 independent loads per lane in flight, partial
// sums combined in a fixed order (bitwise reproducible).  When every
// aggregate is one chunk (`direct`), c is the partial array itself;
// otherwise each CTA sums the partials into shared memory first.
constexpr int GEMV_WPR = 4;
constexpr int GEMV_ROWS = VEC_THREADS / 32 / GEMV_WPR;
struct PcgFin {           // fused PCG epilogue of the second coarse GEMV
  const double* part_rw;  // per-chunk r.w partials (k_combine_chunk)
  const double* part_rc;  // per-chunk R0 r partials (k_update / k_residual0)
  const double* y0;       // A0^{-1} R0 r
  int32_t nch;
  DevState* st;           // null: no epilogue
  const int32_t* rc_ptr;  // first chunk of each aggregate (n0 + 1)
  bool rc_direct;         // every aggregate is one chunk (part_rc is per aggregate)
};

// rows [GEMV_ROWS rg, GEMV_ROWS (rg + 1)) of y = A0^{-1} c (every thread of
// the CTA calls it; c in global memory read through L2 when `cglobal`)
__device__ __forceinline__ void gemv_rowgroup(const double* __restrict__ ainv, const double* c, bool cglobal,
                                              int32_t n0, int rg, double* __restrict__ y) {
  __shared__ double red[VEC_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = rg * GEMV_ROWS + warp / GEMV_WPR;
  const int pw = warp % GEMV_WPR;
  const int span = (n0 + GEMV_WPR - 1) / GEMV_WPR;
  const int j0 = pw * span, j1 = min(n0, j0 + span);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (row < n0) {
    const double* ar = ainv + (int64_t)row * n0;
    int j = j0 + lane;
    for (; j + 7 * 32 < j1; j += 8 * 32) {
      double v[8], cv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        v[u] = __ldg(ar + j + 32 * u);
        cv[u] = cglobal ? __ldcg(c + j + 32 * u) : c[j + 32 * u];
      }
      a0 = fma(v[0], cv[0], a0);
      a1 = fma(v[1], cv[1], a1);
      a2 = fma(v[2], cv[2], a2);
      a3 = fma(v[3], cv[3], a3);
      a0 = fma(v[4], cv[4], a0);
      a1 = fma(v[5], cv[5], a1);
      a2 = fma(v[6], cv[6], a2);
      a3 = fma(v[7], cv[7], a3);
    }
    for (; j < j1; j += 32) a0 = fma(__ldg(ar + j), cglobal ? __ldcg(c + j) : c[j], a0);
  }
  const double acc = warp_sum((a0 + a1) + (a2 + a3));
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x < GEMV_ROWS) {
    const int r = rg * GEMV_ROWS + threadIdx.x;
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < GEMV_WPR; ++k) t += red[threadIdx.x * GEMV_WPR + k];
    if (r < n0) y[r] = t;
  }
  __syncthreads();  // red is reused by the next row group
}

// c[a] = sum of the partials part[ptr[a]] .. part[ptr[a+1]-1], into shared
// memory; 4 segments per thread with their first 3 loads in flight together
__device__ __forceinline__ void sum_segments(const double* __restrict__ part, const int32_t* __restrict__ ptr,
                                             int32_t n0, double* csm) {
  constexpr int U = 4;
  for (int a0 = threadIdx.x; a0 < n0; a0 += U * VEC_THREADS) {
    int e0[U], e1[U];
    double v0[U], v1[U], v2[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int a = a0 + u * VEC_THREADS;
      e0[u] = a < n0 ? ptr[a] : 0;
      e1[u] = a < n0 ? ptr[a + 1] : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int n = e1[u] - e0[u];
      v0[u] = n > 0 ? __ldcg(part + e0[u]) : 0.0;
      v1[u] = n > 1 ? __ldcg(part + e0[u] + 1) : 0.0;
      v2[u] = n > 2 ? __ldcg(part + e0[u] + 2) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int a = a0 + u * VEC_THREADS;
      if (a >= n0) continue;
      const int n = e1[u] - e0[u];
      double s = 0.0;
      if (n > 0) s += v0[u];
      if (n > 1) s += v1[u];
      if (n > 2) s += v2[u];
      for (int e = e0[u] + 3; e < e1[u]; ++e) s += __ldcg(part + e);
      csm[a] = s;
    }
  }
  __syncthreads();
}

// Fused PCG epilogue (one CTA, after y = A0^{-1} R0 A w is complete):
// r.z without materialising z = (w - R0^T y0b) + R0^T y0 (schwarz.py:117-118):
// r.z = r.w + (R0 r).(y0 - y0b); then beta (krylov.py:288-289).  The R0 r
// partials are per reduction chunk: summed per aggregate through rc_ptr
// unless every aggregate is exactly one chunk.
__device__ __forceinline__ void pcg_fin_epilogue(const PcgFin& fin, int32_t n0, const double* y) {
  double rw = 0.0, cd = 0.0;
#pragma unroll 4
  for (int i = threadIdx.x; i < fin.nch; i += VEC_THREADS) rw += __ldcg(fin.part_rw + i);
  if (fin.rc_direct) {  // aggregate a = chunk a
#pragma unroll 4
    for (int a = threadIdx.x; a < n0; a += VEC_THREADS)
      cd = fma(__ldcg(fin.part_rc + a), __ldcg(fin.y0 + a) - __ldcg(y + a), cd);
  } else {
    for (int a = threadIdx.x; a < n0; a += VEC_THREADS) {
      double ra = 0.0;
      for (int ch = fin.rc_ptr[a]; ch < fin.rc_ptr[a + 1]; ++ch) ra += __ldcg(fin.part_rc + ch);
      cd = fma(ra, __ldcg(fin.y0 + a) - __ldcg(y + a), cd);
    }
  }
  const double2 tot = block_sum2(rw, cd);
  rw = tot.x;
  cd = tot.y;
  if (threadIdx.x == 0) {
    DevState* S = fin.st;
    S->ticket[5] = 0;
    S->apply_calls += 1;
    const double rz = rw + cd;
    S->beta = S->have_rz ? rz / S->rz : 0.0;
    S->have_rz = 1;
    S->rz = rz;
  }
}

__global__ void k_coarse_gemv(const double* __restrict__ ainv, const double* __restrict__ part,
                              const int32_t* __restrict__ agg_ptr, int32_t n0, double* __restrict__ y,
                              const DevState* st, bool direct, PcgFin fin) {
  if (skip(st)) return;
  extern __shared__ double csm[];
  const double* c = part;
  if (!direct) {
    sum_segments(part, agg_ptr, n0, csm);
    c = csm;
  }
  gemv_rowgroup(ainv, c, direct, n0, blockIdx.x, y);
  if (fin.st && last_block(&fin.st->ticket[5])) pcg_fin_epilogue(fin, n0, y);
}

// c[a] = sum of the chunk partials of aggregate a (sparse coarse path)
__global__ void k_seg_sum(const double* __restrict__ part, const int32_t* __restrict__ ptr, int32_t n0,
                          double* __restrict__ c, const DevState* st) {
  if (skip(st)) return;
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n0) return;
  double s = 0.0;
  for (int ch = ptr[a]; ch < ptr[a + 1]; ++ch) s += __ldcg(part + ch);
  c[a] = s;
}

// y = the coarse DAG solution (sparse coarse path), then the fused PCG
// epilogue in the last block (as k_coarse_gemv)
__global__ void k_coarse_out(const double* __restrict__ xy, int32_t n0, double* __restrict__ y, const DevState* st,
                             PcgFin fin) {
  if (skip(st)) return;
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a < n0) y[a] = __ldcg(xy + a);
  if (fin.st && last_block(&fin.st->ticket[5])) pcg_fin_epilogue(fin, n0, y);
}

// t = g - Â R0^T y0   (schwarz.py:116: g - A @ F(g))
__global__ void k_tvec(const double* __restrict__ gv, const double* __restrict__ y0,
                       const int32_t* __restrict__ agg, Stencil S, double* __restrict__ t,
                       const DevState* st) {
  if (skip(st)) return;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= S.n) return;
  double acc = S.dhat * y0[agg[g]];
  for (int a = 0; a < 2 * S.d; ++a) {
    const int32_t nb = __ldg(S.nbr + (int64_t)a * S.n + g);
    if (nb >= 0) acc = fma(S.off[a >> 1], y0[agg[nb]], acc);
  }
  t[g] = gv[g] - acc;
}

struct CombineArgs {
  const double* xy;
  const int64_t* ov_start;
  const int64_t* ov_len;
  const int64_t* xy_off;
  const int64_t* dj_start;  // p + 1
  const int32_t* cand_ptr;
  const int32_t* cand;
  const double* wgt;     // omega_i or 1
  const int32_t* count;  // d_matrix weighting: cover counts (nullable)
  const int8_t* fault;   // nullable
  const long long* apply_calls;
  long long fault_index;
  int32_t p;
  int64_t n;
};

// w = sum_i R_i^T D_i A_i^{-1} R_i (.) in subdomain order (schwarz.py:84-100)
__global__ void k_combine(CombineArgs C, double* __restrict__ w, const DevState* st) {
  if (skip(st)) return;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= C.n) return;
  int lo = 0, hi = C.p;  // owner: dj_start[k] <= g < dj_start[k+1]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (C.dj_start[mid] <= g)
      lo = mid;
    else
      hi = mid;
  }
  const bool faulty = C.fault != nullptr && *C.apply_calls == C.fault_index;
  double acc = 0.0;
  for (int c = C.cand_ptr[lo]; c < C.cand_ptr[lo + 1]; ++c) {
    const int i = C.cand[c];
    int64_t off = g - C.ov_start[i];
    if (off < 0) off += C.n;
    if (off >= C.ov_len[i]) continue;
    if (faulty && C.fault[i]) continue;
    double wt = C.count ? 1.0 / (double)C.count[g] : C.wgt[i];
    acc = __dadd_rn(acc, __dmul_rn(wt, __ldcg(C.xy + C.xy_off[i] + off)));
  }
  w[g] = acc;
}

constexpr int COMBINE_MAXC = 32;

// the points [g0, g1) of one reduction chunk: w[g] = sum over the chunk's
// candidate subdomains c (staged in shared memory, ascending) covering g of
// wt_c * xy_c[g - start_c], in candidate order.  Returns this thread's share
// of r.w (rdot != null).  (Batching the candidate loads of several points
// per thread was measured slower: +13 % on C2, +33 % on C3.)
__device__ __forceinline__ double combine_points(const CombineArgs& C, const int64_t* s_start, const int64_t* s_len,
                                                 const int64_t* s_off, const double* s_w, int nc, int64_t g0,
                                                 int64_t g1, double* __restrict__ w, const double* rdot) {
  double rw = 0.0;
  for (int64_t g = g0 + threadIdx.x; g < g1; g += VEC_THREADS) {
    const double dw = C.count ? 1.0 / (double)C.count[g] : 0.0;
    double acc = 0.0;
    for (int c = 0; c < nc; ++c) {
      int64_t off = g - s_start[c];
      if (off < 0) off += C.n;
      if (off < s_len[c]) acc = __dadd_rn(acc, __dmul_rn(C.count ? dw : s_w[c], __ldcg(C.xy + s_off[c] + off)));
    }
    w[g] = acc;
    if (rdot) rw = fma(rdot[g], acc, rw);
  }
  return rw;
}

// The same combination, one CTA per reduction chunk: the chunk's candidate
// subdomains (every overlapped range meeting the chunk, ascending index =
// the reference's accumulation order) are staged in shared memory once, so
// a point costs one range test and one load per covering subdomain.
__global__ void k_combine_chunk(CombineArgs C, const int64_t* __restrict__ cstart,
                                const int32_t* __restrict__ ccand_ptr, const int32_t* __restrict__ ccand,
                                double* __restrict__ w, const DevState* st, const double* __restrict__ rdot,
                                double* __restrict__ part) {
  if (skip(st)) return;
  __shared__ int64_t s_start[COMBINE_MAXC], s_len[COMBINE_MAXC], s_off[COMBINE_MAXC];
  __shared__ double s_w[COMBINE_MAXC];
  const int ch = blockIdx.x;
  const int c0 = ccand_ptr[ch], nc = ccand_ptr[ch + 1] - c0;
  const bool faulty = C.fault != nullptr && *C.apply_calls == C.fault_index;
  if (threadIdx.x < COMBINE_MAXC) {
    const bool on = threadIdx.x < nc;
    const int i = on ? ccand[c0 + threadIdx.x] : 0;
    s_start[threadIdx.x] = on ? C.ov_start[i] : 0;
    // a faulted subdomain contributes nothing in the fault apply
    s_len[threadIdx.x] = (on && !(faulty && C.fault[i])) ? C.ov_len[i] : 0;
    s_off[threadIdx.x] = on ? C.xy_off[i] : 0;
    s_w[threadIdx.x] = on ? C.wgt[i] : 0.0;
  }
  __syncthreads();
  double rw = combine_points(C, s_start, s_len, s_off, s_w, nc, cstart[ch], cstart[ch + 1], w, rdot);
  if (rdot) {  // r.w partials of the fused PCG epilogue (k_coarse_gemv, fin)
    rw = block_sum(rw);
    if (threadIdx.x == 0) part[ch] = rw;
  }
}

// ------------------------------------------------ index-free stencil tiles
// One CTA per tile (tiles.h): own values -> box in shared memory through the
// tile's rank->box table (entries = packed box coordinates), face neighbours
// through the halo rank list, then the stencil in the box.  Same summation
// order as stencil_at (dhat x, then axis 0 -/+, axis 1 -/+, ...; absent
// neighbours skipped): bitwise equal.  PER points per thread, all loads of a
// phase issued before their uses.
template <int D>
__device__ __forceinline__ void tile_coords(uint32_t e, int& u0, int& u1, int& u2) {
  if (D == 3) {
    u0 = e & 31;
    u1 = (e >> 5) & 31;
    u2 = (e >> 10) & 31;
  } else {
    u0 = e & 255;
    u1 = e >> 8;
    u2 = 0;
  }
}

template <int D, int PER, typename Val, typename Epi>
__device__ __forceinline__ void tile_stencil(const Tiles& T, const Stencil& S, int tile, double* Lx, double* H,
                                             Val val, Epi epi) {
  const int r0 = T.r0[tile], np = T.r0[tile + 1] - r0;
  const int n0 = T.dims[3 * tile], n1 = T.dims[3 * tile + 1], n2 = T.dims[3 * tile + 2];
  const uint16_t* tab = T.tab + T.tab_off[tile];
  const int h0 = T.halo_off[tile], nh = T.halo_off[tile + 1] - h0;
  const int32_t* hr = T.halo + h0;
  const int st0 = D == 3 ? n1 * n2 : n1, st1 = D == 3 ? n2 : 1;
  uint32_t e[PER];
  int bl[PER];
  double v[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int k = threadIdx.x + u * VEC_THREADS;
    e[u] = k < np ? __ldg(tab + k) : 0u;
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int k = threadIdx.x + u * VEC_THREADS;
    v[u] = k < np ? val(r0 + k) : 0.0;
  }
  for (int h = threadIdx.x; h < nh; h += VEC_THREADS) {
    const int32_t rk = __ldg(hr + h);
    H[h] = rk >= 0 ? val(rk) : 0.0;
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    int u0, u1, u2;
    tile_coords<D>(e[u], u0, u1, u2);
    bl[u] = u0 * st0 + u1 * st1 + u2;
    if (threadIdx.x + u * VEC_THREADS < np) Lx[bl[u]] = v[u];
  }
  __syncthreads();
  // face f = 2 axis + side; face sizes: axis 0 n1 n2, axis 1 n0 n2, axis 2 n0 n1
  const int fs0 = D == 3 ? n1 * n2 : n1, fs1 = D == 3 ? n0 * n2 : n0, fs2 = D == 3 ? n0 * n1 : 0;
  double acc[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    int u0, u1, u2;
    tile_coords<D>(e[u], u0, u1, u2);
    const int b = bl[u];
    double a = S.dhat * v[u];
    {  // axis 0: face index over (u1[, u2])
      const int fi = D == 3 ? u1 * n2 + u2 : u1;
      if (u0 > 0) a = fma(S.off[0], Lx[b - st0], a);
      else if (__ldg(hr + fi) >= 0) a = fma(S.off[0], H[fi], a);
      if (u0 < n0 - 1) a = fma(S.off[0], Lx[b + st0], a);
      else if (__ldg(hr + fs0 + fi) >= 0) a = fma(S.off[0], H[fs0 + fi], a);
    }
    {  // axis 1: face index over (u0[, u2])
      const int fb = 2 * fs0;
      const int fi = D == 3 ? u0 * n2 + u2 : u0;
      if (u1 > 0) a = fma(S.off[1], Lx[b - st1], a);
      else if (__ldg(hr + fb + fi) >= 0) a = fma(S.off[1], H[fb + fi], a);
      if (u1 < n1 - 1) a = fma(S.off[1], Lx[b + st1], a);
      else if (__ldg(hr + fb + fs1 + fi) >= 0) a = fma(S.off[1], H[fb + fs1 + fi], a);
    }
    if (D == 3) {  // axis 2: face index over (u0, u1)
      const int fb = 2 * fs0 + 2 * fs1;
      const int fi = u0 * n1 + u1;
      if (u2 > 0) a = fma(S.off[2], Lx[b - 1], a);
      else if (__ldg(hr + fb + fi) >= 0) a = fma(S.off[2], H[fb + fi], a);
      if (u2 < n2 - 1) a = fma(S.off[2], Lx[b + 1], a);
      else if (__ldg(hr + fb + fs2 + fi) >= 0) a = fma(S.off[2], H[fb + fs2 + fi], a);
    }
    acc[u] = a;
  }
  epi(r0, np, v, acc);
}

// per-thread points of a tile (PER template argument of the launches)
template <int PER>
__device__ __forceinline__ bool tile_pt(int u, int np) {
  return (int)threadIdx.x + u * VEC_THREADS < np;
}

template <int D, int PER>
__global__ void k_tile_matvec(const double* __restrict__ x, Stencil S, Tiles T, double* __restrict__ y) {
  extern __shared__ double tsm[];
  tile_stencil<D, PER>(T, S, blockIdx.x, tsm, tsm + T.max_points, [&](int64_t i) { return x[i]; },
                       [&](int r0, int np, const double*, const double* acc) {
#pragma unroll
                         for (int u = 0; u < PER; ++u)
                           if (tile_pt<PER>(u, np)) y[r0 + threadIdx.x + u * VEC_THREADS] = acc[u];
                       });
}

// t = g - Â R0^T y0 (k_tvec on tiles)
template <int D, int PER>
__global__ void k_tile_tvec(const double* __restrict__ gv, const double* __restrict__ y0,
                            const int32_t* __restrict__ agg, Stencil S, Tiles T, double* __restrict__ t,
                            const DevState* st) {
  if (skip(st)) return;
  extern __shared__ double tsm[];
  tile_stencil<D, PER>(T, S, blockIdx.x, tsm, tsm + T.max_points, [&](int64_t i) { return __ldg(y0 + agg[i]); },
                       [&](int r0, int np, const double*, const double* acc) {
                         double g[PER];
#pragma unroll
                         for (int u = 0; u < PER; ++u)
                           g[u] = tile_pt<PER>(u, np) ? gv[r0 + threadIdx.x + u * VEC_THREADS] : 0.0;
#pragma unroll
                         for (int u = 0; u < PER; ++u)
                           if (tile_pt<PER>(u, np)) t[r0 + threadIdx.x + u * VEC_THREADS] = g[u] - acc[u];
                       });
}

// p = z + beta p_old with z = (w - R0^T y0b) + R0^T y0, Ap, p.Ap (k_pm_w on tiles)
template <int D, int PER>
__global__ void __launch_bounds__(VEC_THREADS, PER <= 4 ? 7 : 1) k_tile_pm_w(const double* __restrict__ w, const double* __restrict__ y0,
                            const double* __restrict__ y0b, const int32_t* __restrict__ agg,
                            const double* __restrict__ pold, Stencil S, Tiles T, double* __restrict__ pnew,
                            double* __restrict__ ap, double* __restrict__ part, DevState* st) {
  if (skip(st)) return;
  extern __shared__ double tsm[];
  const double beta = st->beta;
  double s = 0.0;
  tile_stencil<D, PER>(
      T, S, blockIdx.x, tsm, tsm + T.max_points,
      [&](int64_t i) {
        const int32_t a = agg[i];
        return __dadd_rn((w[i] - __ldg(y0b + a)) + __ldg(y0 + a), __dmul_rn(beta, pold[i]));
      },
      [&](int r0, int np, const double* pg, const double* acc) {
#pragma unroll
        for (int u = 0; u < PER; ++u)
          if (tile_pt<PER>(u, np)) {
            const int g = r0 + threadIdx.x + u * VEC_THREADS;
            pnew[g] = pg[u];
            ap[g] = acc[u];
            s = fma(pg[u], acc[u], s);
          }
      });
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
  if (last_block(&st->ticket[1])) {
    const double pap = reduce_partials(part, gridDim.x);
    if (threadIdx.x == 0) {
      st->ticket[1] = 0;
      st->pap = pap;
      if (!(pap > 0.0)) {
        st->breakdown = 1;
        st->done = 1;
      } else {
        st->alpha = st->rz / pap;
      }
    }
  }
}

// R0 Â w per (tile, aggregate met) slot (coarse.py:84; aggregates are
// contiguous rank ranges, so a tile's slots are in aggregate order)
template <int D, int PER>
__global__ void k_tile_agg_matvec(const double* __restrict__ w, const int64_t* __restrict__ agg_start,
                                  const int32_t* __restrict__ agg, Stencil S, Tiles T, double* __restrict__ part,
                                  const DevState* sk) {
  if (skip(sk)) return;
  extern __shared__ double tsm[];
  const int tile = blockIdx.x;
  const int r0 = T.r0[tile], np = T.r0[tile + 1] - r0;
  const int a_first = agg[r0], nseg = agg[r0 + np - 1] - a_first + 1;
  int64_t bnd[TILE_MAX_SEGS];  // segment q = ranks [start of a_first+q, start of a_first+q+1)
#pragma unroll
  for (int q = 0; q < TILE_MAX_SEGS; ++q) bnd[q] = q < nseg ? agg_start[a_first + q + 1] : INT64_MAX;
  double loc[TILE_MAX_SEGS];
#pragma unroll
  for (int q = 0; q < TILE_MAX_SEGS; ++q) loc[q] = 0.0;
  tile_stencil<D, PER>(T, S, tile, tsm, tsm + T.max_points, [&](int64_t i) { return w[i]; },
                       [&](int r, int n, const double*, const double* acc) {
#pragma unroll
                         for (int u = 0; u < PER; ++u)
                           if (tile_pt<PER>(u, n)) {
                             const int64_t g = r + threadIdx.x + u * VEC_THREADS;
#pragma unroll
                             for (int q = 0; q < TILE_MAX_SEGS; ++q)
                               if (g < bnd[q] && (q == 0 || g >= bnd[q - 1])) loc[q] += acc[u];
                           }
                       });
  for (int q = 0; q < TILE_MAX_SEGS && q < nseg; ++q) {
    const double v = block_sum(loc[q]);
    if (threadIdx.x == 0) part[T.slot0[tile] + q] = v;
  }
}

// c[a] = sum of aggregate a's tile slots, in tile order
__global__ void k_slot_sums(const double* __restrict__ part, const int32_t* __restrict__ sptr, int32_t n0,
                            double* __restrict__ c, const DevState* sk) {
  if (skip(sk)) return;
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n0) return;
  double v = 0.0;
  for (int q = sptr[a]; q < sptr[a + 1]; ++q) v += __ldcg(part + q);
  c[a] = v;
}

// per-chunk partials of sum (Â w) -> R0 Â w  (coarse.py:84 project_transpose)
__global__ void k_matvec_chunk(const double* __restrict__ w, Stencil S, Chunks C, double* __restrict__ part,
                               const DevState* st) {
  if (skip(st)) return;
  const int ch = blockIdx.x;
  double s = 0.0;
  for (int64_t g = C.start[ch] + threadIdx.x; g < C.start[ch + 1]; g += VEC_THREADS) s += stencil_at(S, w, g);
  s = block_sum(s);
  if (threadIdx.x == 0) part[ch] = s;
}

// h = (w - R0^T y0b) + R0^T y0 (balanced/deflated), w + R0^T y0 (additive),
// w (one-level); optional r.h partials for PCG (krylov.py:288)
__global__ void k_finalize(const double* __restrict__ w, const double* __restrict__ y0,
                           const double* __restrict__ y0b, Chunks C, int mode, double* __restrict__ h,
                           const double* __restrict__ rdot, double* __restrict__ part, DevState* st,
                           bool pcg) {
  if (pcg && skip(st)) return;
  const int ch = blockIdx.x;
  const int a = C.agg ? C.agg[ch] : -1;
  const double c0 = (mode >= 1 && a >= 0) ? y0[a] : 0.0;
  const double c1 = (mode >= 2 && a >= 0) ? y0b[a] : 0.0;
  double s = 0.0;
  const int64_t e1 = C.start[ch + 1];
  for (int64_t b = C.start[ch] + threadIdx.x; b < e1; b += PT * VEC_THREADS) {
    double wv[PT], rv[PT];
#pragma unroll
    for (int u = 0; u < PT; ++u) {
      const int64_t g = b + (int64_t)u * VEC_THREADS;
      const bool ok = g < e1;
      wv[u] = ok ? w[g] : 0.0;
      rv[u] = ok && rdot ? rdot[g] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < PT; ++u) {
      const int64_t g = b + (int64_t)u * VEC_THREADS;
      if (g < e1) {
        double v = wv[u];
        if (mode == 1) v = v + c0;
        if (mode == 2) v = (v - c1) + c0;
        h[g] = v;
        if (rdot) s = fma(rv[u], v, s);
      }
    }
  }
  if (rdot) {
    s = block_sum(s);
    if (threadIdx.x == 0) part[ch] = s;
  }
  if (last_block(&st->ticket[3])) {
    double rz = rdot ? reduce_partials(part, gridDim.x) : 0.0;
    if (threadIdx.x == 0) {
      st->ticket[3] = 0;
      st->apply_calls += 1;
      if (pcg) {
        st->beta = st->have_rz ? rz / st->rz : 0.0;  // krylov.py:289
        st->have_rz = 1;
        st->rz = rz;
      }
    }
  }
}

__global__ void k_matvec(const double* __restrict__ x, Stencil S, double* __restrict__ y) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < S.n) y[g] = stencil_at(S, x, g);
}

// r = b - Â x; ||r||^2 and R0 r partials (krylov.py:267-271)
__global__ void k_residual0(const double* __restrict__ b, const double* __restrict__ x, Stencil S, Chunks C,
                            double* __restrict__ r, double* __restrict__ part_rr,
                            double* __restrict__ part_c, DevState* st, double* hist) {
  const int ch = blockIdx.x;
  double rr = 0.0, cs = 0.0;
  const int64_t c_end = C.start[ch + 1];
  for (int64_t g = C.start[ch] + threadIdx.x; g < c_end; g += VEC_THREADS) {
    const double v = b[g] - stencil_at(S, x, g);
    r[g] = v;
    rr = fma(v, v, rr);
    cs += v;
  }
  rr = block_sum(rr);
  cs = block_sum(cs);
  if (threadIdx.x == 0) {
    part_rr[ch] = rr;
    part_c[ch] = cs;
  }
  if (last_block(&st->ticket[0])) {
    const double tot = reduce_partials(part_rr, gridDim.x);
    if (threadIdx.x == 0) {
      st->ticket[0] = 0;
      const double nrm = sqrt(tot);
      hist[0] = nrm;
      st->hist0 = nrm;
      st->k = 0;
      if (!st->energy_mode && nrm <= st->tol * nrm) {  // krylov.py:268-270 (only for r0 == 0)
        st->converged = 1;
        st->done = 1;
      }
    }
  }
}

// p = z + beta p_old ; Ap = Â p ; p.Ap partials (krylov.py:276-279, 289)
__global__ void k_pm(const double* __restrict__ z, const double* __restrict__ pold, Stencil S, Chunks C,
                     double* __restrict__ pnew, double* __restrict__ ap, double* __restrict__ part,
                     DevState* st) {
  if (skip(st)) return;
  const double beta = st->beta;
  const int ch = blockIdx.x;
  double s = 0.0;
  for (int64_t g = C.start[ch] + threadIdx.x; g < C.start[ch + 1]; g += VEC_THREADS) {
    const double pg = __dadd_rn(z[g], __dmul_rn(beta, pold[g]));
    double acc = S.dhat * pg;
    for (int a = 0; a < 2 * S.d; ++a) {
      const int32_t nb = __ldg(S.nbr + (int64_t)a * S.n + g);
      if (nb >= 0) acc = fma(S.off[a >> 1], __dadd_rn(z[nb], __dmul_rn(beta, pold[nb])), acc);
    }
    pnew[g] = pg;
    ap[g] = acc;
    s = fma(pg, acc, s);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[ch] = s;
  if (last_block(&st->ticket[1])) {
    const double pap = reduce_partials(part, gridDim.x);
    if (threadIdx.x == 0) {
      st->ticket[1] = 0;
      st->pap = pap;
      if (!(pap > 0.0)) {
        st->breakdown = 1;
        st->done = 1;
      } else {
        st->alpha = st->rz / pap;
      }
    }
  }
}

// the same with z = (w - R0^T y0b) + R0^T y0 formed on the fly (fused PCG
// path of the balanced / deflated variants: k_finalize is not launched);
// bitwise the same p and Ap as k_pm over the materialised z
__global__ void k_pm_w(const double* __restrict__ w, const double* __restrict__ y0,
                       const double* __restrict__ y0b, const int32_t* __restrict__ agg,
                       const double* __restrict__ pold, Stencil S, Chunks C, double* __restrict__ pnew,
                       double* __restrict__ ap, double* __restrict__ part, DevState* st) {
  if (skip(st)) return;
  const double beta = st->beta;
  const int ch = blockIdx.x;
  const int a0 = C.agg[ch];
  const double zc = y0[a0], zb = y0b[a0];
  auto zv = [&](int64_t i, double cb, double c0) { return (w[i] - cb) + c0; };
  double s = 0.0;
  for (int64_t g = C.start[ch] + threadIdx.x; g < C.start[ch + 1]; g += VEC_THREADS) {
    const double pg = __dadd_rn(zv(g, zb, zc), __dmul_rn(beta, pold[g]));
    double acc = S.dhat * pg;
    for (int a = 0; a < 2 * S.d; ++a) {
      const int32_t nb = __ldg(S.nbr + (int64_t)a * S.n + g);
      if (nb >= 0) {
        const int32_t an = __ldg(agg + nb);
        acc = fma(S.off[a >> 1], __dadd_rn(zv(nb, __ldg(y0b + an), __ldg(y0 + an)), __dmul_rn(beta, pold[nb])),
                  acc);
      }
    }
    pnew[g] = pg;
    ap[g] = acc;
    s = fma(pg, acc, s);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[ch] = s;
  if (last_block(&st->ticket[1])) {
    const double pap = reduce_partials(part, gridDim.x);
    if (threadIdx.x == 0) {
      st->ticket[1] = 0;
      st->pap = pap;
      if (!(pap > 0.0)) {
        st->breakdown = 1;
        st->done = 1;
      } else {
        st->alpha = st->rz / pap;
      }
    }
  }
}

// x += alpha p ; r -= alpha Ap ; ||r|| -> history ; R0 r partials
__global__ void __launch_bounds__(VEC_THREADS, 7) k_update(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                         const double* __restrict__ ap, Chunks C, double* __restrict__ part_rr,
                         double* __restrict__ part_c, DevState* st, double* hist) {
  if (skip(st)) return;
  const double alpha = st->alpha;
  const int ch = blockIdx.x;
  const int64_t c0 = C.start[ch], c1 = C.start[ch + 1];
  double rr = 0.0, cs = 0.0;
  for (int64_t b = c0 + threadIdx.x; b < c1; b += PT * VEC_THREADS) {
    double xv[PT], pv[PT], rv[PT], av[PT];
#pragma unroll
    for (int u = 0; u < PT; ++u) {
      const int64_t g = b + (int64_t)u * VEC_THREADS;
      const bool ok = g < c1;
      xv[u] = ok ? x[g] : 0.0;
      pv[u] = ok ? p[g] : 0.0;
      rv[u] = ok ? r[g] : 0.0;
      av[u] = ok ? ap[g] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < PT; ++u) {
      const int64_t g = b + (int64_t)u * VEC_THREADS;
      if (g < c1) {
        x[g] = __dadd_rn(xv[u], __dmul_rn(alpha, pv[u]));
        const double v = __dsub_rn(rv[u], __dmul_rn(alpha, av[u]));
        r[g] = v;
        rr = fma(v, v, rr);
        cs += v;
      }
    }
  }
  const double2 red = block_sum2(rr, cs);
  if (threadIdx.x == 0) {
    part_rr[ch] = red.x;
    part_c[ch] = red.y;
  }
  if (last_block(&st->ticket[2])) {
    const double tot = reduce_partials(part_rr, gridDim.x);
    if (threadIdx.x == 0) {
      st->ticket[2] = 0;
      const int k = st->k + 1;
      st->k = k;
      const double nrm = sqrt(tot);
      hist[k] = nrm;
      if (!st->energy_mode) {  // else k_energy decides (after the energy error is known)
        bool stop = false;
        if (nrm <= st->tol * st->hist0) {  // krylov.py:283-286
          st->converged = 1;
          stop = true;
        } else if (k >= st->max_iters) {
          st->exhausted = 1;
          stop = true;
        }
        // with energy tracking the reference still records the energy error
        // of this last iterate (krylov.py:186-200): k_energy turns the
        // pending stop into done after writing ehist[k]
        if (stop) {
          if (st->track_energy)
            st->stop_pending = 1;
          else
            st->done = 1;
        }
      }
    }
  }
}

// energy error of iterate k: ||x - x*||_A = sqrt(max(e.(b - r - A x*), 0)),
// e = x - x* (krylov.py:189-193: A e = (b - r) - A x* needs no matvec); with
// energy stopping it decides convergence / exhaustion (krylov.py:194-200)
__global__ void k_energy(const double* __restrict__ x, const double* __restrict__ ex,
                         const double* __restrict__ b, const double* __restrict__ r,
                         const double* __restrict__ aex, Chunks C, double* __restrict__ part, DevState* st,
                         double* ehist, bool initial) {
  if (!initial && skip(st)) return;
  const int ch = blockIdx.x;
  const int64_t c1 = C.start[ch + 1];
  double s = 0.0;
  for (int64_t g = C.start[ch] + threadIdx.x; g < c1; g += VEC_THREADS)
    s = fma(__dsub_rn(x[g], ex[g]), __dsub_rn(__dsub_rn(b[g], r[g]), aex[g]), s);
  s = block_sum(s);
  if (threadIdx.x == 0) part[ch] = s;
  if (last_block(&st->ticket[4])) {
    const double tot = reduce_partials(part, gridDim.x);
    if (threadIdx.x == 0) {
      st->ticket[4] = 0;
      const int k = st->k;
      const double en = sqrt(fmax(tot, 0.0));
      ehist[k] = en;
      if (initial) st->ehist0 = en;
      if (st->energy_mode && !st->breakdown) {
        if (en <= st->tol * st->ehist0) {
          st->converged = 1;
          st->done = 1;
        } else if (!initial && k >= st->max_iters) {
          st->exhausted = 1;
          st->done = 1;
        }
      }
      if (st->stop_pending) {  // k_update's residual stop of this iteration
        st->stop_pending = 0;
        st->done = 1;
      }
    }
  }
}

__global__ void k_zero_state_pcg(DevState* st, double tol, int32_t max_iters, int32_t track_energy,
                                 int32_t energy_mode) {
  st->track_energy = track_energy;
  st->energy_mode = energy_mode;
  st->ehist0 = 0;
  st->tol = tol;
  st->hist0 = 0;
  st->rz = st->beta = st->pap = st->alpha = 0;
  st->k = st->converged = st->breakdown = st->exhausted = st->have_rz = st->done = st->stop_pending = 0;
  st->max_iters = max_iters;
  st->apply_calls = 0;  // fault mode counts preconditioner calls per solve
  for (int i = 0; i < 8; ++i) st->ticket[i] = 0;
}

}  // namespace

// ----------------------------------------------------------- host helpers
static Stencil stencil_of(const sfcdd_op* op) {
  Stencil S;
  S.d = op->d;
  S.n = op->n;
  S.dhat = op->dhat;
  for (int j = 0; j < MAX_GRID_DIM; ++j) S.off[j] = j < op->d ? op->off[j] : 0.0;
  S.nbr = op->nbr;
  return S;
}

static Chunks chunks_of(const sfcdd_op* op) {
  return Chunks{op->chunk_start, op->n0 > 0 ? op->chunk_agg : nullptr, op->agg_ptr, op->nch};
}

static void* dev_alloc(sfcdd_op* op, size_t bytes) {
  void* p = nullptr;
  CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
  op->dev_bytes += std::max<size_t>(bytes, 16);
  return p;
}

template <typename T>
static T* dev_upload(sfcdd_op* op, const std::vector<T>& v) {
  T* p = (T*)dev_alloc(op, v.size() * sizeof(T));
  if (!v.empty()) CUDA_CHECK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

// optional per-kernel timing (sfcdd_op_profile with SFCDD_PROFILE_KERNELS=1):
// an event after every launch of apply_device / pcg_iteration
struct KernelTimer {
  std::vector<cudaEvent_t> ev;
  std::vector<const char*> name;
  std::vector<double> ms;
  size_t idx = 0;
};
static KernelTimer* g_ktimer = nullptr;
static void kmark(cudaStream_t st, const char* name) {
  KernelTimer* k = g_ktimer;
  if (!k) return;
  if (k->idx == k->ev.size()) {
    cudaEvent_t e;
    CUDA_CHECK(cudaEventCreate(&e));
    k->ev.push_back(e);
    k->name.push_back(name);
    k->ms.push_back(0.0);
  }
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CUDA_CHECK(cudaStreamIsCapturing(st, &cap));
  if (cap == cudaStreamCaptureStatusActive)  // an event-record node of the graph
    CUDA_CHECK(cudaEventRecordWithFlags(k->ev[k->idx], st, cudaEventRecordExternal));
  else
    CUDA_CHECK(cudaEventRecord(k->ev[k->idx], st));
  k->name[k->idx] = name;
  ++k->idx;
}

static int mode_of(int variant) {
  switch (variant) {
    case SFCDD_VARIANT_ONE_LEVEL: return 0;
    case SFCDD_VARIANT_ADDITIVE: return 1;
    default: return 2;
  }
}

// stencil-tile launches (d = 2 or 3)
#define TILE_LAUNCH(KERNEL, OP, ST, ...)                                                                  \
  do {                                                                                                   \
    const size_t smem_ = (size_t)(OP)->tiles.smem_doubles * 8;                                           \
    const int per_ = ((OP)->tiles.max_points + VEC_THREADS - 1) / VEC_THREADS;                           \
    const unsigned g_ = (unsigned)(OP)->tiles.ntiles;                                                    \
    if ((OP)->d == 2 && per_ <= 4)                                                                        \
      KERNEL<2, 4><<<g_, VEC_THREADS, smem_, ST>>>(__VA_ARGS__);                                         \
    else if ((OP)->d == 2)                                                                                \
      KERNEL<2, 16><<<g_, VEC_THREADS, smem_, ST>>>(__VA_ARGS__);                                        \
    else if (per_ <= 2)                                                                                   \
      KERNEL<3, 2><<<g_, VEC_THREADS, smem_, ST>>>(__VA_ARGS__);                                         \
    else                                                                                                  \
      KERNEL<3, 16><<<g_, VEC_THREADS, smem_, ST>>>(__VA_ARGS__);                                        \
  } while (0)

static void launch_matvec(sfcdd_op* op, const double* x, double* y, cudaStream_t st) {
  if (op->tiled)
    TILE_LAUNCH(k_tile_matvec, op, st, x, stencil_of(op), op->tiles, y);
  else
    k_matvec<<<nblocks(op->n, VEC_THREADS), VEC_THREADS, 0, st>>>(x, stencil_of(op), y);
}

static CombineArgs combine_args(sfcdd_op* op) {
  CombineArgs ca;
  ca.xy = op->dag->xy();
  ca.ov_start = op->d_ov_start;
  ca.ov_len = op->d_ov_len;
  ca.xy_off = op->d_xy_off;
  ca.dj_start = op->d_dj_start;
  ca.cand_ptr = op->cand_ptr;
  ca.cand = op->cand;
  ca.wgt = op->d_wgt;
  ca.count = op->weighting == SFCDD_WEIGHT_DMATRIX ? op->d_count : nullptr;
  ca.fault = op->d_fault;
  ca.apply_calls = &op->st->apply_calls;
  ca.fault_index = op->stats.reserved[0];
  ca.p = op->p;
  ca.n = op->n;
  return ca;
}

// y = A0^{-1} c, c[a] = sum of part[ptr[a]] .. part[ptr[a+1]-1] (ptr ignored
// when `direct`: c = part).  Dense redundant inverse (GEMV) up to
// COARSE_DENSE_MAX coarse DOFs, else the sparse supernodal factor of A0
// through its own DAG solve; optional fused PCG epilogue (fin).
static void coarse_solve(sfcdd_op* op, const double* part, const int32_t* ptr, bool direct, double* y,
                         const DevState* sk, const PcgFin& fin, cudaStream_t st) {
  if (op->ainv) {
    const size_t csm = direct ? 0 : (size_t)op->n0 * sizeof(double);
    k_coarse_gemv<<<nblocks(op->n0, GEMV_ROWS), VEC_THREADS, csm, st>>>(op->ainv, part, ptr, op->n0, y, sk, direct,
                                                                       fin);
    return;
  }
  const double* c = part;
  if (!direct) {
    k_seg_sum<<<nblocks(op->n0, VEC_THREADS), VEC_THREADS, 0, st>>>(part, ptr, op->n0, op->cvec0, sk);
    c = op->cvec0;
  }
  op->coarse_dag->solve(c, st, sk ? &op->st->done : nullptr);
  k_coarse_out<<<nblocks(op->n0, VEC_THREADS), VEC_THREADS, 0, st>>>(op->coarse_dag->xy(), op->n0, y, sk, fin);
}

// kernel launches of coarse_solve / apply_device (the gpu_launches accounting
// of sfcdd_op_pcg_ex and sfcdd_op_profile; keep in step with those functions)
static int64_t coarse_solve_launches(const sfcdd_op* op, bool direct) {
  return op->ainv ? 1 : (direct ? 0 : 1) + 1 + 1;  // GEMV | [segment sums] + DAG + output
}
// the tile-slot sums of R0 Â w ride in the second coarse GEMV (dense inverse, few aggregates)
static bool slot_sums_fused(const sfcdd_op* op) { return op->ainv != nullptr && op->n0 <= 2048; }

static int64_t apply_launches(const sfcdd_op* op, bool pcg, bool partials_ready) {
  const int v = op->variant;
  const bool direct = op->nch == op->n0;
  int64_t k = 0;
  if (v != SFCDD_VARIANT_ONE_LEVEL) k += (partials_ready ? 0 : 1) + coarse_solve_launches(op, direct);
  if (v == SFCDD_VARIANT_BALANCED) k += 1;  // t
  k += 1 + 1;                               // DAG + combine
  if (mode_of(v) == 2)
    k += op->tile_agg ? (slot_sums_fused(op) ? 1 : 2) + coarse_solve_launches(op, true)
                      : 1 + coarse_solve_launches(op, direct);
  if (!(pcg && mode_of(v) == 2)) k += 1;    // finalize
  return k;
}

// the preconditioner apply on device: h = C^{-1} g.  If `pcg`, the R0 g
// partials are already in part_c (fused into k_update) and r.h partials are
// produced for the PCG scalars.
static void apply_device(sfcdd_op* op, const double* g, double* h, cudaStream_t st, bool pcg,
                         bool partials_ready) {
  const Stencil S = stencil_of(op);
  const Chunks C = chunks_of(op);
  DevState* dst = op->st;
  const DevState* sk = pcg ? op->st : nullptr;
  const int v = op->variant;
  const bool coarse = v != SFCDD_VARIANT_ONE_LEVEL;
  const bool direct = op->nch == op->n0;  // one chunk per aggregate: c = partials
  if (coarse) {
    if (!partials_ready) k_chunk_sum<<<op->nch, VEC_THREADS, 0, st>>>(g, C, op->part_c);
    if (!partials_ready) kmark(st, "chunk_sum");
    coarse_solve(op, op->part_c, op->agg_ptr, direct, op->y0, sk, PcgFin{}, st);
    kmark(st, "coarse_gemv");
  }
  const double* rhs = g;
  if (v == SFCDD_VARIANT_BALANCED) {
    if (op->tiled)
      TILE_LAUNCH(k_tile_tvec, op, st, g, op->y0, op->agg, S, op->tiles, op->t, sk);
    else
      k_tvec<<<nblocks(op->n, VEC_THREADS), VEC_THREADS, 0, st>>>(g, op->y0, op->agg, S, op->t, sk);
    kmark(st, "tvec");
    rhs = op->t;
  }
  op->dag->solve(rhs, st, sk ? &op->st->done : nullptr);
  kmark(st, "dag");
  const CombineArgs ca = combine_args(op);
  const int mode = mode_of(v);
  // PCG with a two-sided coarse correction: z is never materialised; r.z and
  // beta come from the second GEMV's epilogue and k_pm_w forms z on the fly
  const bool fused = pcg && mode == 2;
  k_combine_chunk<<<op->nch, VEC_THREADS, 0, st>>>(ca, op->chunk_start, op->ccand_ptr, op->ccand, op->w, sk,
                                                   fused ? op->r : nullptr, op->part_a);
  kmark(st, "combine");
  if (mode == 2) {
    PcgFin fin{op->part_a, op->part_c, op->y0, op->nch, fused ? dst : nullptr, op->agg_ptr, direct};
    if (op->tile_agg) {  // c = R0 Â w per aggregate from the tile slots
      TILE_LAUNCH(k_tile_agg_matvec, op, st, op->w, op->d_agg_start, op->agg, S, op->tiles, op->part_t, sk);
      if (slot_sums_fused(op)) {
        // small dense coarse problems: every GEMV CTA sums the slots itself (same order
        // as k_slot_sums: bitwise equal), one launch less on the iteration's critical path
        kmark(st, "matvec_chunk");
        coarse_solve(op, op->part_t, op->tiles.sptr, false, op->y0b, sk, fin, st);
      } else {
        k_slot_sums<<<nblocks(op->n0, VEC_THREADS), VEC_THREADS, 0, st>>>(op->part_t, op->tiles.sptr, op->n0,
                                                                         op->cvec, sk);
        kmark(st, "matvec_chunk");
        coarse_solve(op, op->cvec, op->agg_ptr, true, op->y0b, sk, fin, st);
      }
    } else {
      k_matvec_chunk<<<op->nch, VEC_THREADS, 0, st>>>(op->w, S, C, op->part_b, sk);
      kmark(st, "matvec_chunk");
      coarse_solve(op, op->part_b, op->agg_ptr, direct, op->y0b, sk, fin, st);
    }
    kmark(st, "coarse_gemv2");
  }
  if (!fused) {
    k_finalize<<<op->nch, VEC_THREADS, 0, st>>>(op->w, op->y0, op->y0b, C, mode, h, pcg ? op->r : nullptr,
                                                op->part_a, dst, pcg);
    kmark(st, "finalize");
  }
  CUDA_CHECK(cudaGetLastError());
}

// one PCG iteration (krylov.py:275-290) -- captured into a CUDA graph
static void pcg_iteration(sfcdd_op* op, double* x, const double* pold, double* pnew, cudaStream_t st) {
  const Stencil S = stencil_of(op);
  const Chunks C = chunks_of(op);
  if (mode_of(op->variant) == 2 && op->tiled)
    TILE_LAUNCH(k_tile_pm_w, op, st, op->w, op->y0, op->y0b, op->agg, pold, S, op->tiles, pnew, op->ap, op->part_t,
                op->st);
  else if (mode_of(op->variant) == 2)
    k_pm_w<<<op->nch, VEC_THREADS, 0, st>>>(op->w, op->y0, op->y0b, op->agg, pold, S, C, pnew, op->ap, op->part_a,
                                            op->st);
  else
    k_pm<<<op->nch, VEC_THREADS, 0, st>>>(op->z, pold, S, C, pnew, op->ap, op->part_a, op->st);
  kmark(st, "pm");
  k_update<<<op->nch, VEC_THREADS, 0, st>>>(x, op->r, pnew, op->ap, C, op->part_b, op->part_c, op->st,
                                            op->hist);
  kmark(st, "update");
  if (op->pcg_exact)
    k_energy<<<op->nch, VEC_THREADS, 0, st>>>(x, op->pcg_exact, op->pcg_b, op->r, op->aex, C, op->part_e, op->st,
                                              op->ehist, false);
  apply_device(op, op->r, op->z, st, true, true);
}

// Numeric factorization of the local blocks with their values placed into
// the deferred-value DAG plan.  Host path: multifrontal Cholesky per block on
// host threads, each block's packed values streamed to the device and placed
// by the plan's value descriptors as soon as it is done (host memory holds a
// few blocks' values at a time).
template <class BlockFn>
void numeric_factor_blocks_host(sfcdd_op* op, std::vector<HostFactor>& fs, int32_t sf, BlockFn&& local_block) {
  const int64_t nf = (int64_t)fs.size();
  int64_t max_stored = 1;
  for (const HostFactor& F : fs) max_stored = std::max(max_stored, F.stored);
  const int threads = (int)std::max<int64_t>(1, std::min<int64_t>(op->threads, nf));
  std::vector<double*> stage(threads, nullptr);
  std::vector<cudaStream_t> streams(threads, nullptr);
  for (int t = 0; t < threads; ++t) {
    CUDA_CHECK(cudaMalloc(&stage[t], max_stored * 8));
    CUDA_CHECK(cudaStreamCreateWithFlags(&streams[t], cudaStreamNonBlocking));
  }
  std::atomic<int64_t> next{0};
  std::exception_ptr err;
  std::mutex mu;
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t]() {
      try {
        CUDA_CHECK(cudaSetDevice(op->device));
        for (;;) {
          const int64_t li = next.fetch_add(1);
          if (li >= nf) return;
          HostFactor& F = fs[li];
          numeric_host(local_block(sf + li), F);
          CUDA_CHECK(cudaMemcpyAsync(stage[t], F.val.data(), F.stored * 8, cudaMemcpyHostToDevice, streams[t]));
          const int64_t base = 0;
          op->dag->place_values((int32_t)li, (int32_t)li + 1, stage[t], &base, streams[t]);
          CUDA_CHECK(cudaStreamSynchronize(streams[t]));
          std::vector<double>().swap(F.val);
        }
      } catch (...) {
        std::lock_guard<std::mutex> g(mu);
        if (!err) err = std::current_exception();
        next = nf;
      }
    });
  for (auto& th : pool) th.join();
  for (int t = 0; t < threads; ++t) {
    cudaFree(stage[t]);
    cudaStreamDestroy(streams[t]);
  }
  if (err) std::rethrow_exception(err);
}

// Device path (default): batches of blocks, sized to the free device memory,
// factorized by gpu_factor_batch straight into a device value buffer that
// place_values moves into the blobs.  SFCDD_HOST_NUMERIC=1 selects the host
// path (A/B comparisons).
template <class BlockFn>
void numeric_factor_blocks_device(sfcdd_op* op, std::vector<HostFactor>& fs, int32_t sf, BlockFn&& local_block) {
  const int64_t nf = (int64_t)fs.size();
  size_t free_b = 0, total_b = 0;
  CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
  int64_t budget = std::min<int64_t>((int64_t)(0.6 * (double)free_b), int64_t(48) << 30);
  if (const char* e = std::getenv("SFCDD_FACTOR_BUDGET_GB")) budget = (int64_t)(std::atof(e) * (1 << 30));
  cudaStream_t st = op->own_stream;
  double dev_s = 0.0;
  int64_t f0 = 0;
  while (f0 < nf) {
    // batch [f0, f1): values + update matrices + tier-3 workspace within budget
    int64_t f1 = f0, need = 0;
    while (f1 < nf) {
      const HostFactor& F = fs[f1];
      const int64_t b = 8 * (F.stored + gpu_factor_update_doubles(F) + gpu_factor_work_bound(F)) + 64 * (int64_t)F.sn.size();
      if (f1 > f0 && need + b > budget) break;
      need += b;
      ++f1;
    }
    std::vector<GpuFactorInput> in(f1 - f0);
    parallel_for(f1 - f0, op->threads,
                 [&](int64_t i) { gpu_factor_prepare(fs[f0 + i], local_block(sf + f0 + i), in[i]); });
    std::vector<const HostFactor*> fp;
    std::vector<const GpuFactorInput*> ip;
    std::vector<int64_t> base;
    int64_t tot = 0;
    for (int64_t i = f0; i < f1; ++i) {
      fp.push_back(&fs[i]);
      ip.push_back(&in[i - f0]);
      base.push_back(tot);
      tot += fs[i].stored;
    }
    double* vals = nullptr;
    CUDA_CHECK(cudaMallocAsync(&vals, std::max<int64_t>(tot, 2) * 8, st));
    try {
      gpu_factor_batch(fp, ip, vals, base, st, &dev_s);
      op->dag->place_values((int32_t)f0, (int32_t)f1, vals, base.data(), st);
      CUDA_CHECK(cudaFreeAsync(vals, st));
      CUDA_CHECK(cudaStreamSynchronize(st));
    } catch (...) {
      cudaFreeAsync(vals, st);
      cudaStreamSynchronize(st);
      throw;
    }
    f0 = f1;
  }
  op->stats.reserved[6] = (int64_t)(1e6 * dev_s);  // device factorization time (us)
}

template <class BlockFn>
void numeric_factor_blocks(sfcdd_op* op, std::vector<HostFactor>& fs, int32_t sf, BlockFn&& local_block) {
  const char* e = std::getenv("SFCDD_HOST_NUMERIC");
  if (e && std::atoi(e) != 0)
    numeric_factor_blocks_host(op, fs, sf, local_block);
  else
    numeric_factor_blocks_device(op, fs, sf, local_block);
}

OpScope::OpScope(sfcdd_op* op, cudaStream_t caller) : op_(op), caller_(caller), lk_(op->mu) {
  CUDA_CHECK(cudaEventRecord(op->ev_in, caller));
  CUDA_CHECK(cudaStreamWaitEvent(op->own_stream, op->ev_in, 0));
}

OpScope::~OpScope() noexcept(false) {
  // the caller's stream resumes after the handle's work (also on the error
  // path, so a failed call never leaves the caller unordered)
  cudaError_t e1 = cudaEventRecord(op_->ev_out, op_->own_stream);
  cudaError_t e2 = cudaStreamWaitEvent(caller_, op_->ev_out, 0);
  if (!std::uncaught_exceptions()) {
    CUDA_CHECK(e1);
    CUDA_CHECK(e2);
  }
}

}  // namespace sfcdd

using namespace sfcdd;

// ================================================================ C ABI
extern "C" int sfcdd_op_create(const sfcdd_op_desc* desc, sfcdd_op** out) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(desc && out, SFCDD_EVALUE, "null argument");
  std::unique_ptr<sfcdd_op> op(new sfcdd_op());
  op->device = desc->device;
  op->d = desc->dim;
  SFCDD_REQUIRE(op->d >= 1 && op->d <= 8, SFCDD_EVALUE, "grid dimension must be in [1, 8]");
  op->n = 1;
  double diag = 0.0;
  for (int j = 0; j < op->d; ++j) {
    op->levels[j] = desc->levels[j];
    SFCDD_REQUIRE(desc->levels[j] >= 1 && desc->levels[j] <= 31, SFCDD_EVALUE, "level out of range");
    const int64_t s = ((int64_t)1 << desc->levels[j]) - 1;
    SFCDD_REQUIRE(op->n <= ((int64_t)1 << 62) / s, SFCDD_EOVERFLOW, "dof count exceeds 2^62");
    op->n *= s;
    diag = diag + 2.0 * std::ldexp(1.0, 2 * desc->levels[j]);  // kron-sum diagonal (grid.py:101-110)
  }
  SFCDD_REQUIRE(desc->raw_laplacian == 0 || desc->raw_laplacian == 1, SFCDD_EVALUE, "raw_laplacian must be 0 or 1");
  SFCDD_REQUIRE(op->n < ((int64_t)1 << 31), SFCDD_EVALUE, "grids above 2^31 points need multi-GPU sharding");
  // T A T with t = diag^-1/2 (grid.py:117-130): entries fl(fl(t a) t)
  const double t = 1.0 / std::sqrt(diag);
  op->tscale = t;
  op->raw = desc->raw_laplacian;
  if (op->raw) {  // unscaled A: exact integer entries 2 sum 4^l and -4^l_j
    op->dhat = diag;
    for (int j = 0; j < op->d; ++j) op->off[j] = -std::ldexp(1.0, 2 * desc->levels[j]);
  } else {
    op->dhat = (t * diag) * t;
    for (int j = 0; j < op->d; ++j) op->off[j] = (t * -std::ldexp(1.0, 2 * desc->levels[j])) * t;
  }
  op->p = desc->p;
  op->q = desc->q;
  op->variant = desc->variant;
  op->weighting = desc->weighting;
  op->threads = desc->host_threads > 0 ? desc->host_threads : hardware_threads();
  op->shard_first = desc->shard_first;
  op->shard_count = desc->shard_count;
  op->curve = desc->curve;
  SFCDD_REQUIRE(op->curve == 0 || op->curve == 1, SFCDD_EVALUE, "unknown curve");
  if (op->shard_count > 0)
    SFCDD_REQUIRE(desc->shard_first >= 0 && desc->shard_first + desc->shard_count <= desc->p && desc->q >= 1,
                  SFCDD_EVALUE, "invalid shard (needs a coarse space and owned subdomains within [0, P))");
  SFCDD_REQUIRE(op->p >= 1 && op->p <= op->n, SFCDD_EVALUE, "need 1 <= P <= N");
  SFCDD_REQUIRE(op->variant >= 0 && op->variant <= 3, SFCDD_EVALUE, "unknown variant");
  SFCDD_REQUIRE(op->weighting >= 0 && op->weighting <= 2, SFCDD_EVALUE, "unknown weighting");
  const bool coarse = op->variant != SFCDD_VARIANT_ONE_LEVEL;
  if (coarse) SFCDD_REQUIRE(op->q >= 1 && op->q <= op->n / op->p, SFCDD_EVALUE, "need 1 <= q <= floor(N/P)");
  if (desc->ov_start) {
    SFCDD_REQUIRE(desc->ov_len && desc->dj_start && desc->dj_len, SFCDD_EVALUE, "incomplete ranges");
    op->ov_start.assign(desc->ov_start, desc->ov_start + op->p);
    op->ov_len.assign(desc->ov_len, desc->ov_len + op->p);
    op->dj_start.assign(desc->dj_start, desc->dj_start + op->p);
    op->dj_len.assign(desc->dj_len, desc->dj_len + op->p);
  } else {  // the library's own partition (partition.py:130-133)
    partition_ranges(op->n, op->p, desc->gamma_num, desc->gamma_den, op->dj_start, op->dj_len, op->ov_start,
                     op->ov_len);
  }
  if (desc->omega) {
    op->omega.assign(desc->omega, desc->omega + op->p);
  } else {  // partition.py:151-157
    op->omega.resize(op->p);
    partition_weights(op->n, op->p, op->ov_start.data(), op->ov_len.data(), nullptr, op->omega.data());
  }
  int64_t acc = 0;
  for (int i = 0; i < op->p; ++i) {
    SFCDD_REQUIRE(op->dj_start[i] == acc, SFCDD_EVALUE, "disjoint ranges must tile [0, N) in order");
    acc += op->dj_len[i];
    SFCDD_REQUIRE(op->ov_start[i] >= 0 && op->ov_start[i] < op->n && op->ov_len[i] >= 1 &&
                      op->ov_len[i] <= op->n,
                  SFCDD_EVALUE, "overlapped range out of bounds");
  }
  SFCDD_REQUIRE(acc == op->n, SFCDD_EVALUE, "disjoint ranges must cover N");

  CUDA_CHECK(cudaSetDevice(op->device));
  CUDA_CHECK(cudaStreamCreateWithFlags(&op->own_stream, cudaStreamNonBlocking));
  CUDA_CHECK(cudaEventCreate(&op->ev0));
  CUDA_CHECK(cudaEventCreate(&op->ev1));
  CUDA_CHECK(cudaEventCreateWithFlags(&op->ev_in, cudaEventDisableTiming));
  CUDA_CHECK(cudaEventCreateWithFlags(&op->ev_out, cudaEventDisableTiming));
  cudaStream_t st = op->own_stream;
  // SFC permutation and neighbour table
  int64_t* perm = (int64_t*)dev_alloc(op.get(), op->n * 8);
  int64_t* rank = (int64_t*)dev_alloc(op.get(), op->n * 8);
  sfc_perm_device(op->d, op->levels, perm, rank, false, st, op->curve);
  GridGeom g{};
  g.d = op->d;
  g.n = op->n;
  for (int j = 0; j < op->d; ++j) g.shape[j] = ((int64_t)1 << op->levels[j]) - 1;
  op->nbr = (int32_t*)dev_alloc(op.get(), (size_t)2 * op->d * op->n * 4);
  k_nbr<<<nblocks(op->n, 256), 256, 0, st>>>(g, perm, rank, op->nbr);
  CUDA_CHECK(cudaGetLastError());
  CUDA_CHECK(cudaStreamSynchronize(st));
  // stencil tiles (2-D / 3-D, single-GPU operator; SFCDD_NO_TILES=1 keeps the
  // neighbour-table kernels)
  std::vector<int64_t> perm_host;
  if ((op->d == 2 || op->d == 3) && op->shard_count == 0 && !std::getenv("SFCDD_NO_TILES")) {
    perm_host.resize(op->n);
    CUDA_CHECK(cudaMemcpy(perm_host.data(), perm, op->n * 8, cudaMemcpyDeviceToHost));
  }
  CUDA_CHECK(cudaFree(perm));
  CUDA_CHECK(cudaFree(rank));
  op->dev_bytes -= 2 * std::max<int64_t>(op->n * 8, 16);
  // aggregates (coarse.py:44-55) and reduction chunks
  std::vector<int64_t> cstart{0};
  std::vector<int32_t> cagg, aptr{0};
  if (coarse) {
    op->n0 = op->q * op->p;
    op->agg_start.assign(1, 0);
    for (int i = 0; i < op->p; ++i) {
      const int64_t base = op->dj_len[i] / op->q, extra = op->dj_len[i] % op->q;
      for (int mm = 0; mm < op->q; ++mm) op->agg_start.push_back(op->agg_start.back() + base + (mm < extra));
    }
    for (int32_t a = 0; a < op->n0; ++a) {
      for (int64_t s0 = op->agg_start[a]; s0 < op->agg_start[a + 1]; s0 += CHUNK) {
        cstart.push_back(std::min<int64_t>(s0 + CHUNK, op->agg_start[a + 1]));
        cagg.push_back(a);
      }
      aptr.push_back((int32_t)cagg.size());
    }
    op->agg = (int32_t*)dev_alloc(op.get(), op->n * 4);
    int64_t* das = dev_upload(op.get(), op->agg_start);
    k_fill_agg<<<op->n0, 256, 0, st>>>(das, op->n0, op->agg);
    CUDA_CHECK(cudaStreamSynchronize(st));
    CUDA_CHECK(cudaFree(das));
  } else {
    // one-level: chunks never cross a disjoint range, so the subdomains
    // meeting one chunk are those covering one owner's points (a fixed
    // 2048-point grid would meet > COMBINE_MAXC ranges for tiny subdomains)
    for (int i = 0; i < op->p; ++i) {
      const int64_t e = op->dj_start[i] + op->dj_len[i];
      for (int64_t s0 = op->dj_start[i]; s0 < e; s0 += CHUNK) {
        cstart.push_back(std::min<int64_t>(s0 + CHUNK, e));
        cagg.push_back(-1);
      }
    }
  }
  op->nch = (int32_t)cagg.size();
  op->chunk_start = dev_upload(op.get(), cstart);
  op->chunk_agg = dev_upload(op.get(), cagg);
  op->agg_ptr = dev_upload(op.get(), aptr);
  HostTiles ht;
  if (!perm_host.empty()) {
    int lshift[MAX_GRID_DIM];
    int lmax = 0;
    for (int j = 0; j < op->d; ++j) lmax = std::max(lmax, op->levels[j]);
    for (int j = 0; j < op->d; ++j) lshift[j] = lmax - op->levels[j];
    try {
      ht = build_tiles(op->d, g.shape, lshift, perm_host);
    } catch (const Error&) {
      // blocks the packed tile tables cannot describe (e.g. grids of extreme
      // anisotropy such as levels (1, 11)): keep the neighbour-table stencil
      ht.ntiles = 0;
    }
    perm_host.clear();
    perm_host.shrink_to_fit();
  }
  if (ht.ntiles > 0) {
    // R0 Â w slots: one per (tile, aggregate met), in rank order
    std::vector<int32_t> slot0{0}, sptr;
    int max_seg = 0;
    if (coarse) {
      sptr.assign(op->n0 + 1, 0);
      for (int32_t t = 0; t < ht.ntiles; ++t) {
        const int64_t a = ht.r0[t], b = ht.r0[t + 1] - 1;  // first/last rank of the tile
        const int32_t fa = (int32_t)(std::upper_bound(op->agg_start.begin(), op->agg_start.end(), a) -
                                     op->agg_start.begin()) - 1;
        const int32_t la = (int32_t)(std::upper_bound(op->agg_start.begin(), op->agg_start.end(), b) -
                                     op->agg_start.begin()) - 1;
        max_seg = std::max(max_seg, la - fa + 1);
        for (int32_t q = fa; q <= la; ++q) ++sptr[q + 1];
        slot0.push_back(slot0.back() + (la - fa + 1));
      }
      for (int32_t q = 0; q < op->n0; ++q) sptr[q + 1] += sptr[q];
    }
    Tiles& T = op->tiles;
    T.d = op->d;
    T.ntiles = ht.ntiles;
    T.r0 = dev_upload(op.get(), ht.r0);
    T.dims = dev_upload(op.get(), ht.dims);
    T.tab_off = dev_upload(op.get(), ht.tab_off);
    T.tab = dev_upload(op.get(), ht.tab);
    T.halo_off = dev_upload(op.get(), ht.halo_off);
    T.halo = dev_upload(op.get(), ht.halo);
    int32_t maxp = 0;
    for (int32_t t = 0; t < ht.ntiles; ++t) maxp = std::max(maxp, ht.r0[t + 1] - ht.r0[t]);
    T.max_points = maxp;
    T.smem_doubles = maxp + ht.max_halo;
    op->tiled = true;
    op->tile_agg = coarse && max_seg <= TILE_MAX_SEGS;
    if (op->tile_agg) {
      T.slot0 = dev_upload(op.get(), slot0);
      T.sptr = dev_upload(op.get(), sptr);
      op->cvec = (double*)dev_alloc(op.get(), (size_t)op->n0 * 8);
      op->d_agg_start = dev_upload(op.get(), op->agg_start);
    }
    op->part_t = (double*)dev_alloc(op.get(), (size_t)std::max<int64_t>(slot0.back(), ht.ntiles) * 8);
    const int smem = T.smem_doubles * 8;
    SFCDD_REQUIRE(smem <= 227 * 1024, SFCDD_EINTERNAL, "stencil tile exceeds shared memory");
    if (smem > 48 * 1024) {
      const void* ks[] = {(const void*)k_tile_matvec<2, 16>,     (const void*)k_tile_matvec<3, 16>,
                          (const void*)k_tile_tvec<2, 16>,       (const void*)k_tile_tvec<3, 16>,
                          (const void*)k_tile_pm_w<2, 16>,       (const void*)k_tile_pm_w<3, 16>,
                          (const void*)k_tile_agg_matvec<2, 16>, (const void*)k_tile_agg_matvec<3, 16>};
      for (const void* k : ks) CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
  }
  *out = op.release();
  SFCDD_API_END
}

extern "C" int sfcdd_op_setup(sfcdd_op* op, void* stream) {
  SFCDD_API_BEGIN
  (void)stream;
  SFCDD_REQUIRE(op, SFCDD_EVALUE, "null handle");
  CUDA_CHECK(cudaSetDevice(op->device));
  auto t0 = std::chrono::steady_clock::now();
  const int64_t n = op->n;
  const int d = op->d;
  // host copy of the neighbour table (setup only)
  std::vector<int32_t> nbr((size_t)2 * d * n);
  CUDA_CHECK(cudaMemcpy(nbr.data(), op->nbr, nbr.size() * 4, cudaMemcpyDeviceToHost));
  // local blocks Â_i = Â[idx_i][:, idx_i] (schwarz.py:58-61)
  // shard mode: only the owned subdomains [sf, sf + sc) are factorized
  const int32_t sf = op->shard_count > 0 ? op->shard_first : 0;
  const int32_t sc = op->shard_count > 0 ? op->shard_count : op->p;
  auto local_block = [&](int64_t i) {
    const int64_t start = op->ov_start[i], len = op->ov_len[i];
    CsrMatrix B;
    B.n = len;
    B.indptr.assign(len + 1, 0);
    B.indices.reserve(len * (2 * d + 1));
    B.data.reserve(len * (2 * d + 1));
    for (int64_t ro = 0; ro < len; ++ro) {
      int64_t gg = start + ro;
      if (gg >= n) gg -= n;
      B.indices.push_back((int32_t)ro);
      B.data.push_back(op->dhat);
      for (int a = 0; a < 2 * d; ++a) {
        const int32_t nb = nbr[(size_t)a * n + gg];
        if (nb < 0) continue;
        int64_t c = nb - start;
        if (c < 0) c += n;
        if (c < len) {
          B.indices.push_back((int32_t)c);
          B.data.push_back(op->off[a >> 1]);
        }
      }
      B.indptr[ro + 1] = B.indices.size();
    }
    return B;
  };
  // 1. ordering + symbolic analysis of every block (host threads)
  std::vector<HostFactor> fs(sc);
  FactorOptions fo;
  parallel_for(sc, op->threads, [&](int64_t li) { fs[li] = analyze_host(local_block(sf + li), fo); });
  auto t1 = std::chrono::steady_clock::now();
  std::vector<const HostFactor*> ptrs;
  std::vector<int64_t> gs, gm, xyoff(op->p, -1);
  int64_t xo = 0;
  for (int li = 0; li < sc; ++li) {
    ptrs.push_back(&fs[li]);
    gs.push_back(op->ov_start[sf + li]);
    gm.push_back(n);
    xyoff[sf + li] = xo;
    xo += op->ov_len[sf + li];
  }
  // shard mode: slots for the foreign subdomains covering owned points, filled
  // by the orchestrator's exchange before the combination
  op->own_g0 = op->dj_start[sf];
  op->own_g1 = op->dj_start[sf + sc - 1] + op->dj_len[sf + sc - 1];
  int64_t extra = 0;
  for (int j = 0; j < op->p; ++j) {
    if (j >= sf && j < sf + sc) continue;
    int64_t off = op->own_g0 - op->ov_start[j];
    if (off < 0) off += n;
    const bool hit = off < op->ov_len[j] || (op->ov_start[j] >= op->own_g0 && op->ov_start[j] < op->own_g1);
    if (op->shard_count > 0 && hit) {
      xyoff[j] = xo + extra;
      extra += op->ov_len[j];
    }
  }
  op->xy_off_host = xyoff;
  // 2. execution plan from the symbolic factors (metadata now, values later)
  PlanOptions po;
  CUDA_CHECK(cudaDeviceGetAttribute(&po.sms, cudaDevAttrMultiProcessorCount, op->device));
  po.defer_values = true;
  po.threads = op->threads;
  choose_blob_shape(ptrs, po);
  DevicePlan plan = build_plan(ptrs, gs, gm, po);
  auto t2p = std::chrono::steady_clock::now();
  op->stats.factor_nnz = plan.stored;
  op->stats.factor_nnz_l = plan.nnz_l;
  op->stats.num_tasks = (int64_t)plan.tasks.size();
  op->stats.num_supernodes = plan.num_supernodes;
  op->dag.reset(new DagSolver(plan, op->device, extra));
  op->dev_bytes += op->dag->device_bytes();
  plan = DevicePlan();
  // 3. numeric factorization of every block, values placed into the blobs
  numeric_factor_blocks(op, fs, sf, local_block);
  fs.clear();
  auto t2n = std::chrono::steady_clock::now();
  op->stats.reserved[4] = (int64_t)(1e6 * std::chrono::duration<double>(t2p - t1).count());   // plan us
  op->stats.reserved[5] = (int64_t)(1e6 * std::chrono::duration<double>(t2n - t2p).count());  // numeric us
  // combination tables: candidates per disjoint range (ascending subdomain)
  std::vector<int32_t> cptr{0}, cand;
  for (int k = 0; k < op->p; ++k) {
    const int64_t a0 = op->dj_start[k], a1 = a0 + op->dj_len[k];  // [a0, a1)
    for (int i = 0; i < op->p; ++i) {
      // does cyclic range i intersect [a0, a1)?
      const int64_t s = op->ov_start[i], l = op->ov_len[i];
      bool hit = false;
      int64_t off = a0 - s;
      if (off < 0) off += n;
      if (off < l) hit = true;
      if (!hit) {
        const int64_t e = s;  // start of i inside [a0, a1)?
        if (e >= a0 && e < a1) hit = true;
      }
      if (hit) cand.push_back(i);
    }
    cptr.push_back((int32_t)cand.size());
  }
  op->cand_ptr = dev_upload(op, cptr);
  op->cand = dev_upload(op, cand);
  {  // per reduction chunk: the subdomains meeting it, ascending (k_combine_chunk)
    std::vector<int64_t> cs((size_t)op->nch + 1);
    CUDA_CHECK(cudaMemcpy(cs.data(), op->chunk_start, cs.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<int32_t> qptr{0}, qc;
    std::vector<int32_t> tmp;
    for (int32_t ch = 0; ch < op->nch; ++ch) {
      const int64_t c0 = cs[ch], c1 = cs[ch + 1];
      // owners of the chunk's points: disjoint ranges k with [dj_k) meeting [c0, c1)
      int k0 = (int)(std::upper_bound(op->dj_start.begin(), op->dj_start.end(), c0) - op->dj_start.begin()) - 1;
      tmp.clear();
      for (int k = std::max(k0, 0); k < op->p && op->dj_start[k] < c1; ++k)
        for (int e = cptr[k]; e < cptr[k + 1]; ++e) {
          const int i = cand[e];
          const int64_t st0 = op->ov_start[i], l = op->ov_len[i];
          int64_t off = c0 - st0;  // does cyclic range i meet [c0, c1)?
          if (off < 0) off += n;
          const bool hit = off < l || (st0 >= c0 && st0 < c1);
          if (hit) tmp.push_back(i);
        }
      std::sort(tmp.begin(), tmp.end());
      tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
      SFCDD_REQUIRE((int)tmp.size() <= COMBINE_MAXC, SFCDD_EVALUE,
                    "more than " + std::to_string(COMBINE_MAXC) +
                        " overlapped subdomains cover one disjoint range (overlap gamma too large)");
      qc.insert(qc.end(), tmp.begin(), tmp.end());
      qptr.push_back((int32_t)qc.size());
    }
    op->ccand_ptr = dev_upload(op, qptr);
    op->ccand = dev_upload(op, qc);
  }
  op->d_ov_start = dev_upload(op, op->ov_start);
  op->d_ov_len = dev_upload(op, op->ov_len);
  op->d_xy_off = dev_upload(op, xyoff);
  std::vector<int64_t> djs(op->dj_start);
  djs.push_back(n);
  op->d_dj_start = dev_upload(op, djs);
  std::vector<double> wgt(op->p, 1.0);
  if (op->weighting == SFCDD_WEIGHT_OMEGA) wgt = op->omega;
  op->d_wgt = dev_upload(op, wgt);
  if (op->weighting == SFCDD_WEIGHT_DMATRIX) {
    std::vector<int32_t> cnt(n, 0);  // partition.py:151-155
    for (int i = 0; i < op->p; ++i)
      for (int64_t ro = 0; ro < op->ov_len[i]; ++ro) {
        int64_t gg = op->ov_start[i] + ro;
        if (gg >= n) gg -= n;
        cnt[gg]++;
      }
    op->d_count = dev_upload(op, cnt);
  }
  std::vector<int8_t> fault(op->p, 0);
  op->d_fault = nullptr;
  (void)fault;
  // coarse problem A0 = R0 Â R0^T, symmetrized (linalg.py:83-91), dense inverse
  if (op->n0 > 0) {
    const int32_t n0 = op->n0;
    std::vector<int32_t> aggh(n);
    for (int32_t a = 0; a < n0; ++a)
      for (int64_t g2 = op->agg_start[a]; g2 < op->agg_start[a + 1]; ++g2) aggh[g2] = a;
    std::vector<std::vector<std::pair<int32_t, double>>> rows(n0);
    parallel_for(n0, op->threads, [&](int64_t a) {
      std::map<int32_t, double> acc;
      for (int64_t g2 = op->agg_start[a]; g2 < op->agg_start[a + 1]; ++g2) {
        acc[(int32_t)a] += op->dhat;
        for (int aa = 0; aa < 2 * d; ++aa) {
          const int32_t nb = nbr[(size_t)aa * n + g2];
          if (nb >= 0) acc[aggh[nb]] += op->off[aa >> 1];
        }
      }
      rows[a].assign(acc.begin(), acc.end());
    });
    // symmetrize: (B + B^T) / 2
    std::vector<std::map<int32_t, double>> sym(n0);
    for (int32_t a = 0; a < n0; ++a)
      for (auto& e : rows[a]) {
        sym[a][e.first] += 0.5 * e.second;
        sym[e.first][a] += 0.5 * e.second;
      }
    CsrMatrix& A0 = op->a0;
    A0.n = n0;
    A0.indptr.assign(n0 + 1, 0);
    for (int32_t a = 0; a < n0; ++a) {
      for (auto& e : sym[a]) {
        A0.indices.push_back(e.first);
        A0.data.push_back(e.second);
      }
      A0.indptr[a + 1] = A0.indices.size();
    }
    op->stats.coarse_nnz = A0.indices.size();
    HostFactor F0 = factorize_host(A0, fo);
    int dense_max = COARSE_DENSE_MAX;  // SFCDD_COARSE_DENSE_MAX lowers it (tests of the sparse path)
    if (const char* e = std::getenv("SFCDD_COARSE_DENSE_MAX")) dense_max = std::min(dense_max, std::atoi(e));
    if (n0 <= dense_max) {
      // Bank-Holst redundant copy as a dense inverse: one GEMV per coarse solve
      std::vector<double> ainv((size_t)n0 * n0);
      parallel_for(n0, op->threads, [&](int64_t j) {
        std::vector<double> e(n0, 0.0), col(n0);
        e[j] = 1.0;
        host_block_solve(F0, e.data(), col.data());
        for (int32_t i = 0; i < n0; ++i) ainv[(size_t)j * n0 + i] = col[i];  // symmetric: row j
      });
      op->ainv = dev_upload(op, ainv);
    } else {
      // large coarse problems: supernodal factor of A0 solved by the DAG kernel
      PlanOptions pc;
      CUDA_CHECK(cudaDeviceGetAttribute(&pc.sms, cudaDevAttrMultiProcessorCount, op->device));
      DevicePlan cplan = build_plan({&F0}, {0}, {(int64_t)n0}, pc);
      op->coarse_dag.reset(new DagSolver(cplan, op->device));
      op->dev_bytes += op->coarse_dag->device_bytes();
      op->cvec0 = (double*)dev_alloc(op, (size_t)n0 * 8);
    }
    op->y0 = (double*)dev_alloc(op, n0 * 8);
    op->y0b = (double*)dev_alloc(op, n0 * 8);
    CUDA_CHECK(cudaMemset(op->y0, 0, n0 * 8));
    CUDA_CHECK(cudaMemset(op->y0b, 0, n0 * 8));
    if (op->ainv && (size_t)n0 * 8 > 48 * 1024)  // per-function attribute: always the maximum
      CUDA_CHECK(cudaFuncSetAttribute(k_coarse_gemv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      COARSE_DENSE_MAX * 8));
  }
  // work vectors
  op->t = (double*)dev_alloc(op, n * 8);
  op->w = (double*)dev_alloc(op, n * 8);
  op->r = (double*)dev_alloc(op, n * 8);
  op->z = (double*)dev_alloc(op, n * 8);
  op->p0 = (double*)dev_alloc(op, n * 8);
  op->p1 = (double*)dev_alloc(op, n * 8);
  op->ap = (double*)dev_alloc(op, n * 8);
  op->part_a = (double*)dev_alloc(op, op->nch * 8);
  op->part_b = (double*)dev_alloc(op, op->nch * 8);
  op->part_c = (double*)dev_alloc(op, op->nch * 8);
  op->st = (DevState*)dev_alloc(op, sizeof(DevState));
  CUDA_CHECK(cudaMemset(op->st, 0, sizeof(DevState)));
  op->stats.reserved[0] = -1;  // fault index
  op->hist_cap = 0;
  op->ready = true;
  auto t2 = std::chrono::steady_clock::now();
  op->stats.n = n;
  op->stats.n0 = op->n0;
  op->stats.order_seconds = std::chrono::duration<double>(t1 - t0).count();
  op->stats.factor_seconds = std::chrono::duration<double>(t2n - t2p).count();
  op->stats.setup_seconds = std::chrono::duration<double>(t2 - t0).count();
  SFCDD_API_END
}

extern "C" int sfcdd_op_apply(sfcdd_op* op, const double* g_dev, double* h_dev, void* stream) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(op && op->ready, SFCDD_EVALUE, "operator not set up");
  CUDA_CHECK(cudaSetDevice(op->device));
  OpScope scope(op, (cudaStream_t)stream);  // NULL = legacy default stream
  apply_device(op, g_dev, h_dev, scope.stream(), false, false);
  SFCDD_API_END
}

extern "C" int sfcdd_op_matvec(sfcdd_op* op, const double* x_dev, double* y_dev, void* stream) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(op, SFCDD_EVALUE, "null handle");
  CUDA_CHECK(cudaSetDevice(op->device));
  OpScope scope(op, (cudaStream_t)stream);  // NULL = legacy default stream
  launch_matvec(op, x_dev, y_dev, scope.stream());
  CUDA_CHECK(cudaGetLastError());
  SFCDD_API_END
}

extern "C" int sfcdd_op_pcg(sfcdd_op* op, const double* b_dev, double* x_dev, double tol, int32_t max_iters,
                            double* res_hist_host, int32_t* iters, int32_t* converged, void* stream) {
  return sfcdd_op_pcg_ex(op, b_dev, x_dev, nullptr, 0, tol, max_iters, res_hist_host, nullptr, iters, converged,
                         stream);
}

extern "C" int sfcdd_op_pcg_ex(sfcdd_op* op, const double* b_dev, double* x_dev, const double* exact_dev,
                               int32_t tol_kind, double tol, int32_t max_iters, double* res_hist_host,
                               double* energy_hist_host, int32_t* iters, int32_t* converged, void* stream) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(op && op->ready, SFCDD_EVALUE, "operator not set up");
  SFCDD_REQUIRE(tol > 0, SFCDD_EVALUE, "tolerance must be positive");
  SFCDD_REQUIRE(max_iters >= 0, SFCDD_EVALUE, "max_iters must be nonnegative");
  SFCDD_REQUIRE(tol_kind == 0 || tol_kind == 1, SFCDD_EVALUE, "unknown tolerance kind");
  SFCDD_REQUIRE(tol_kind == 0 || exact_dev, SFCDD_EVALUE, "energy stopping needs the exact solution");
  CUDA_CHECK(cudaSetDevice(op->device));
  OpScope scope(op, (cudaStream_t)stream);  // NULL = legacy default stream
  cudaStream_t st = scope.stream();
  if (op->hist_cap < max_iters + 1) {
    if (op->hist) CUDA_CHECK(cudaFree(op->hist));
    if (op->ehist) CUDA_CHECK(cudaFree(op->ehist));
    op->hist = (double*)dev_alloc(op, (size_t)(max_iters + 1) * 8);
    op->ehist = (double*)dev_alloc(op, (size_t)(max_iters + 1) * 8);
    op->hist_cap = max_iters + 1;
    // the captured iteration graph holds the old history addresses
    if (op->pcg_graph) CUDA_CHECK(cudaGraphExecDestroy(op->pcg_graph));
    op->pcg_graph = nullptr;
  }
  const Stencil S = stencil_of(op);
  const Chunks C = chunks_of(op);
  if (exact_dev) {
    if (!op->aex) {
      op->aex = (double*)dev_alloc(op, op->n * 8);
      op->part_e = (double*)dev_alloc(op, op->nch * 8);
    }
    launch_matvec(op, exact_dev, op->aex, st);  // A x*
  }
  // the captured iteration graph reads b / x* only for the energy error
  if (op->pcg_b != (exact_dev ? b_dev : nullptr) || op->pcg_exact != exact_dev) {
    if (op->pcg_graph) CUDA_CHECK(cudaGraphExecDestroy(op->pcg_graph));
    op->pcg_graph = nullptr;
  }
  op->pcg_b = exact_dev ? b_dev : nullptr;
  op->pcg_exact = exact_dev;
  k_zero_state_pcg<<<1, 1, 0, st>>>(op->st, tol, max_iters, exact_dev ? 1 : 0, tol_kind);
  CUDA_CHECK(cudaMemsetAsync(op->p0, 0, op->n * 8, st));
  k_residual0<<<op->nch, VEC_THREADS, 0, st>>>(b_dev, x_dev, S, C, op->r, op->part_b, op->part_c, op->st,
                                               op->hist);
  if (exact_dev)
    k_energy<<<op->nch, VEC_THREADS, 0, st>>>(x_dev, exact_dev, b_dev, op->r, op->aex, C, op->part_e, op->st,
                                              op->ehist, true);
  // z = C^{-1} r (krylov.py:272); skipped on device if r0 == 0
  apply_device(op, op->r, op->z, st, true, true);
  if (max_iters > 0) {
    // capture two iterations (p buffers ping-pong) once per stream/x; replay
    // the graph until the device flags convergence / breakdown / max_iters
    // (captured on the handle's private stream: the legacy default stream
    // cannot be captured; the graph is then launched on the caller's stream)
    if (!op->pcg_graph || op->stats.reserved[1] != (int64_t)x_dev) {
      if (op->pcg_graph) CUDA_CHECK(cudaGraphExecDestroy(op->pcg_graph));
      cudaGraph_t graph;
      cudaStream_t cs = op->own_stream;
      CUDA_CHECK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      pcg_iteration(op, x_dev, op->p0, op->p1, cs);
      pcg_iteration(op, x_dev, op->p1, op->p0, cs);
      CUDA_CHECK(cudaStreamEndCapture(cs, &graph));
      CUDA_CHECK(cudaGraphInstantiate(&op->pcg_graph, graph, 0));
      CUDA_CHECK(cudaGraphDestroy(graph));
      op->stats.reserved[1] = (int64_t)x_dev;
    }
    DevState hs;
    int launched = 0;  // iterations launched (2 per graph)
    int chunk = 2;     // graph launches between host polls
    while (launched < max_iters) {
      for (int i = 0; i < chunk && launched < max_iters; ++i) {
        CUDA_CHECK(cudaGraphLaunch(op->pcg_graph, st));
        launched += 2;
      }
      CUDA_CHECK(cudaMemcpyAsync(&hs, op->st, sizeof(DevState), cudaMemcpyDeviceToHost, st));
      CUDA_CHECK(cudaStreamSynchronize(st));
      if (hs.done) break;
      chunk = std::min(chunk * 2, 8);
    }
    op->stats.reserved[3] = launched;
  } else {
    op->stats.reserved[3] = 0;
  }
  DevState hs;
  CUDA_CHECK(cudaMemcpyAsync(&hs, op->st, sizeof(DevState), cudaMemcpyDeviceToHost, st));
  CUDA_CHECK(cudaStreamSynchronize(st));
  {
    // kernel launches of this call: init (zero, residual [+ A x*, energy], apply) + the iterations
    const int64_t per_apply = apply_launches(op, true, true);
    // per iteration: p-update/matvec, x/r update [+ energy error]
    const int64_t per_it = 2 + (exact_dev ? 1 : 0);
    op->stats.reserved[2] = 2 + (exact_dev ? 2 : 0) + per_apply + op->stats.reserved[3] * (per_it + per_apply);
  }
  const int k = hs.k;
  if (res_hist_host) CUDA_CHECK(cudaMemcpy(res_hist_host, op->hist, (size_t)(k + 1) * 8, cudaMemcpyDeviceToHost));
  if (energy_hist_host && exact_dev)
    CUDA_CHECK(cudaMemcpy(energy_hist_host, op->ehist, (size_t)(k + 1) * 8, cudaMemcpyDeviceToHost));
  *iters = k;
  *converged = hs.converged;
  if (hs.breakdown) throw Error(SFCDD_EBREAKDOWN, "nonpositive curvature at iteration " + std::to_string(k + 1));
  SFCDD_API_END
}

extern "C" int sfcdd_op_set_fault(sfcdd_op* op, int64_t apply_index, const int32_t* ids_host, int32_t nids) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(op && op->ready, SFCDD_EVALUE, "operator not set up");
  CUDA_CHECK(cudaSetDevice(op->device));
  if (nids <= 0) {
    op->stats.reserved[0] = -1;
    if (op->d_fault) CUDA_CHECK(cudaFree(op->d_fault));
    op->d_fault = nullptr;
    return SFCDD_OK;
  }
  std::vector<int8_t> mask(op->p, 0);
  for (int32_t i = 0; i < nids; ++i) {
    SFCDD_REQUIRE(ids_host[i] >= 0 && ids_host[i] < op->p, SFCDD_EVALUE, "fault subdomain out of range");
    mask[ids_host[i]] = 1;
  }
  if (!op->d_fault) op->d_fault = (int8_t*)dev_alloc(op, op->p);
  CUDA_CHECK(cudaMemcpy(op->d_fault, mask.data(), op->p, cudaMemcpyHostToDevice));
  op->stats.reserved[0] = apply_index;
  // the PCG graph bakes kernel arguments: force re-capture
  if (op->pcg_graph) CUDA_CHECK(cudaGraphExecDestroy(op->pcg_graph));
  op->pcg_graph = nullptr;
  SFCDD_API_END
}

extern "C" int sfcdd_op_profile(sfcdd_op* op, const double* g_dev, double* scratch_dev, int32_t reps,
                                double* ms, int32_t* launches, void* stream) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(op && op->ready && reps >= 1, SFCDD_EVALUE, "operator not set up");
  CUDA_CHECK(cudaSetDevice(op->device));
  cudaStream_t st = (cudaStream_t)stream;  // NULL = legacy default stream
  float t = 0.f;
  // local solves alone
  op->dag->solve(g_dev, st);
  CUDA_CHECK(cudaEventRecord(op->ev0, st));
  for (int i = 0; i < reps; ++i) op->dag->solve(g_dev, st);
  CUDA_CHECK(cudaEventRecord(op->ev1, st));
  CUDA_CHECK(cudaEventSynchronize(op->ev1));
  CUDA_CHECK(cudaEventElapsedTime(&t, op->ev0, op->ev1));
  ms[0] = t / reps;
  // full apply
  CUDA_CHECK(cudaEventRecord(op->ev0, st));
  for (int i = 0; i < reps; ++i) apply_device(op, g_dev, scratch_dev, st, false, false);
  CUDA_CHECK(cudaEventRecord(op->ev1, st));
  CUDA_CHECK(cudaEventSynchronize(op->ev1));
  CUDA_CHECK(cudaEventElapsedTime(&t, op->ev0, op->ev1));
  ms[1] = t / reps;
  // matvec (one untimed launch first: lazy module loading of the kernel)
  launch_matvec(op, g_dev, scratch_dev, st);
  CUDA_CHECK(cudaEventRecord(op->ev0, st));
  for (int i = 0; i < reps; ++i)
    launch_matvec(op, g_dev, scratch_dev, st);
  CUDA_CHECK(cudaEventRecord(op->ev1, st));
  CUDA_CHECK(cudaEventSynchronize(op->ev1));
  CUDA_CHECK(cudaEventElapsedTime(&t, op->ev0, op->ev1));
  ms[2] = t / reps;
  if (std::getenv("SFCDD_PROFILE_KERNELS")) {
    // one PCG iteration's kernels, each timed by the events between launches
    // (warm, back to back on the stream; the solver state is reset per rep so
    // no kernel early-exits)
    KernelTimer kt;
    if (op->pcg_graph) CUDA_CHECK(cudaGraphExecDestroy(op->pcg_graph));
    op->pcg_graph = nullptr;
    op->pcg_exact = op->pcg_b = nullptr;
    if (op->hist_cap < 2) {  // k_update records the residual history
      if (op->hist) CUDA_CHECK(cudaFree(op->hist));
      if (op->ehist) CUDA_CHECK(cudaFree(op->ehist));
      op->hist = (double*)dev_alloc(op, 2 * 8);
      op->ehist = (double*)dev_alloc(op, 2 * 8);
      op->hist_cap = 2;
    }
    double* xs = (double*)dev_alloc(op, op->n * 8);
    CUDA_CHECK(cudaMemsetAsync(xs, 0, op->n * 8, st));
    CUDA_CHECK(cudaMemsetAsync(op->p0, 0, op->n * 8, st));
    CUDA_CHECK(cudaMemcpyAsync(op->r, g_dev, op->n * 8, cudaMemcpyDeviceToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(op->z, g_dev, op->n * 8, cudaMemcpyDeviceToDevice, st));
    // captured as a CUDA graph (event-record nodes between the kernels), as
    // the PCG loop runs it, so host launch latency is not measured
    CUDA_CHECK(cudaStreamSynchronize(st));
    cudaGraph_t graph;
    cudaGraphExec_t gexec;
    cudaStream_t cs = op->own_stream;
    CUDA_CHECK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    k_zero_state_pcg<<<1, 1, 0, cs>>>(op->st, 1e-300, 1 << 30, 0, 0);
    g_ktimer = &kt;
    kt.idx = 0;
    kmark(cs, "start");
    pcg_iteration(op, xs, op->p0, op->p1, cs);
    g_ktimer = nullptr;
    CUDA_CHECK(cudaStreamEndCapture(cs, &graph));
    CUDA_CHECK(cudaGraphInstantiate(&gexec, graph, 0));
    CUDA_CHECK(cudaGraphDestroy(graph));
    for (int i = 0; i < reps + 1; ++i) {
      CUDA_CHECK(cudaGraphLaunch(gexec, st));
      CUDA_CHECK(cudaStreamSynchronize(st));
      if (i == 0) continue;  // warm-up
      for (size_t e = 1; e < kt.idx; ++e) {
        float dt = 0.f;
        CUDA_CHECK(cudaEventElapsedTime(&dt, kt.ev[e - 1], kt.ev[e]));
        kt.ms[e] += dt / reps;
      }
    }
    double tot = 0.0;
    for (size_t e = 1; e < kt.idx; ++e) tot += kt.ms[e];
    for (size_t e = 1; e < kt.idx; ++e)
      std::fprintf(stderr, "[kernels] %-14s %8.1f us\n", kt.name[e], 1e3 * kt.ms[e]);
    std::fprintf(stderr, "[kernels] %-14s %8.1f us\n", "total", 1e3 * tot);
    CUDA_CHECK(cudaGraphExecDestroy(gexec));
    {  // each vector kernel alone, 20 back-to-back launches
      const Stencil S = stencil_of(op);
      const Chunks C = chunks_of(op);
      const bool direct = op->nch == op->n0;
      auto iso = [&](const char* name, auto fn) {
        fn();
        CUDA_CHECK(cudaEventRecord(op->ev0, st));
        for (int i = 0; i < 20; ++i) fn();
        CUDA_CHECK(cudaEventRecord(op->ev1, st));
        CUDA_CHECK(cudaEventSynchronize(op->ev1));
        float dt = 0.f;
        CUDA_CHECK(cudaEventElapsedTime(&dt, op->ev0, op->ev1));
        std::fprintf(stderr, "[isolated] %-14s %8.1f us\n", name, 1e3 * dt / 20);
      };
      iso("coarse_solve", [&] { coarse_solve(op, op->part_c, op->agg_ptr, direct, op->y0, nullptr, PcgFin{}, st); });
      iso("tvec", [&] {
        k_tvec<<<nblocks(op->n, VEC_THREADS), VEC_THREADS, 0, st>>>(op->r, op->y0, op->agg, S, op->t, nullptr);
      });
      iso("matvec_chunk", [&] { k_matvec_chunk<<<op->nch, VEC_THREADS, 0, st>>>(op->w, S, C, op->part_b, nullptr); });
      iso("matvec", [&] { launch_matvec(op, op->w, op->t, st); });
      iso("chunk_sum", [&] { k_chunk_sum<<<op->nch, VEC_THREADS, 0, st>>>(op->w, C, op->part_c); });
      iso("copy", [&] { CUDA_CHECK(cudaMemcpyAsync(op->t, op->w, op->n * 8, cudaMemcpyDeviceToDevice, st)); });
    }
    for (cudaEvent_t e : kt.ev) cudaEventDestroy(e);
    CUDA_CHECK(cudaFree(xs));
    op->dev_bytes -= op->n * 8;
  }
  long long zero = 0;
  CUDA_CHECK(cudaMemcpy(&op->st->apply_calls, &zero, sizeof(zero), cudaMemcpyHostToDevice));
  if (launches) {
    launches[0] = 1;
    launches[1] = apply_launches(op, false, false);
    launches[2] = 1;
  }
  SFCDD_API_END
}

extern "C" int sfcdd_op_trace(sfcdd_op* op, const double* g_dev, uint64_t* out_host, int64_t* ntask) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(op && op->ready, SFCDD_EVALUE, "operator not set up");
  const int64_t nt = op->dag->ntask();
  *ntask = nt;
  if (!out_host) return SFCDD_OK;
  CUDA_CHECK(cudaSetDevice(op->device));
  unsigned long long* buf = nullptr;
  CUDA_CHECK(cudaMalloc(&buf, nt * 21 * 8));
  CUDA_CHECK(cudaMemset(buf, 0, nt * 21 * 8));
  op->dag->solve(g_dev, nullptr);  // warm
  op->dag->set_trace(buf);
  op->dag->solve(g_dev, nullptr);
  op->dag->set_trace(nullptr);
  CUDA_CHECK(cudaDeviceSynchronize());
  std::vector<unsigned long long> h(nt * 21);
  CUDA_CHECK(cudaMemcpy(h.data(), buf, nt * 21 * 8, cudaMemcpyDeviceToHost));
  CUDA_CHECK(cudaFree(buf));
  for (int64_t t = 0; t < nt; ++t) {
    const TaskDev& T = op->dag->host_tasks[t];
    for (int j = 0; j < 5; ++j) out_host[24 * t + j] = h[5 * t + j];
    out_host[24 * t + 5] = (uint64_t)T.kind;
    out_host[24 * t + 6] = (uint64_t)T.copy_bytes;
    out_host[24 * t + 7] = (uint64_t)T.group;
    out_host[24 * t + 8] = (uint64_t)T.values;
    out_host[24 * t + 9] = (uint64_t)(int64_t)T.wait_idx;
    out_host[24 * t + 10] = (uint64_t)T.wait_target;
    out_host[24 * t + 11] = (uint64_t)T.signal_idx;
    for (int j = 12; j < 24; ++j) out_host[24 * t + j] = 0;
    // FRAG forward phase stamps (clock64): [0] start [1] prologue done
    // [2+2l, 3+2l] level l assembly / rows done (l < 4) [10] end [11] nlev
    // (BLOB ROW tasks: [0] start [1] front in the slot [2] products + stores issued [11] 100 + rows)
    if (T.kind == TK_FRAG_FWD || T.kind == TK_FRAG_BWD || T.kind == TK_ROW_FWD)
      for (int j = 0; j < 12; ++j) out_host[24 * t + 12 + j] = h[5 * nt + 16 * t + (j < 10 ? j : j + 4)];
  }
  SFCDD_API_END
}

extern "C" int sfcdd_op_reset_calls(sfcdd_op* op) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(op && op->ready, SFCDD_EVALUE, "operator not set up");
  CUDA_CHECK(cudaSetDevice(op->device));
  long long zero = 0;
  CUDA_CHECK(cudaMemcpy(&op->st->apply_calls, &zero, sizeof(zero), cudaMemcpyHostToDevice));
  SFCDD_API_END
}

extern "C" int sfcdd_op_stats(sfcdd_op* op, sfcdd_stats* out) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(op && out, SFCDD_EVALUE, "null argument");
  *out = op->stats;
  out->device_bytes = op->dev_bytes;
  if (op->ready) {
    long long calls = 0;
    CUDA_CHECK(cudaSetDevice(op->device));
    CUDA_CHECK(cudaMemcpy(&calls, &op->st->apply_calls, sizeof(calls), cudaMemcpyDeviceToHost));
    out->apply_calls = calls;
  }
  SFCDD_API_END
}

extern "C" int sfcdd_op_stencil(sfcdd_op* op, double* diag, double* off, double* t) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(op, SFCDD_EVALUE, "null handle");
  if (diag) *diag = op->dhat;
  if (off)
    for (int j = 0; j < op->d; ++j) off[j] = op->off[j];
  if (t) *t = op->tscale;
  SFCDD_API_END
}

extern "C" int sfcdd_op_coarse_dense(sfcdd_op* op, double* a0_host) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(op && op->ready, SFCDD_EVALUE, "operator not set up");
  SFCDD_REQUIRE(op->a0.n > 0, SFCDD_EVALUE, "no coarse space");
  const int64_t n0 = op->a0.n;
  std::fill(a0_host, a0_host + n0 * n0, 0.0);
  for (int64_t a = 0; a < n0; ++a)
    for (int64_t e = op->a0.indptr[a]; e < op->a0.indptr[a + 1]; ++e) a0_host[a * n0 + op->a0.indices[e]] = op->a0.data[e];
  SFCDD_API_END
}

extern "C" void sfcdd_op_destroy(sfcdd_op* op) {
  if (!op) return;
  cudaSetDevice(op->device);
  if (op->pcg_graph) cudaGraphExecDestroy(op->pcg_graph);
  void* ptrs[] = {op->nbr, op->agg, op->chunk_start, op->chunk_agg, op->agg_ptr, op->ainv, op->d_ov_start,
                  op->d_ov_len, op->d_xy_off, op->d_dj_start, op->cand_ptr, op->cand, op->ccand_ptr, op->ccand,
                  op->d_wgt, op->d_count,
                  op->d_fault, op->st, op->hist, op->t, op->w, op->y0, op->y0b, op->part_a, op->part_b,
                  op->part_c, op->r, op->z, op->p0, op->p1, op->ap, op->aex, op->part_e, op->ehist,
                  (void*)op->tiles.r0, (void*)op->tiles.dims, (void*)op->tiles.tab_off, (void*)op->tiles.tab,
                  (void*)op->tiles.halo_off, (void*)op->tiles.halo, (void*)op->tiles.slot0, (void*)op->tiles.sptr,
                  op->part_t, op->cvec, op->d_agg_start};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  op->dag.reset();
  if (op->srt) destroy_shard_runtime(op->srt);
  if (op->ev_in) cudaEventDestroy(op->ev_in);
  if (op->ev_out) cudaEventDestroy(op->ev_out);
  if (op->ev0) cudaEventDestroy(op->ev0);
  if (op->ev1) cudaEventDestroy(op->ev1);
  if (op->own_stream) cudaStreamDestroy(op->own_stream);
  delete op;
}

// ========================================================= shard mode
// One handle per rank (multi-GPU).  Vectors stay full length N
// on every rank but each step only computes the owned SFC segment / owned
// chunks; the Python orchestrator (paper_2110_11211_b200/distributed.py)
// moves halo / overlap / foreign-solution values with NCCL between steps and
// reduces the partial scalars.
namespace sfcdd {
namespace {

__global__ void k_sh_residual(const double* __restrict__ b, const double* __restrict__ x, Stencil S, Chunks C,
                              int ch0, double* __restrict__ r, double* __restrict__ prr, double* __restrict__ pc) {
  const int ch = ch0 + blockIdx.x;
  double rr = 0.0, cs = 0.0;
  const int64_t c_end = C.start[ch + 1];
  for (int64_t g = C.start[ch] + threadIdx.x; g < c_end; g += VEC_THREADS) {
    const double v = b[g] - stencil_at(S, x, g);
    r[g] = v;
    rr = fma(v, v, rr);
    cs += v;
  }
  rr = block_sum(rr);
  cs = block_sum(cs);
  if (threadIdx.x == 0) {
    prr[ch] = rr;
    pc[ch] = cs;
  }
}

__global__ void k_sh_pm(const double* __restrict__ z, const double* __restrict__ pold, double beta_h, Stencil S,
                        Chunks C, int ch0, double* __restrict__ pnew, double* __restrict__ ap,
                        double* __restrict__ part, const double* __restrict__ beta_d = nullptr) {
  const double beta = beta_d ? *beta_d : beta_h;  // device-driven PCG: beta on the device
  const int ch = ch0 + blockIdx.x;
  double s = 0.0;
  const int64_t c_end = C.start[ch + 1];
  for (int64_t g = C.start[ch] + threadIdx.x; g < c_end; g += VEC_THREADS) {
    const double pg = __dadd_rn(z[g], __dmul_rn(beta, pold[g]));
    double acc = S.dhat * pg;
    for (int a = 0; a < 2 * S.d; ++a) {
      const int32_t nb = __ldg(S.nbr + (int64_t)a * S.n + g);
      if (nb >= 0) acc = fma(S.off[a >> 1], __dadd_rn(z[nb], __dmul_rn(beta, pold[nb])), acc);
    }
    pnew[g] = pg;
    ap[g] = acc;
    s = fma(pg, acc, s);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[ch] = s;
}

__global__ void k_sh_update(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                            const double* __restrict__ ap, double alpha_h, Chunks C, int ch0,
                            double* __restrict__ prr, double* __restrict__ pc,
                            const double* __restrict__ alpha_d = nullptr, const int32_t* __restrict__ skip = nullptr) {
  if (skip && *skip) return;  // breakdown: x and r stay those of the last iterate
  const double alpha = alpha_d ? *alpha_d : alpha_h;
  const int ch = ch0 + blockIdx.x;
  double rr = 0.0, cs = 0.0;
  const int64_t c_end = C.start[ch + 1];
  for (int64_t g = C.start[ch] + threadIdx.x; g < c_end; g += VEC_THREADS) {
    x[g] = __dadd_rn(x[g], __dmul_rn(alpha, p[g]));
    const double v = __dsub_rn(r[g], __dmul_rn(alpha, ap[g]));
    r[g] = v;
    rr = fma(v, v, rr);
    cs += v;
  }
  rr = block_sum(rr);
  cs = block_sum(cs);
  if (threadIdx.x == 0) {
    prr[ch] = rr;
    pc[ch] = cs;
  }
}

__global__ void k_sh_stencil_chunks(const double* __restrict__ w, Stencil S, Chunks C, int ch0,
                                    double* __restrict__ part) {
  const int ch = ch0 + blockIdx.x;
  double s = 0.0;
  const int64_t c_end = C.start[ch + 1];
  for (int64_t g = C.start[ch] + threadIdx.x; g < c_end; g += VEC_THREADS) s += stencil_at(S, w, g);
  s = block_sum(s);
  if (threadIdx.x == 0) part[ch] = s;
}

__global__ void k_sh_finalize(const double* __restrict__ w, const double* __restrict__ y0,
                              const double* __restrict__ y0b, Chunks C, int ch0, int mode, double* __restrict__ h,
                              const double* __restrict__ rdot, double* __restrict__ part) {
  const int ch = ch0 + blockIdx.x;
  const int a = C.agg[ch];
  const double c0 = mode >= 1 ? y0[a] : 0.0;
  const double c1 = mode >= 2 ? y0b[a] : 0.0;
  double s = 0.0;
  const int64_t c_end = C.start[ch + 1];
  for (int64_t g = C.start[ch] + threadIdx.x; g < c_end; g += VEC_THREADS) {
    double v = w[g];
    if (mode == 1) v = v + c0;
    if (mode == 2) v = (v - c1) + c0;
    h[g] = v;
    if (rdot) s = fma(rdot[g], v, s);
  }
  if (rdot) {
    s = block_sum(s);
    if (threadIdx.x == 0) part[ch] = s;
  }
}

// fixed-order sum of part[ch0, ch1) into *out (one block)
__global__ void k_sum_range(const double* __restrict__ part, int ch0, int ch1, double* __restrict__ out) {
  double v = 0.0;
  for (int i = ch0 + threadIdx.x; i < ch1; i += VEC_THREADS) v += part[i];
  v = block_sum(v);
  if (threadIdx.x == 0) *out = v;
}

// per-aggregate sums of the chunk partials for aggregates [a0, a1)
__global__ void k_agg_sums(const double* __restrict__ part, const int32_t* __restrict__ agg_ptr, int a0, int a1,
                           double* __restrict__ out) {
  const int a = a0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= a1) return;
  double s = 0.0;
  for (int ch = agg_ptr[a]; ch < agg_ptr[a + 1]; ++ch) s += part[ch];
  out[a - a0] = s;
}

__global__ void k_gemv_c(const double* __restrict__ ainv, const double* __restrict__ cin, int32_t n0,
                         double* __restrict__ y) {
  extern __shared__ double c[];
  for (int a = threadIdx.x; a < n0; a += VEC_THREADS) c[a] = cin[a];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (VEC_THREADS / 32) + (threadIdx.x >> 5);
  if (row >= n0) return;
  const double* ar = ainv + (int64_t)row * n0;
  double acc = 0.0;
  for (int j = lane; j < n0; j += 32) acc = fma(__ldg(ar + j), c[j], acc);
  acc = warp_sum(acc);
  if (lane == 0) y[row] = acc;
}

__global__ void k_sh_tvec(const double* __restrict__ gv, const double* __restrict__ y0,
                          const int32_t* __restrict__ agg, Stencil S, int64_t g0, int64_t g1,
                          double* __restrict__ t) {
  const int64_t g = g0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= g1) return;
  double acc = S.dhat * y0[agg[g]];
  for (int a = 0; a < 2 * S.d; ++a) {
    const int32_t nb = __ldg(S.nbr + (int64_t)a * S.n + g);
    if (nb >= 0) acc = fma(S.off[a >> 1], y0[agg[nb]], acc);
  }
  t[g] = gv[g] - acc;
}

__global__ void k_sh_combine(CombineArgs C, int64_t g0, int64_t g1, double* __restrict__ w) {
  const int64_t g = g0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= g1) return;
  int lo = 0, hi = C.p;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (C.dj_start[mid] <= g)
      lo = mid;
    else
      hi = mid;
  }
  double acc = 0.0;
  for (int c = C.cand_ptr[lo]; c < C.cand_ptr[lo + 1]; ++c) {
    const int i = C.cand[c];
    int64_t off = g - C.ov_start[i];
    if (off < 0) off += C.n;
    if (off >= C.ov_len[i]) continue;
    const double wt = C.count ? 1.0 / (double)C.count[g] : C.wgt[i];
    acc = __dadd_rn(acc, __dmul_rn(wt, __ldcg(C.xy + C.xy_off[i] + off)));
  }
  w[g] = acc;
}

__global__ void k_pack(const double* __restrict__ src, const int64_t* __restrict__ idx, int64_t n,
                       double* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

__global__ void k_unpack(const double* __restrict__ src, const int64_t* __restrict__ idx, int64_t n,
                         double* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[idx[i]] = src[i];
}

}  // namespace

struct ShardRange {
  int ch0, ch1, a0, a1;
  int64_t g0, g1;
};

static ShardRange shard_range(const sfcdd_op* op) {
  const int32_t sf = op->shard_count > 0 ? op->shard_first : 0;
  const int32_t sc = op->shard_count > 0 ? op->shard_count : op->p;
  ShardRange r;
  r.a0 = sf * op->q;
  r.a1 = (sf + sc) * op->q;
  std::vector<int32_t> aptr(op->n0 + 1);
  // agg_ptr lives on device; the host copy is rebuilt from agg_start sizes
  int32_t c = 0;
  aptr[0] = 0;
  for (int32_t a = 0; a < op->n0; ++a) {
    const int64_t len = op->agg_start[a + 1] - op->agg_start[a];
    c += (int32_t)((len + CHUNK - 1) / CHUNK);
    aptr[a + 1] = c;
  }
  r.ch0 = aptr[r.a0];
  r.ch1 = aptr[r.a1];
  r.g0 = op->agg_start[r.a0];
  r.g1 = op->agg_start[r.a1];
  return r;
}

}  // namespace sfcdd

extern "C" int sfcdd_shard_info(sfcdd_op* op, int64_t* info, int64_t* xy_off_host) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(op && op->ready && op->n0 > 0, SFCDD_EVALUE, "shard mode needs a set-up operator with a coarse space");
  const ShardRange r = shard_range(op);
  info[0] = r.g0;
  info[1] = r.g1;
  info[2] = r.ch0;
  info[3] = r.ch1;
  info[4] = r.a0;
  info[5] = r.a1;
  info[6] = op->dag->xy_doubles();
  info[7] = op->n0;
  if (xy_off_host)
    for (int i = 0; i < op->p; ++i) xy_off_host[i] = op->xy_off_host[i];
  SFCDD_API_END
}

extern "C" int sfcdd_op_neighbors(sfcdd_op* op, int32_t* nbr_host) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(op && nbr_host, SFCDD_EVALUE, "null argument");
  CUDA_CHECK(cudaSetDevice(op->device));
  CUDA_CHECK(cudaMemcpy(nbr_host, op->nbr, (size_t)2 * op->d * op->n * 4, cudaMemcpyDeviceToHost));
  SFCDD_API_END
}

extern "C" int sfcdd_shard_xy(sfcdd_op* op, double** xy) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(op && op->ready, SFCDD_EVALUE, "operator not set up");
  *xy = op->dag->xy();
  SFCDD_API_END
}

extern "C" int sfcdd_shard_residual(sfcdd_op* op, const double* b, const double* x, double* r, double* rr_out,
                                    double* cagg_out, void* stream) {
  SFCDD_API_BEGIN
  const ShardRange R = shard_range(op);
  cudaStream_t st = (cudaStream_t)stream;
  k_sh_residual<<<R.ch1 - R.ch0, VEC_THREADS, 0, st>>>(b, x, stencil_of(op), chunks_of(op), R.ch0, r, op->part_b,
                                                       op->part_c);
  k_sum_range<<<1, VEC_THREADS, 0, st>>>(op->part_b, R.ch0, R.ch1, rr_out);
  k_agg_sums<<<nblocks(R.a1 - R.a0, 128), 128, 0, st>>>(op->part_c, op->agg_ptr, R.a0, R.a1, cagg_out);
  CUDA_CHECK(cudaGetLastError());
  SFCDD_API_END
}

extern "C" int sfcdd_shard_pm(sfcdd_op* op, const double* z, const double* pold, double beta, double* pnew,
                              double* ap, double* pap_out, void* stream) {
  SFCDD_API_BEGIN
  const ShardRange R = shard_range(op);
  cudaStream_t st = (cudaStream_t)stream;
  k_sh_pm<<<R.ch1 - R.ch0, VEC_THREADS, 0, st>>>(z, pold, beta, stencil_of(op), chunks_of(op), R.ch0, pnew, ap,
                                                 op->part_a);
  k_sum_range<<<1, VEC_THREADS, 0, st>>>(op->part_a, R.ch0, R.ch1, pap_out);
  CUDA_CHECK(cudaGetLastError());
  SFCDD_API_END
}

extern "C" int sfcdd_shard_update(sfcdd_op* op, double* x, double* r, const double* p, const double* ap, double alpha,
                                  double* rr_out, double* cagg_out, void* stream) {
  SFCDD_API_BEGIN
  const ShardRange R = shard_range(op);
  cudaStream_t st = (cudaStream_t)stream;
  k_sh_update<<<R.ch1 - R.ch0, VEC_THREADS, 0, st>>>(x, r, p, ap, alpha, chunks_of(op), R.ch0, op->part_b,
                                                     op->part_c);
  k_sum_range<<<1, VEC_THREADS, 0, st>>>(op->part_b, R.ch0, R.ch1, rr_out);
  k_agg_sums<<<nblocks(R.a1 - R.a0, 128), 128, 0, st>>>(op->part_c, op->agg_ptr, R.a0, R.a1, cagg_out);
  CUDA_CHECK(cudaGetLastError());
  SFCDD_API_END
}

extern "C" int sfcdd_shard_coarse(sfcdd_op* op, const double* c, double* y, void* stream) {
  SFCDD_API_BEGIN
  cudaStream_t st = (cudaStream_t)stream;
  if (!op->ainv) {  // sparse coarse factor
    op->coarse_dag->solve(c, st);
    CUDA_CHECK(cudaMemcpyAsync(y, op->coarse_dag->xy(), (size_t)op->n0 * 8, cudaMemcpyDeviceToDevice, st));
    CUDA_CHECK(cudaGetLastError());
    return SFCDD_OK;
  }
  const size_t smem = (size_t)op->n0 * 8;
  if (smem > 48 * 1024)
    CUDA_CHECK(cudaFuncSetAttribute(k_gemv_c, cudaFuncAttributeMaxDynamicSharedMemorySize, COARSE_DENSE_MAX * 8));
  k_gemv_c<<<nblocks(op->n0, VEC_THREADS / 32), VEC_THREADS, smem, st>>>(op->ainv, c, op->n0, y);
  CUDA_CHECK(cudaGetLastError());
  SFCDD_API_END
}

extern "C" int sfcdd_shard_tvec(sfcdd_op* op, const double* g, const double* y0, double* t, void* stream) {
  SFCDD_API_BEGIN
  const ShardRange R = shard_range(op);
  k_sh_tvec<<<nblocks(R.g1 - R.g0, VEC_THREADS), VEC_THREADS, 0, (cudaStream_t)stream>>>(g, y0, op->agg,
                                                                                       stencil_of(op), R.g0, R.g1, t);
  CUDA_CHECK(cudaGetLastError());
  SFCDD_API_END
}

extern "C" int sfcdd_shard_local_solve(sfcdd_op* op, const double* t, void* stream) {
  SFCDD_API_BEGIN
  op->dag->solve(t, (cudaStream_t)stream);
  SFCDD_API_END
}

extern "C" int sfcdd_shard_combine(sfcdd_op* op, double* w, void* stream) {
  SFCDD_API_BEGIN
  const ShardRange R = shard_range(op);
  CombineArgs ca;
  ca.xy = op->dag->xy();
  ca.ov_start = op->d_ov_start;
  ca.ov_len = op->d_ov_len;
  ca.xy_off = op->d_xy_off;
  ca.dj_start = op->d_dj_start;
  ca.cand_ptr = op->cand_ptr;
  ca.cand = op->cand;
  ca.wgt = op->d_wgt;
  ca.count = op->weighting == SFCDD_WEIGHT_DMATRIX ? op->d_count : nullptr;
  ca.fault = nullptr;
  ca.apply_calls = nullptr;
  ca.fault_index = -1;
  ca.p = op->p;
  ca.n = op->n;
  k_sh_combine<<<nblocks(R.g1 - R.g0, VEC_THREADS), VEC_THREADS, 0, (cudaStream_t)stream>>>(ca, R.g0, R.g1, w);
  CUDA_CHECK(cudaGetLastError());
  SFCDD_API_END
}

extern "C" int sfcdd_shard_stencil_restrict(sfcdd_op* op, const double* w, double* cagg_out, void* stream) {
  SFCDD_API_BEGIN
  const ShardRange R = shard_range(op);
  cudaStream_t st = (cudaStream_t)stream;
  k_sh_stencil_chunks<<<R.ch1 - R.ch0, VEC_THREADS, 0, st>>>(w, stencil_of(op), chunks_of(op), R.ch0, op->part_b);
  k_agg_sums<<<nblocks(R.a1 - R.a0, 128), 128, 0, st>>>(op->part_b, op->agg_ptr, R.a0, R.a1, cagg_out);
  CUDA_CHECK(cudaGetLastError());
  SFCDD_API_END
}

extern "C" int sfcdd_shard_finalize(sfcdd_op* op, const double* w, const double* y0, const double* y0b, double* z,
                                    const double* r, double* rz_out, void* stream) {
  SFCDD_API_BEGIN
  const ShardRange R = shard_range(op);
  cudaStream_t st = (cudaStream_t)stream;
  k_sh_finalize<<<R.ch1 - R.ch0, VEC_THREADS, 0, st>>>(w, y0, y0b, chunks_of(op), R.ch0, mode_of(op->variant), z, r,
                                                       op->part_a);
  if (r) k_sum_range<<<1, VEC_THREADS, 0, st>>>(op->part_a, R.ch0, R.ch1, rz_out);
  CUDA_CHECK(cudaGetLastError());
  SFCDD_API_END
}

extern "C" int sfcdd_pack(const double* src, const int64_t* idx, int64_t n, double* dst, void* stream) {
  SFCDD_API_BEGIN
  if (n > 0) k_pack<<<nblocks(n, 256), 256, 0, (cudaStream_t)stream>>>(src, idx, n, dst);
  CUDA_CHECK(cudaGetLastError());
  SFCDD_API_END
}

extern "C" int sfcdd_unpack(const double* src, const int64_t* idx, int64_t n, double* dst, void* stream) {
  SFCDD_API_BEGIN
  if (n > 0) k_unpack<<<nblocks(n, 256), 256, 0, (cudaStream_t)stream>>>(src, idx, n, dst);
  CUDA_CHECK(cudaGetLastError());
  SFCDD_API_END
}

// ------------------------------------------------- generic sparse factor
struct sfcdd_factor {
  int device = 0;
  int64_t n = 0;
  std::unique_ptr<DagSolver> dag;
  int64_t nnz_l = 0, stored = 0, nsuper = 0;
};

extern "C" int sfcdd_factor_create(int64_t n, const int64_t* indptr, const int32_t* indices, const double* data,
                                   int32_t device, sfcdd_factor** out) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(n >= 1 && out, SFCDD_EVALUE, "invalid arguments");
  CsrMatrix A;
  A.n = n;
  A.indptr.assign(indptr, indptr + n + 1);
  A.indices.assign(indices, indices + indptr[n]);
  A.data.assign(data, data + indptr[n]);
  FactorOptions fo;
  HostFactor F = factorize_host(A, fo);
  std::unique_ptr<sfcdd_factor> f(new sfcdd_factor());
  f->device = device;
  f->n = n;
  f->nnz_l = F.nnz_l;
  f->stored = F.stored;
  f->nsuper = F.sn.size();
  PlanOptions po;
  CUDA_CHECK(cudaDeviceGetAttribute(&po.sms, cudaDevAttrMultiProcessorCount, device));
  DevicePlan plan = build_plan({&F}, {0}, {n}, po);
  CUDA_CHECK(cudaSetDevice(device));
  f->dag.reset(new DagSolver(plan, device));
  *out = f.release();
  SFCDD_API_END
}

extern "C" int sfcdd_factor_solve(sfcdd_factor* f, const double* b_dev, double* x_dev, void* stream) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(f, SFCDD_EVALUE, "null handle");
  CUDA_CHECK(cudaSetDevice(f->device));
  cudaStream_t st = (cudaStream_t)stream;
  f->dag->solve(b_dev, st);
  CUDA_CHECK(cudaMemcpyAsync(x_dev, f->dag->xy(), f->n * 8, cudaMemcpyDeviceToDevice, st));
  SFCDD_API_END
}

extern "C" int sfcdd_factor_info(sfcdd_factor* f, int64_t* nnz_l, int64_t* stored, int64_t* nsuper) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(f, SFCDD_EVALUE, "null handle");
  if (nnz_l) *nnz_l = f->nnz_l;
  if (stored) *stored = f->stored;
  if (nsuper) *nsuper = f->nsuper;
  SFCDD_API_END
}

extern "C" void sfcdd_factor_destroy(sfcdd_factor* f) {
  if (!f) return;
  cudaSetDevice(f->device);
  f->dag.reset();
  delete f;
}

// ------------------------------------------------------------ BLAS-1 API
namespace sfcdd {
namespace {
constexpr int DOT_BLOCKS = 592;  // 4 x 148 SMs; fixed -> fixed summation order
__global__ void k_dot_part(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                           double* __restrict__ part) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * VEC_THREADS + threadIdx.x; i < n; i += (int64_t)DOT_BLOCKS * VEC_THREADS)
    s = fma(x[i], y[i], s);
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void k_dot_final(const double* __restrict__ part, double* __restrict__ out) {
  const double s = reduce_partials(part, DOT_BLOCKS);
  if (threadIdx.x == 0) *out = s;
}
__global__ void k_axpby(double a, const double* __restrict__ x, double b, double* __restrict__ y, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = b == 0.0 ? a * x[i] : fma(a, x[i], b * y[i]);
}
}  // namespace
}  // namespace sfcdd

extern "C" int sfcdd_vec_dot(const double* x_dev, const double* y_dev, int64_t n, double* out_host, void* stream) {
  using namespace sfcdd;
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(n >= 0 && out_host, SFCDD_EVALUE, "bad dot arguments");
  cudaStream_t st = (cudaStream_t)stream;
  static thread_local double* buf = nullptr;  // DOT_BLOCKS partials + result (per thread, per process)
  static thread_local int buf_dev = -1;
  int dev = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  if (!buf || buf_dev != dev) {
    CUDA_CHECK(cudaMalloc(&buf, (DOT_BLOCKS + 1) * 8));
    buf_dev = dev;
  }
  k_dot_part<<<DOT_BLOCKS, VEC_THREADS, 0, st>>>(x_dev, y_dev, n, buf);
  k_dot_final<<<1, VEC_THREADS, 0, st>>>(buf, buf + DOT_BLOCKS);
  CUDA_CHECK(cudaMemcpyAsync(out_host, buf + DOT_BLOCKS, 8, cudaMemcpyDeviceToHost, st));
  CUDA_CHECK(cudaStreamSynchronize(st));
  SFCDD_API_END
}

extern "C" int sfcdd_vec_axpby(double a, const double* x_dev, double b, double* y_dev, int64_t n, void* stream) {
  using namespace sfcdd;
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(n >= 0, SFCDD_EVALUE, "bad axpby arguments");
  if (n == 0) return SFCDD_OK;
  const unsigned blocks = (unsigned)std::min<int64_t>(4 * 148, (n + VEC_THREADS - 1) / VEC_THREADS);
  k_axpby<<<blocks, VEC_THREADS, 0, (cudaStream_t)stream>>>(a, x_dev, b, y_dev, n);
  CUDA_CHECK(cudaGetLastError());
  SFCDD_API_END
}

// ================================================ device-driven shard PCG
// Multi-GPU (VERDICT r1 "next" 4): one rank's balanced-Schwarz
// PCG (krylov.py:257-291 over schwarz.py:103-118) with every exchange and
// every scalar on the device -- NCCL point-to-point for the halo / overlap
// / foreign-solution exchanges, NCCL allgathers for the Bank-Holst coarse
// restrictions (every rank then solves the full coarse problem) and for the
// CG scalar partials (summed in rank order on the device, so all ranks take
// bitwise identical decisions) -- captured ONCE as a CUDA graph whose
// iteration loop is a conditional WHILE node: a solve is one graph launch,
// with no host round trip per iteration.  Same step order and exchange
// plans as distributed.pcg_program (the host-driven reference
// implementation of this program, kept for lockstep and gloo tests).
// NCCL is loaded with dlopen (libnccl.so.2, the one torch already loaded
// when present), so the library itself has no link dependency on it.
#include <dlfcn.h>
#include <nccl.h>

namespace sfcdd {
namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.AllGather &&
             api.GroupStart && api.GroupEnd && api.GetErrorString;
  });
  return api;
}

#define NCCL_CHECK(expr)                                                                       \
  do {                                                                                         \
    ncclResult_t _r = (expr);                                                                  \
    if (_r != ncclSuccess)                                                                     \
      throw ::sfcdd::Error(SFCDD_ECUDA, std::string("NCCL: ") + nccl().GetErrorString(_r));  \
  } while (0)

// device scalars of the sharded PCG
struct ShState {
  double rz, pap, alpha, beta, h0, tol;
  int32_t k, done, conv, brk, max_iters, pad;
};

__device__ __forceinline__ double rank_sum(const double* v, int world) {
  double s = 0.0;
  for (int i = 0; i < world; ++i) s += v[i];  // rank order: identical on every rank
  return s;
}

struct ShParams {
  double tol;
  int32_t max_iters, pad;
};
__global__ void k_sc_start(ShState* st, const ShParams* prm) {
  st->tol = prm->tol;
  st->max_iters = prm->max_iters;
  st->k = st->done = st->conv = st->brk = 0;
  st->rz = st->pap = st->alpha = st->beta = st->h0 = 0.0;
}
// ||r0|| (krylov.py:267-271)
__global__ void k_sc_r0(ShState* st, const double* all, int world, double* hist) {
  const double h0 = sqrt(rank_sum(all, world));
  st->h0 = h0;
  hist[0] = h0;
  if (h0 <= st->tol * h0) st->done = st->conv = 1;
}
__global__ void k_sc_rz0(ShState* st, const double* all, int world) { st->rz = rank_sum(all, world); }
// alpha = rz / p.Ap; nonpositive curvature stops the loop (krylov.py:276-281)
__global__ void k_sc_alpha(ShState* st, const double* all, int world) {
  const double pap = rank_sum(all, world);
  st->pap = pap;
  if (!(pap > 0.0)) {
    st->brk = 1;
    st->done = 1;
  } else {
    st->alpha = st->rz / pap;
  }
}
// history and stopping (krylov.py:283-286); sets the WHILE condition
__global__ void k_sc_rr(ShState* st, const double* all, int world, double* hist, cudaGraphConditionalHandle h) {
  if (!st->brk) {
    const int k = st->k + 1;
    st->k = k;
    const double nrm = sqrt(rank_sum(all, world));
    hist[k] = nrm;
    if (nrm <= st->tol * st->h0) {
      st->conv = 1;
      st->done = 1;
    } else if (k >= st->max_iters) {
      st->done = 1;
    }
  }
  cudaGraphSetConditional(h, st->done ? 0u : 1u);
}
// beta = rz' / rz (krylov.py:287-290)
__global__ void k_sc_beta(ShState* st, const double* all, int world) {
  const double rzn = rank_sum(all, world);
  st->beta = rzn / st->rz;
  st->rz = rzn;
}
__global__ void k_copy(const double* __restrict__ a, double* __restrict__ b, int64_t g0, int64_t g1) {
  const int64_t g = g0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < g1) b[g] = a[g];
}
// allgathered, padded coarse restrictions -> the full N0 vector
__global__ void k_unpad(const double* __restrict__ all, const int64_t* __restrict__ off, int world, int64_t mx,
                        double* __restrict__ out) {
  const int h = blockIdx.y;
  const int64_t cnt = off[h + 1] - off[h];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
    out[off[h] + i] = all[h * mx + i];
}

}  // namespace

struct ShardExchange {
  std::vector<int32_t> peers;
  std::vector<int64_t> ns, nr, soff, roff;
  int64_t stot = 0, rtot = 0;
  int64_t *sidx = nullptr, *ridx = nullptr;
  double *sbuf = nullptr, *rbuf = nullptr;
};

struct ShardRuntime {
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  bool coll = false;  // collectives through NCCL (world > 1, or forced at world 1 with an id: tests)
  ShardExchange ex[3];  // 0 halo, 1 ext (overlap extension of t), 2 xy (foreign solutions)
  std::vector<int64_t> agg_off;  // allgather layout (world + 1)
  int64_t agg_max = 0;
  int64_t* d_agg_off = nullptr;
  double *gsend = nullptr, *gall = nullptr, *c1 = nullptr, *c2 = nullptr;
  double *spart = nullptr, *sall = nullptr;
  double *r = nullptr, *z = nullptr, *w = nullptr, *t = nullptr, *pold = nullptr, *pnew = nullptr, *ap = nullptr;
  double *y0 = nullptr, *y0b = nullptr;
  ShState* st = nullptr;
  ShParams* prm = nullptr;  // tol / max_iters of the next solve (read by the graph's first kernel)
  ShParams prm_host{};
  double* hist = nullptr;
  int32_t hist_cap = 0;
  cudaGraphExec_t graph = nullptr;
  const double* gb = nullptr;
  double* gx = nullptr;
  int64_t k_pro = 0, k_body = 0, nk = 0;  // our kernels: prologue, one loop iteration (capture counter)
  std::vector<void*> owned;
  ~ShardRuntime() {
    if (graph) cudaGraphExecDestroy(graph);
    for (void* p : owned) cudaFree(p);
    if (comm && nccl().ok) nccl().CommDestroy(comm);
  }
  template <class T>
  T* alloc(int64_t n) {
    T* p = nullptr;
    CUDA_CHECK(cudaMalloc(&p, std::max<int64_t>(n, 1) * sizeof(T)));
    owned.push_back(p);
    return p;
  }
};

void destroy_shard_runtime(ShardRuntime* r) { delete r; }

namespace {

ShardRuntime& runtime(sfcdd_op* op) {
  SFCDD_REQUIRE(op && op->ready && op->shard_count > 0, SFCDD_EVALUE, "needs a set-up shard-mode operator");
  if (!op->srt) {
    op->srt = new ShardRuntime();
    op->srt->agg_off.assign(2, 0);
  }
  return *op->srt;
}

// one exchange: pack -> grouped send / recv -> unpack (no-op without peers)
void sh_exchange(sfcdd_op* op, ShardRuntime& R, int kind, double* buf, cudaStream_t st) {
  ShardExchange& E = R.ex[kind];
  if (E.peers.empty()) return;
  if (E.stot) k_pack<<<nblocks(E.stot, 256), 256, 0, st>>>(buf, E.sidx, E.stot, E.sbuf);
  R.nk += (E.stot > 0) + (E.rtot > 0);
  NCCL_CHECK(nccl().GroupStart());
  for (size_t i = 0; i < E.peers.size(); ++i) {
    if (E.ns[i]) NCCL_CHECK(nccl().Send(E.sbuf + E.soff[i], E.ns[i], ncclDouble, E.peers[i], R.comm, st));
    if (E.nr[i]) NCCL_CHECK(nccl().Recv(E.rbuf + E.roff[i], E.nr[i], ncclDouble, E.peers[i], R.comm, st));
  }
  NCCL_CHECK(nccl().GroupEnd());
  if (E.rtot) k_unpack<<<nblocks(E.rtot, 256), 256, 0, st>>>(E.rbuf, E.ridx, E.rtot, buf);
  (void)op;
}

// rank partial (one double at spart) -> sall[world]
const double* sh_scalars(ShardRuntime& R, cudaStream_t st) {
  if (!R.coll) return R.spart;
  NCCL_CHECK(nccl().AllGather(R.spart, R.sall, 1, ncclDouble, R.comm, st));
  return R.sall;  // rank order (identical sum on every rank)
}

// owned coarse restrictions (at gsend) -> full N0 vector out
void sh_coarse_gather(sfcdd_op* op, ShardRuntime& R, double* out, cudaStream_t st) {
  if (!R.coll) {
    CUDA_CHECK(cudaMemcpyAsync(out, R.gsend, (size_t)op->n0 * 8, cudaMemcpyDeviceToDevice, st));
    return;
  }
  NCCL_CHECK(nccl().AllGather(R.gsend, R.gall, R.agg_max, ncclDouble, R.comm, st));
  k_unpad<<<dim3(nblocks(R.agg_max, 256), R.world), 256, 0, st>>>(R.gall, R.d_agg_off, R.world, R.agg_max, out);
  R.nk += 1;
}

void sh_coarse_solve(sfcdd_op* op, ShardRuntime& R, const double* c, double* y, cudaStream_t st) {
  R.nk += 1;
  if (!op->ainv) {
    op->coarse_dag->solve(c, st);
    CUDA_CHECK(cudaMemcpyAsync(y, op->coarse_dag->xy(), (size_t)op->n0 * 8, cudaMemcpyDeviceToDevice, st));
  } else {
    k_gemv_c<<<nblocks(op->n0, VEC_THREADS / 32), VEC_THREADS, (size_t)op->n0 * 8, st>>>(op->ainv, c, op->n0, y);
  }
}

// z = C^{-1} g with rz partial = g.z (schwarz.py:103-118 balanced branch);
// cagg at gsend holds the owned R0 g
void sh_apply(sfcdd_op* op, ShardRuntime& R, const double* g, cudaStream_t st) {
  const ShardRange SR = shard_range(op);
  sh_coarse_gather(op, R, R.c1, st);
  sh_coarse_solve(op, R, R.c1, R.y0, st);
  k_sh_tvec<<<nblocks(SR.g1 - SR.g0, VEC_THREADS), VEC_THREADS, 0, st>>>(g, R.y0, op->agg, stencil_of(op), SR.g0,
                                                                         SR.g1, R.t);
  sh_exchange(op, R, 1, R.t, st);
  op->dag->solve(R.t, st);
  sh_exchange(op, R, 2, op->dag->xy(), st);
  CUDA_CHECK(sfcdd_shard_combine(op, R.w, st) == SFCDD_OK ? cudaSuccess : cudaErrorUnknown);
  sh_exchange(op, R, 0, R.w, st);
  k_sh_stencil_chunks<<<SR.ch1 - SR.ch0, VEC_THREADS, 0, st>>>(R.w, stencil_of(op), chunks_of(op), SR.ch0,
                                                               op->part_b);
  k_agg_sums<<<nblocks(SR.a1 - SR.a0, 128), 128, 0, st>>>(op->part_b, op->agg_ptr, SR.a0, SR.a1, R.gsend);
  sh_coarse_gather(op, R, R.c2, st);
  sh_coarse_solve(op, R, R.c2, R.y0b, st);
  k_sh_finalize<<<SR.ch1 - SR.ch0, VEC_THREADS, 0, st>>>(R.w, R.y0, R.y0b, chunks_of(op), SR.ch0,
                                                         mode_of(op->variant), R.z, g, op->part_a);
  k_sum_range<<<1, VEC_THREADS, 0, st>>>(op->part_a, SR.ch0, SR.ch1, R.spart);
  R.nk += 8;  // tvec, DAG, combine, stencil chunks, aggregate sums, finalize, range sum (+ DAG counter reset)
}

// first half of an iteration: p = z + beta p_old, Ap, alpha, x/r update,
// ||r||, R0 r; k_sc_rr sets the loop condition
void sh_half(sfcdd_op* op, ShardRuntime& R, double* x, cudaGraphConditionalHandle h, cudaStream_t st) {
  const ShardRange SR = shard_range(op);
  sh_exchange(op, R, 0, R.z, st);
  sh_exchange(op, R, 0, R.pold, st);
  k_sh_pm<<<SR.ch1 - SR.ch0, VEC_THREADS, 0, st>>>(R.z, R.pold, 0.0, stencil_of(op), chunks_of(op), SR.ch0,
                                                   R.pnew, R.ap, op->part_a, &R.st->beta);
  k_sum_range<<<1, VEC_THREADS, 0, st>>>(op->part_a, SR.ch0, SR.ch1, R.spart);
  k_sc_alpha<<<1, 1, 0, st>>>(R.st, sh_scalars(R, st), R.world);
  k_sh_update<<<SR.ch1 - SR.ch0, VEC_THREADS, 0, st>>>(x, R.r, R.pnew, R.ap, 0.0, chunks_of(op), SR.ch0, op->part_b,
                                                       op->part_c, &R.st->alpha, &R.st->brk);
  k_sum_range<<<1, VEC_THREADS, 0, st>>>(op->part_b, SR.ch0, SR.ch1, R.spart);
  k_agg_sums<<<nblocks(SR.a1 - SR.a0, 128), 128, 0, st>>>(op->part_c, op->agg_ptr, SR.a0, SR.a1, R.gsend);
  k_sc_rr<<<1, 1, 0, st>>>(R.st, sh_scalars(R, st), R.world, R.hist, h);
  R.nk += 8;  // pm, range sum, alpha, update, range sum, aggregate sums, rr
}

// the whole solve as one graph: start, r0, z0 = C^{-1} r0, first half
// iteration, then WHILE (not done) { z = C^{-1} r, beta, p_old <- p, half }
void sh_build_graph(sfcdd_op* op, ShardRuntime& R, const double* b, double* x) {
  const ShardRange SR = shard_range(op);
  cudaStream_t cs = op->own_stream;
  cudaGraph_t graph;
  CUDA_CHECK(cudaGraphCreate(&graph, 0));
  cudaGraphConditionalHandle h;
  CUDA_CHECK(cudaGraphConditionalHandleCreate(&h, graph, 0, cudaGraphCondAssignDefault));
  // prologue
  CUDA_CHECK(cudaStreamBeginCaptureToGraph(cs, graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  R.nk = 0;
  k_sc_start<<<1, 1, 0, cs>>>(R.st, R.prm);
  sh_exchange(op, R, 0, x, cs);
  k_sh_residual<<<SR.ch1 - SR.ch0, VEC_THREADS, 0, cs>>>(b, x, stencil_of(op), chunks_of(op), SR.ch0, R.r,
                                                         op->part_b, op->part_c);
  k_sum_range<<<1, VEC_THREADS, 0, cs>>>(op->part_b, SR.ch0, SR.ch1, R.spart);
  k_agg_sums<<<nblocks(SR.a1 - SR.a0, 128), 128, 0, cs>>>(op->part_c, op->agg_ptr, SR.a0, SR.a1, R.gsend);
  k_sc_r0<<<1, 1, 0, cs>>>(R.st, sh_scalars(R, cs), R.world, R.hist);
  sh_apply(op, R, R.r, cs);
  k_sc_rz0<<<1, 1, 0, cs>>>(R.st, sh_scalars(R, cs), R.world);
  CUDA_CHECK(cudaMemsetAsync(R.pold, 0, (size_t)op->n * 8, cs));
  sh_half(op, R, x, h, cs);
  R.nk += 6;  // start, residual, range sum, aggregate sums, r0, rz0
  R.k_pro = R.nk;
  // the loop node after the prologue
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  cudaStreamCaptureStatus cst;
  CUDA_CHECK(cudaStreamGetCaptureInfo(cs, &cst, nullptr, nullptr, &deps, &ndeps));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t loop;
  CUDA_CHECK(cudaGraphAddNode(&loop, graph, deps, ndeps, &cp));
  CUDA_CHECK(cudaStreamUpdateCaptureDependencies(cs, &loop, 1, cudaStreamSetCaptureDependencies));
  cudaGraph_t tmp;
  CUDA_CHECK(cudaStreamEndCapture(cs, &tmp));
  // loop body
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CUDA_CHECK(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  R.nk = 0;
  sh_apply(op, R, R.r, cs);
  k_sc_beta<<<1, 1, 0, cs>>>(R.st, sh_scalars(R, cs), R.world);
  k_copy<<<nblocks(op->n, 256), 256, 0, cs>>>(R.pnew, R.pold, 0, op->n);
  sh_half(op, R, x, h, cs);
  R.nk += 2;
  R.k_body = R.nk;
  CUDA_CHECK(cudaStreamEndCapture(cs, &tmp));
  if (R.graph) CUDA_CHECK(cudaGraphExecDestroy(R.graph));
  CUDA_CHECK(cudaGraphInstantiate(&R.graph, graph, 0));
  CUDA_CHECK(cudaGraphDestroy(graph));
  R.gb = b;
  R.gx = x;
}

}  // namespace
}  // namespace sfcdd

extern "C" int sfcdd_nccl_unique_id(void* id_out) {
  SFCDD_API_BEGIN
  SFCDD_REQUIRE(id_out, SFCDD_EVALUE, "null argument");
  SFCDD_REQUIRE(nccl().ok, SFCDD_ECUDA, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  NCCL_CHECK(nccl().GetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  SFCDD_API_END
}

extern "C" int sfcdd_shard_attach(sfcdd_op* op, const void* nccl_id, int32_t rank, int32_t world,
                                  const int64_t* agg_counts) {
  SFCDD_API_BEGIN
  ShardRuntime& R = runtime(op);
  SFCDD_REQUIRE(world >= 1 && rank >= 0 && rank < world, SFCDD_EVALUE, "invalid rank / world");
  CUDA_CHECK(cudaSetDevice(op->device));
  R.rank = rank;
  R.world = world;
  if (world > 1 || nccl_id) {  // a world-1 communicator runs the same collectives (tests)
    SFCDD_REQUIRE(nccl_id, SFCDD_EVALUE, "world > 1 needs an NCCL unique id");
    R.coll = true;
    SFCDD_REQUIRE(nccl().ok, SFCDD_ECUDA, "libnccl.so.2 could not be loaded");
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    NCCL_CHECK(nccl().CommInitRank(&R.comm, world, id, rank));
  }
  R.agg_off.assign(world + 1, 0);
  for (int h = 0; h < world; ++h) {
    R.agg_off[h + 1] = R.agg_off[h] + agg_counts[h];
    R.agg_max = std::max<int64_t>(R.agg_max, agg_counts[h]);
  }
  SFCDD_REQUIRE(R.agg_off[world] == op->n0, SFCDD_EVALUE, "aggregate counts must sum to N0");
  const ShardRange SR = shard_range(op);
  SFCDD_REQUIRE(agg_counts[rank] == SR.a1 - SR.a0, SFCDD_EVALUE, "own aggregate count mismatch");
  R.d_agg_off = R.alloc<int64_t>(world + 1);
  CUDA_CHECK(cudaMemcpy(R.d_agg_off, R.agg_off.data(), (world + 1) * 8, cudaMemcpyHostToDevice));
  R.gsend = R.alloc<double>(std::max<int64_t>(R.agg_max, op->n0));
  R.gall = R.alloc<double>(R.agg_max * world);
  R.c1 = R.alloc<double>(op->n0);
  R.c2 = R.alloc<double>(op->n0);
  R.spart = R.alloc<double>(1);
  R.sall = R.alloc<double>(world);
  for (double** v : {&R.r, &R.z, &R.w, &R.t, &R.pold, &R.pnew, &R.ap}) {
    *v = R.alloc<double>(op->n);
    CUDA_CHECK(cudaMemset(*v, 0, (size_t)op->n * 8));
  }
  R.y0 = R.alloc<double>(op->n0);
  R.y0b = R.alloc<double>(op->n0);
  R.st = R.alloc<ShState>(1);
  R.prm = R.alloc<ShParams>(1);
  if (op->ainv && (size_t)op->n0 * 8 > 48 * 1024)
    CUDA_CHECK(cudaFuncSetAttribute(k_gemv_c, cudaFuncAttributeMaxDynamicSharedMemorySize, COARSE_DENSE_MAX * 8));
  SFCDD_API_END
}

// kind 0 halo, 1 ext, 2 xy: the (peer, send indices, recv indices) lists of
// distributed.build_plans, concatenated per kind (peers ascending)
extern "C" int sfcdd_shard_set_exchange(sfcdd_op* op, int32_t kind, int32_t npeer, const int32_t* peers,
                                        const int64_t* nsend, const int64_t* send_idx, const int64_t* nrecv,
                                        const int64_t* recv_idx) {
  SFCDD_API_BEGIN
  ShardRuntime& R = runtime(op);
  SFCDD_REQUIRE(kind >= 0 && kind < 3, SFCDD_EVALUE, "exchange kind must be 0, 1 or 2");
  SFCDD_REQUIRE(npeer == 0 || R.world > 1, SFCDD_EVALUE, "exchanges need world > 1");
  ShardExchange& E = R.ex[kind];
  E = ShardExchange();
  for (int i = 0; i < npeer; ++i) {
    SFCDD_REQUIRE(peers[i] >= 0 && peers[i] < R.world && peers[i] != R.rank, SFCDD_EVALUE, "invalid peer");
    E.peers.push_back(peers[i]);
    E.ns.push_back(nsend[i]);
    E.nr.push_back(nrecv[i]);
    E.soff.push_back(E.stot);
    E.roff.push_back(E.rtot);
    E.stot += nsend[i];
    E.rtot += nrecv[i];
  }
  E.sidx = R.alloc<int64_t>(E.stot);
  E.ridx = R.alloc<int64_t>(E.rtot);
  E.sbuf = R.alloc<double>(E.stot);
  E.rbuf = R.alloc<double>(E.rtot);
  if (E.stot) CUDA_CHECK(cudaMemcpy(E.sidx, send_idx, E.stot * 8, cudaMemcpyHostToDevice));
  if (E.rtot) CUDA_CHECK(cudaMemcpy(E.ridx, recv_idx, E.rtot * 8, cudaMemcpyHostToDevice));
  if (R.graph) CUDA_CHECK(cudaGraphExecDestroy(R.graph));
  R.graph = nullptr;
  SFCDD_API_END
}

// one sharded PCG solve (x holds x0 on entry; the owned segment of the
// solution on exit); res_hist_host: max_iters + 1 doubles
extern "C" int sfcdd_shard_pcg(sfcdd_op* op, const double* b, double* x, double tol, int32_t max_iters,
                               double* res_hist_host, int32_t* iters, int32_t* converged, void* stream) {
  SFCDD_API_BEGIN
  ShardRuntime& R = runtime(op);
  SFCDD_REQUIRE(R.st, SFCDD_EVALUE, "call sfcdd_shard_attach first");
  SFCDD_REQUIRE(tol > 0 && max_iters >= 1, SFCDD_EVALUE, "need tol > 0 and max_iters >= 1");
  CUDA_CHECK(cudaSetDevice(op->device));
  OpScope scope(op, (cudaStream_t)stream);
  cudaStream_t st = scope.stream();
  if (R.hist_cap < max_iters + 1) {
    R.hist = R.alloc<double>(max_iters + 1);
    R.hist_cap = max_iters + 1;
    if (R.graph) CUDA_CHECK(cudaGraphExecDestroy(R.graph));
    R.graph = nullptr;
  }
  if (!R.graph || R.gb != b || R.gx != x) sh_build_graph(op, R, b, x);
  R.prm_host = ShParams{tol, max_iters, 0};
  CUDA_CHECK(cudaMemcpyAsync(R.prm, &R.prm_host, sizeof(ShParams), cudaMemcpyHostToDevice, st));
  CUDA_CHECK(cudaGraphLaunch(R.graph, st));
  ShState hs;
  CUDA_CHECK(cudaMemcpyAsync(&hs, R.st, sizeof(ShState), cudaMemcpyDeviceToHost, st));
  CUDA_CHECK(cudaStreamSynchronize(st));
  if (res_hist_host) CUDA_CHECK(cudaMemcpy(res_hist_host, R.hist, (size_t)(hs.k + 1) * 8, cudaMemcpyDeviceToHost));
  *iters = hs.k;
  *converged = hs.conv;
  // kernels launched by this solve (graph kernel nodes: the prologue holds the
  // first half iteration, every further iteration is one body execution)
  op->stats.reserved[7] = R.k_pro + (int64_t)std::max(0, hs.k - 1) * R.k_body;
  if (hs.brk) throw Error(SFCDD_EBREAKDOWN, "nonpositive curvature at iteration " + std::to_string(hs.k + 1));
  SFCDD_API_END
}
