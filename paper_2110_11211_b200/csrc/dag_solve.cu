// Batched block-inverse supernodal triangular solves as ONE persistent
// dataflow kernel (forward + backward sweeps of all subdomain factors).
//
// Replaces the per-subdomain SuperLU gstrs calls of the reference's
// one-level Schwarz sweep (schwarz.py:81-101 -> linalg.py:67-72) together
// with the R_i gather (schwarz.py:82).  Design:
//  * every supernode stores M = [L_JJ^{-1}; L_BJ L_JJ^{-1}], so each
//    supernode is a dependency-free GEMV (forward) / GEMV^T (backward);
//  * factor trees are cut into fragments whose factor bytes + metadata are
//    ONE contiguous blob, moved HBM -> shared memory by a single
//    cp.async.bulk (TMA bulk copy) completing on an mbarrier;
//  * two blob buffers per CTA: the NEXT task's blob is in flight while the
//    current one computes; big supernodes are streamed column-chunk by
//    column-chunk through a 3-stage ring of bulk copies;
//  * all gathers of a fragment (right-hand side, external child updates,
//    ancestor solution values) happen once in a prologue, the level loop runs
//    entirely out of shared memory, results leave in one epilogue;
//  * CTAs pull tasks from a global queue in topological order and wait on
//    per-fragment counters (acquire/release) -- no grid barrier, no host
//    round trip, deadlock-free because a task only waits on earlier tasks;
//  * multifrontal update vectors are summed by the parent in fixed child
//    order, so results are bitwise reproducible run to run.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

#include "common.h"
#include "dag_solve.h"

namespace sfcdd {

namespace {

constexpr int DAG_THREADS = 256;
constexpr int NWARP = DAG_THREADS / 32;
constexpr int NSTAGE = 6;       // big-supernode chunk ring depth (ring = both blob buffers)
constexpr int RMAX = 8;         // rows per thread in the big forward (s+m <= 2048)
constexpr int SMALL_ROWS = SMALL_MAX_S / 32;

struct DagArgs {
  const TaskDev* tasks;
  int32_t ntask;
  int32_t nfrag;
  const uint8_t* blobs;
  const FactorDev* factors;
  const double* rhs;
  double* xy;
  double* upd;
  int32_t* ctr;  // [0] queue head | fwd_cnt[nfrag] | fwd_done[nfrag] | bwd_done[nfrag]
  int32_t blob_max;
  int32_t chunk_bytes;
  const int32_t* skip;  // optional: nonzero -> whole solve skipped (PCG done)
  unsigned long long* trace;  // optional: per task {sm, t_top, t_deps, t_data, t_end} (ns)
  unsigned long long* ptrace;  // optional: per task 16 clock64 stamps inside run_small
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// TMA bulk copy global -> shared, completion signalled on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ int32_t ld_acquire(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(int32_t* p, int32_t v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int64_t gidx(const FactorDev& F, int32_t ro) {
  int64_t g = F.gstart + ro;
  return g >= F.gmod ? g - F.gmod : g;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int64_t coloff(int64_t s, int64_t m, int64_t k) { return k * (s + m) - k * (k - 1) / 2; }
// packed offsets of one supernode fit 32 bits (s+m <= 2048)
__device__ __forceinline__ int coloff32(int s, int m, int k) { return k * (s + m) - ((k * (k - 1)) >> 1); }

// barrier of the 256 compute threads (warp 8 is the scheduler)
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// Gather n values with all their global loads in flight before any store
// (8 per thread per round): one memory latency instead of one per element.
template <typename Load, typename Store>
__device__ __forceinline__ void batched_gather(int n, Load ld, Store st) {
  constexpr int RB = 8;
  for (int base = 0; base < n; base += RB * DAG_THREADS) {
    double v[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int c = base + threadIdx.x + DAG_THREADS * r;
      v[r] = c < n ? ld(c) : 0.0;
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int c = base + threadIdx.x + DAG_THREADS * r;
      if (c < n) st(c, v[r]);
    }
  }
}

// ===================================================== small fragments
__device__ __forceinline__ int lo16(int32_t v) { return (int)((uint32_t)v & 0xffffu); }
__device__ __forceinline__ int hi16(int32_t v) { return (int)((uint32_t)v >> 16); }

// forward row i of a supernode: y_i (i < s) or u_i = f_i - (W f_J)_i.
// M[k][i-k] sits at coloff(k) + i - k; successive k advance by s+m-1-k.
__device__ __forceinline__ void fwd_row(const int32_t* R, const double* vals, double* S, int i) {
  const int s = R[R_S], m = R[R_M];
  if (i >= s + m) return;
  double* f = S + R[R_SCR];
  const double* M = vals + R[R_VAL];
  const int kmax = i < s ? i : s - 1;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int idx = i, step = s + m - 1;
  int k = 0;
  for (; k + 3 <= kmax; k += 4) {
    const int i1 = idx + step, i2 = i1 + step - 1, i3 = i2 + step - 2;
    a0 = fma(M[idx], f[k], a0);
    a1 = fma(M[i1], f[k + 1], a1);
    a2 = fma(M[i2], f[k + 2], a2);
    a3 = fma(M[i3], f[k + 3], a3);
    idx = i3 + step - 3;
    step -= 4;
  }
  for (; k <= kmax; ++k) {
    a0 = fma(M[idx], f[k], a0);
    idx += step;
    --step;
  }
  const double acc = (a0 + a1) + (a2 + a3);
  if (i < s)
    S[R[R_CPOS] + i] = acc;  // y_J
  else
    f[i] -= acc;  // u = f_B - W f_J (only f[0:s) is read by other rows)
}

// backward column k of a supernode by one warp (lanes = rows, warp reduce)
__device__ __forceinline__ void bwd_col(const int32_t* R, const double* vals, double* S, int k, int lane) {
  const int s = R[R_S], m = R[R_M];
  const double* v = S + R[R_SCR];
  const double* col = vals + R[R_VAL] + coloff(s, m, k);
  const int len = s + m - k;
  double a0 = 0.0, a1 = 0.0;
  int t = lane;
  for (; t + 32 < len; t += 64) {
    a0 = fma(col[t], v[k + t], a0);
    a1 = fma(col[t + 32], v[k + t + 32], a1);
  }
  if (t < len) a0 = fma(col[t], v[k + t], a0);
  const double x = warp_sum(a0 + a1);
  if (lane == 0) S[R[R_CPOS] + k] = x;
}

// packed item: lanes carry the rows of `cnt` consecutive small supernodes
// starting at record x (sum of fronts <= 32).  Returns the lane's record
// (or null), its row and the first lane of its segment; *smax = max s.
__device__ __forceinline__ const int32_t* packed_map(const int32_t* recs, int x, int cnt, int lane, int& row,
                                                     int& seg_lo, int* smax) {
  int fr = 0, s_own = 0;
  if (lane < cnt) {
    const int32_t* R = recs + R_WORDS * (x + lane);
    s_own = R[R_S];
    fr = s_own + R[R_M];
  }
  int incl = fr;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += o;
  }
  const unsigned starts = __reduce_or_sync(0xffffffffu, lane < cnt ? (1u << (incl - fr)) : 0u);
  const int total = __shfl_sync(0xffffffffu, incl, cnt - 1);
  if (smax) *smax = (int)__reduce_max_sync(0xffffffffu, (unsigned)s_own);
  if (lane >= total) {
    row = 0;
    seg_lo = lane;
    return nullptr;
  }
  const unsigned upto = starts & ((2u << lane) - 1u);
  seg_lo = 31 - __clz(upto);
  row = lane - seg_lo;
  return recs + R_WORDS * (x + __popc(upto) - 1);
}

// backward of packed small supernodes: lanes = rows, x_k by segmented scans
__device__ __forceinline__ void bwd_packed(const int32_t* recs, const double* vals, double* S, int x, int cnt,
                                           unsigned mask, int lane) {
  const unsigned upto = mask & ((2u << lane) - 1u);
  const int seg = __popc(upto) - 1;
  const int seg_lo = 31 - __clz(upto);
  const int i = lane - seg_lo;
  const int32_t* R = seg < cnt ? recs + R_WORDS * (x + seg) : nullptr;
  const int s = R ? R[R_S] : 0, m = R ? R[R_M] : 0;
  const int smax = (int)__reduce_max_sync(0xffffffffu, (unsigned)s);
  const double vi = R ? S[R[R_SCR] + i] : 0.0;
  const double* M = R ? vals + R[R_VAL] : vals;
  const bool seg_end = R && i == s + m - 1;
  for (int k = 0; k < smax; ++k) {
    double val = (R && k < s && i >= k) ? M[coloff(s, m, k) + (i - k)] * vi : 0.0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double o = __shfl_up_sync(0xffffffffu, val, d);
      if (lane - d >= seg_lo) val += o;
    }
    if (seg_end && k < s) S[R[R_CPOS] + k] = val;
  }
}

__device__ __forceinline__ void run_small(const int32_t* h, bool fwd, double* S, const DagArgs& A, const FactorDev& F,
                          int lane, int warp, unsigned long long* pt) {
  const double* vals = reinterpret_cast<const double*>(reinterpret_cast<const uint8_t*>(h) + h[H_VAL_OFF]);
  const int nlev = h[H_NLEV];
  auto stamp = [&](int i) {
    if (pt && threadIdx.x == 0 && i < 15) pt[i] = clock64();
  };
  if (pt && threadIdx.x == 0) pt[15] = nlev;
  stamp(0);
  const int32_t* levtab = h + h[H_LEVELS];
  const int32_t* runs = h + h[H_RUNS];
  const int32_t* gp = h + h[H_GPAIRS];
  const int32_t* bp = h + h[H_BPAIRS];
  const int2* items = reinterpret_cast<const int2*>(h + h[H_ITEMS]);
  const int32_t* recs = h + h[H_REC];
  const int32_t* cols = h + h[H_COLS];
  const int32_t* colpos = h + h[H_COLPOS];
  const int ncol = h[H_NCOL];
  double* xy = A.xy + F.xy_off;
  if (fwd) {
    for (int i = threadIdx.x; i < h[H_SCRATCH]; i += DAG_THREADS) S[i] = 0.0;
    csync();
    {  // one batched gather: right-hand side at the columns + external child updates
      const int32_t* eu = h + h[H_EXTU];
      const int nu = h[H_NEXTU], ub = h[H_EXTU_BASE];
      batched_gather(ncol + nu,
                     [&](int c) { return c < ncol ? __ldg(A.rhs + gidx(F, cols[c])) : __ldcg(A.upd + eu[c - ncol]); },
                     [&](int c, double v) { S[c < ncol ? lo16(colpos[c]) : ub + (c - ncol)] = v; });
    }
    csync();
    stamp(1);
    for (int lv = 0; lv < nlev; ++lv) {
      const int32_t* L = levtab + L_WORDS * lv;
      // phase 1: multifrontal assembly in gather form (fixed child order per dst)
      if (L[L_RUN1] > L[L_RUN0]) {
        for (int r = L[L_RUN0] + threadIdx.x; r < L[L_RUN1]; r += DAG_THREADS) {
          const int p0 = runs[r], p1 = runs[r + 1];
          const int dst = lo16(gp[p0]);
          double acc = S[dst];
          for (int p = p0; p < p1; ++p) acc += S[hi16(gp[p])];
          S[dst] = acc;
        }
        csync();
      }
      if (lv < 6) stamp(2 + 2 * lv);
      // phase 2: row items over all warps (lanes = rows)
      for (int it = L[L_FW + warp]; it < L[L_FW + warp + 1]; ++it) {
        const int2 item = items[it];
        const int cnt = item.x >> 16;
        if (cnt == 0) {
          fwd_row(recs + R_WORDS * item.x, vals, S, 32 * item.y + lane);
        } else {
          const unsigned upto = (unsigned)item.y & ((2u << lane) - 1u);
          const int seg = __popc(upto) - 1;
          if (seg < cnt) fwd_row(recs + R_WORDS * ((item.x & 0xffff) + seg), vals, S, lane - (31 - __clz(upto)));
        }
      }
      csync();
      if (lv < 6) stamp(3 + 2 * lv);
    }
    for (int c = threadIdx.x; c < ncol; c += DAG_THREADS) __stcg(xy + cols[c], S[hi16(colpos[c])]);
    if (h[H_TOP_UPD] >= 0) {
      const int32_t* R = recs + R_WORDS * h[H_TOP];
      const double* u = S + R[R_SCR] + R[R_S];
      for (int a = threadIdx.x; a < R[R_M]; a += DAG_THREADS) __stcg(A.upd + h[H_TOP_UPD] + a, u[a]);
    }
    stamp(14);
  } else {
    {  // one batched gather: y at the columns + x of the external ancestor rows
      const int32_t* ex = h + h[H_EXTX];
      const int nx = h[H_NEXTX], xb = h[H_EXTX_BASE];
      batched_gather(ncol + nx, [&](int c) { return __ldcg(xy + (c < ncol ? cols[c] : ex[c - ncol])); },
                     [&](int c, double v) { S[c < ncol ? lo16(colpos[c]) : xb + (c - ncol)] = v; });
    }
    csync();
    for (int lv = nlev - 1; lv >= 0; --lv) {
      const int32_t* L = levtab + L_WORDS * lv;
      // phase 1: v_B = -x(rows)
      if (L[L_BP1] > L[L_BP0]) {
        for (int p = L[L_BP0] + threadIdx.x; p < L[L_BP1]; p += DAG_THREADS) S[lo16(bp[p])] = -S[hi16(bp[p])];
        csync();
      }
      // phase 2: column items / packed small supernodes over all warps
      for (int it = L[L_BW + warp]; it < L[L_BW + warp + 1]; ++it) {
        const int2 item = items[it];
        if ((item.x >> 16) == 0)
          bwd_col(recs + R_WORDS * item.x, vals, S, item.y, lane);
        else
          bwd_packed(recs, vals, S, item.x & 0xffff, item.x >> 16, (unsigned)item.y, lane);
      }
      csync();
    }
    for (int c = threadIdx.x; c < ncol; c += DAG_THREADS) __stcg(xy + cols[c], S[hi16(colpos[c])]);
  }
}

// ======================================================= big supernodes
// The packed block (total = s(s+1)/2 + s m doubles, 16-byte aligned) is
// streamed in fixed chunks of CHD doubles through an NSTAGE ring of TMA bulk
// copies; a chunk may cut a column, so every column intersecting the chunk
// is processed over its in-chunk row range.
__device__ __forceinline__ void issue_chunk(uint8_t* stage, uint64_t* bar, const double* vbase, int64_t e0,
                                            int64_t e1) {
  const uint32_t bytes = (uint32_t)(((e1 - e0) * 8 + 15) & ~int64_t(15));
  mbar_expect_tx(bar, bytes);
  bulk_g2s(stage, vbase + e0, bytes, bar);
}

__device__ __forceinline__ void run_big(const uint8_t* gblob, bool fwd, uint8_t* ring, uint64_t* cbar, uint32_t& cphase,
                        double* S, const DagArgs& A, const FactorDev& F, int lane, int warp) {
  const int32_t* hg = reinterpret_cast<const int32_t*>(gblob);
  const int32_t* R = hg + __ldg(hg + H_REC);
  const int s = __ldg(R + R_S), m = __ldg(R + R_M);
  const int N = s + m;
  const double* vbase = reinterpret_cast<const double*>(gblob + __ldg(hg + H_VAL_OFF));
  const int32_t* cols = hg + __ldg(hg + H_COLS);
  const int32_t* rows = hg + __ldg(R + R_ROWS);
  double* xy = A.xy + F.xy_off;
  const int total = coloff32(s, m, s);
  const int CHD = (A.chunk_bytes / 8) & ~1;
  const int nchunk = (total + CHD - 1) / CHD;
  // kick off the first chunks before the gathers
  if (threadIdx.x == 0) {
    for (int c = 0; c < NSTAGE && c < nchunk; ++c) {
      fence_proxy_async();
      issue_chunk(ring + c * A.chunk_bytes, cbar + c, vbase, c * CHD, min(total, (c + 1) * CHD));
    }
  }
  double* xacc = S + N;  // backward partial column sums (columns may span chunks)
  if (!fwd)
    for (int k = threadIdx.x; k < s; k += DAG_THREADS) xacc[k] = 0.0;
  // gathers into shared memory: f (forward) or v (backward), length s+m
  if (fwd) {
    batched_gather(s + m, [&](int i) { return i < s ? __ldg(A.rhs + gidx(F, __ldg(cols + i))) : 0.0; },
                   [&](int i, double v) { S[i] = v; });
    csync();
    const int nch = __ldg(R + R_NCH);
    const int32_t* chr = hg + __ldg(R + R_CH);
    for (int q = 0; q < nch; ++q) {
      const int slot = __ldg(chr + CH_WORDS * q), mk = __ldg(chr + CH_WORDS * q + 1);
      const int32_t* rel = hg + __ldg(chr + CH_WORDS * q + 2);
      for (int a = threadIdx.x; a < mk; a += DAG_THREADS) S[__ldg(rel + a)] += __ldcg(A.upd + slot + a);
      csync();
    }
  } else {
    batched_gather(s + m,
                   [&](int i) { return i < s ? __ldcg(xy + __ldg(cols + i)) : -__ldcg(xy + __ldg(rows + (i - s))); },
                   [&](int i, double v) { S[i] = v; });
    csync();
  }
  double acc[RMAX];
#pragma unroll
  for (int r = 0; r < RMAX; ++r) acc[r] = 0.0;
  int k = 0, ck = 0;  // first column intersecting the current chunk and its offset
  for (int c = 0; c < nchunk; ++c) {
    const int e0 = c * CHD, e1 = min(total, e0 + CHD);
    const int st = c % NSTAGE;
    const double* stage = reinterpret_cast<const double*>(ring + st * A.chunk_bytes) - e0;  // stage[e]
    mbar_wait(cbar + st, (cphase >> st) & 1u);
    cphase ^= 1u << st;
    while (ck + (N - k) <= e0) {
      ck += N - k;
      ++k;
    }
    int kc = k;
    for (int cs = ck; kc < s && cs < e1; cs += N - kc, ++kc) {
      const int t0 = max(0, e0 - cs), t1 = min(N - kc, e1 - cs);
      const double* colp = stage + cs;  // colp[t] = M[kc + t][kc]
      if (fwd) {
        const double fk = S[kc];
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
          const int t = threadIdx.x + DAG_THREADS * r - kc;  // row i = t + kc
          if (t >= t0 && t < t1) acc[r] = fma(colp[t], fk, acc[r]);
        }
      } else if (((kc - k) & (NWARP - 1)) == warp) {
        double a0 = 0.0, a1 = 0.0;
        int t = t0 + lane;
        for (; t + 32 < t1; t += 64) {
          a0 = fma(colp[t], S[kc + t], a0);
          a1 = fma(colp[t + 32], S[kc + t + 32], a1);
        }
        if (t < t1) a0 = fma(colp[t], S[kc + t], a0);
        const double x = warp_sum(a0 + a1);
        if (lane == 0) xacc[kc] += x;
      }
    }
    csync();  // stage st free again
    if (threadIdx.x == 0 && c + NSTAGE < nchunk) {
      fence_proxy_async();
      const int n0 = (c + NSTAGE) * CHD;
      issue_chunk(ring + st * A.chunk_bytes, cbar + st, vbase, n0, min(total, n0 + CHD));
    }
  }
  if (!fwd)
    for (int kk = threadIdx.x; kk < s; kk += DAG_THREADS) __stcg(xy + __ldg(cols + kk), xacc[kk]);
  if (fwd) {
    const int top_upd = __ldg(hg + H_TOP_UPD);
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      const int i = threadIdx.x + DAG_THREADS * r;
      if (i < s)
        __stcg(xy + __ldg(cols + i), acc[r]);
      else if (i < s + m && top_upd >= 0)
        __stcg(A.upd + top_upd + (i - s), S[i] - acc[r]);
    }
  }
}

// ================================================================ kernel
// Warp-specialized CTA: warps 0..7 compute, warp 8 schedules.  The
// scheduler holds two dequeued tasks (one per blob buffer), issues their
// blob copies at dequeue time, polls their dependencies without blocking,
// and hands the first ready one (lower queue index first) to the compute
// warps through named barrier 2.  Compute warps signal completion (global
// release + shared flag); the scheduler then refills that slot.  A CTA
// blocks only when both of its tasks wait on others, and the smallest
// unfinished task in the queue is always ready, so the scheme cannot
// deadlock.
__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ int ld_volatile_shared(const int* p) { return *(volatile const int*)p; }

__global__ void __launch_bounds__(DAG_THREADS + 32, 2) k_dag(DagArgs A) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t tbar[2];
  __shared__ __align__(8) uint64_t cbar[NSTAGE];
  __shared__ int32_t s_run, s_run_task, s_run_par, s_done;
  if (A.skip && *A.skip) return;
  uint8_t* buf[2] = {smem, smem + A.blob_max};
  double* S = reinterpret_cast<double*>(smem + 2 * A.blob_max);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int32_t* fwd_cnt = A.ctr + 1;
  int32_t* fwd_done = fwd_cnt + A.nfrag;
  int32_t* bwd_done = fwd_done + A.nfrag;
  if (tid == DAG_THREADS) {
    mbar_init(&tbar[0], 1);
    mbar_init(&tbar[1], 1);
    for (int i = 0; i < NSTAGE; ++i) mbar_init(&cbar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_done = 0;
  }
  __syncthreads();
  if (warp == NWARP) {
    // ------------------------------------------------------------ scheduler
    int32_t task[2] = {A.ntask, A.ntask};
    int pref[2] = {0, 0};      // blob copy in flight / landed for the slot's task
    uint32_t par[2] = {0, 0};  // mbarrier parity of the next completion per buffer
    bool ready[2] = {false, false};
    auto dequeue = [&](int i) {
      task[i] = atomicAdd(A.ctr, 1);
      ready[i] = false;
      pref[i] = 0;
      if (task[i] < A.ntask) {
        if (A.trace) A.trace[5 * (size_t)task[i] + 1] = gtimer();
        if (!(A.tasks[task[i]].flags & TASK_BIG)) {
          fence_proxy_async();
          mbar_expect_tx(&tbar[i], (uint32_t)A.tasks[task[i]].copy_bytes);
          bulk_g2s(buf[i], A.blobs + A.tasks[task[i]].blob_off, (uint32_t)A.tasks[task[i]].copy_bytes, &tbar[i]);
          pref[i] = 1;
        }
      }
    };
    auto poll = [&](int i) {
      if (task[i] >= A.ntask || ready[i]) return;
      const TaskDev& T = A.tasks[task[i]];
      bool ok;
      if (!(T.flags & TASK_BWD))
        ok = T.wait_on <= 0 || ld_acquire(fwd_cnt + T.frag) >= T.wait_on;
      else
        ok = ld_acquire(T.wait_on >= 0 ? bwd_done + T.wait_on : fwd_done + T.frag) != 0;
      if (ok) {
        ready[i] = true;
        if (A.trace) A.trace[5 * (size_t)task[i] + 2] = gtimer();
      }
    };
    if (lane == 0) {
      dequeue(0);
      dequeue(1);
    }
    for (;;) {
      int chosen = -1;
      if (lane == 0) {
        for (;;) {
          const int first = task[0] <= task[1] ? 0 : 1;
          poll(first);
          if (ready[first]) {
            chosen = first;
            break;
          }
          poll(first ^ 1);
          if (ready[first ^ 1]) {
            chosen = first ^ 1;
            break;
          }
          if (task[0] >= A.ntask && task[1] >= A.ntask) break;
          __nanosleep(32);
        }
        if (chosen >= 0) {
          const int32_t t = task[chosen];
          const bool big = (A.tasks[t].flags & TASK_BIG) != 0;
          if (big && pref[chosen ^ 1]) {
            // the big task streams through both buffers: retire the other
            // slot's copy first and re-issue it later
            mbar_wait(&tbar[chosen ^ 1], par[chosen ^ 1]);
            par[chosen ^ 1] ^= 1u;
            pref[chosen ^ 1] = 0;
          }
          if (!big && !pref[chosen]) {
            fence_proxy_async();
            mbar_expect_tx(&tbar[chosen], (uint32_t)A.tasks[t].copy_bytes);
            bulk_g2s(buf[chosen], A.blobs + A.tasks[t].blob_off, (uint32_t)A.tasks[t].copy_bytes, &tbar[chosen]);
            pref[chosen] = 1;
          }
          s_run = chosen;
          s_run_task = t;
          s_run_par = (int)par[chosen];
          if (!big) par[chosen] ^= 1u;
        } else {
          s_run = -1;
        }
      }
      chosen = __shfl_sync(0xffffffffu, chosen, 0);
      __syncwarp();
      bar_arrive(2, DAG_THREADS + 32);  // hand the task to the compute warps
      if (chosen < 0) break;
      if (lane == 0) {
        // while the compute warps run: poll the other slot, wait for completion
        while (!ld_volatile_shared(&s_done)) {
          poll(chosen ^ 1);
          __nanosleep(64);
        }
        s_done = 0;
        dequeue(chosen);
        if (pref[chosen ^ 1] == 0 && task[chosen ^ 1] < A.ntask &&
            !(A.tasks[task[chosen ^ 1]].flags & TASK_BIG)) {
          // re-issue a copy retired by a big task
          fence_proxy_async();
          mbar_expect_tx(&tbar[chosen ^ 1], (uint32_t)A.tasks[task[chosen ^ 1]].copy_bytes);
          bulk_g2s(buf[chosen ^ 1], A.blobs + A.tasks[task[chosen ^ 1]].blob_off,
                   (uint32_t)A.tasks[task[chosen ^ 1]].copy_bytes, &tbar[chosen ^ 1]);
          pref[chosen ^ 1] = 1;
        }
      }
      __syncwarp();
    }
    return;
  }
  // -------------------------------------------------------------- compute
  uint32_t cphase = 0;
  for (;;) {
    bar_sync(2, DAG_THREADS + 32);
    const int slot = s_run;
    if (slot < 0) break;
    const int32_t t = s_run_task;
    const uint32_t par = (uint32_t)s_run_par;
    const TaskDev T = A.tasks[t];
    const bool fwd = !(T.flags & TASK_BWD);
    const bool big = (T.flags & TASK_BIG) != 0;
    const FactorDev F = A.factors[T.factor];
    if (!big) mbar_wait(&tbar[slot], par);
    unsigned long long* tr = A.trace ? A.trace + 5 * (size_t)t : nullptr;
    if (tid == 0 && tr) {
      tr[0] = smid();
      tr[3] = gtimer();
    }
    if (big)
      run_big(A.blobs + T.blob_off, fwd, smem, cbar, cphase, S, A, F, lane, warp);
    else
      // address computed from the shared base (not via buf[]) so the compiler
      // keeps the shared state space and emits LDS for all blob reads
      run_small(reinterpret_cast<const int32_t*>(smem + (size_t)slot * A.blob_max), fwd, S, A, F, lane, warp,
                A.ptrace ? A.ptrace + 16 * (size_t)t : nullptr);
    bar_sync(1, DAG_THREADS);
    if (tid == 0) {
      __threadfence();  // cumulative over the compute warps' writes (bar.sync above)
      if (fwd) {
        if (T.signal >= 0) atomicAdd(fwd_cnt + T.signal, 1);
        st_release(fwd_done + T.frag, 1);
      } else {
        st_release(bwd_done + T.frag, 1);
      }
      if (tr) tr[4] = gtimer();
      *(volatile int*)&s_done = 1;
    }
  }
}

}  // namespace

DagSolver::DagSolver(const DevicePlan& plan, int device, int64_t extra_xy) : device_(device) {
  CUDA_CHECK(cudaSetDevice(device));
  nfrag_ = plan.nfrag;
  ntask_ = (int32_t)plan.tasks.size();
  host_tasks = plan.tasks;
  xy_doubles_ = plan.xy_doubles;
  blob_max_ = (plan.blob_max + 127) / 128 * 128;
  chunk_bytes_ = (2 * blob_max_ / NSTAGE) & ~127;
  smem_ = 2 * blob_max_ + 8 * std::max(plan.max_scratch, 2);
  SFCDD_REQUIRE(smem_ <= 227 * 1024, SFCDD_EINTERNAL, "DAG shared-memory footprint exceeds 227 KB");
  auto up = [&](void** dst, const void* src, size_t bytes) {
    CUDA_CHECK(cudaMalloc(dst, std::max<size_t>(bytes, 16)));
    if (bytes) CUDA_CHECK(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
    bytes_ += std::max<size_t>(bytes, 16);
  };
  up((void**)&blobs_, plan.blobs.data(), plan.blobs.size());
  up((void**)&tasks_, plan.tasks.data(), plan.tasks.size() * sizeof(TaskDev));
  up((void**)&factors_, plan.factors.data(), plan.factors.size() * sizeof(FactorDev));
  CUDA_CHECK(cudaMalloc(&upd_, std::max<int64_t>(plan.upd_doubles, 2) * 8));
  CUDA_CHECK(cudaMalloc(&xy_, std::max<int64_t>(plan.xy_doubles + extra_xy, 2) * 8));
  xy_doubles_ = plan.xy_doubles + extra_xy;
  ctr_words_ = 1 + 3 * nfrag_;
  CUDA_CHECK(cudaMalloc(&ctr_, ctr_words_ * 4));
  bytes_ += std::max<int64_t>(plan.upd_doubles, 2) * 8 + std::max<int64_t>(plan.xy_doubles, 2) * 8 + ctr_words_ * 4;
  {
    // the attribute is per function: only ever raise it, so every live
    // solver (several handles per process in shard emulation) can launch
    static std::mutex mu;
    static int max_smem = 0;
    std::lock_guard<std::mutex> g(mu);
    if (smem_ > max_smem) {
      CUDA_CHECK(cudaFuncSetAttribute(k_dag, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_));
      max_smem = smem_;
    }
  }
  int per_sm = 0, sms = 0;
  CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dag, DAG_THREADS + 32, smem_));
  CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  SFCDD_REQUIRE(per_sm >= 1, SFCDD_EINTERNAL, "DAG kernel cannot be resident");
  grid_ = std::max(1, std::min(per_sm * sms, ntask_));
}

DagSolver::~DagSolver() {
  cudaFree(blobs_);
  cudaFree(tasks_);
  cudaFree(factors_);
  cudaFree(upd_);
  cudaFree(xy_);
  cudaFree(ctr_);
}

int DagSolver::big_front_max(int blob_max) {
  (void)blob_max;  // chunks may cut columns: only the forward row registers bound the front
  return RMAX * DAG_THREADS;
}

void DagSolver::solve(const double* rhs, cudaStream_t st, const int32_t* skip) {
  if (ntask_ == 0) return;
  CUDA_CHECK(cudaMemsetAsync(ctr_, 0, ctr_words_ * 4, st));
  DagArgs a;
  a.tasks = tasks_;
  a.ntask = ntask_;
  a.nfrag = nfrag_;
  a.blobs = blobs_;
  a.factors = factors_;
  a.rhs = rhs;
  a.xy = xy_;
  a.upd = upd_;
  a.ctr = ctr_;
  a.blob_max = blob_max_;
  a.chunk_bytes = chunk_bytes_;
  a.skip = skip;
  a.trace = trace_;
  a.ptrace = trace_ ? trace_ + 5 * (size_t)ntask_ : nullptr;
  k_dag<<<grid_, DAG_THREADS + 32, smem_, st>>>(a);
  CUDA_CHECK(cudaGetLastError());
}

void DagSolver::set_trace(unsigned long long* dev_buf) { trace_ = dev_buf; }

}  // namespace sfcdd
