// Batched block-inverse supernodal triangular solves as ONE persistent
// dataflow kernel of independent WARP workers (forward + backward sweeps of
// all subdomain factors).
//
// Replaces the per-subdomain SuperLU gstrs calls of the reference's
// one-level Schwarz sweep (schwarz.py:81-101 -> linalg.py:67-72) together
// with the R_i gather (schwarz.py:82).  Design:
//  * every supernode stores M = [L_JJ^{-1}; L_BJ L_JJ^{-1}], so each
//    supernode is a dependency-free GEMV (forward) / GEMV^T (backward);
//  * the work is cut into warp tasks (plan.h): FRAG tasks run a small
//    subtree level by level, ROW / COL tasks a block of rows / columns of one
//    big supernode.  A task's metadata + factor values are ONE blob moved
//    HBM -> the warp's shared-memory slot by a single cp.async.bulk completing
//    on the warp's mbarrier; the copy is issued before the dependency wait;
//  * every warp pulls tasks from a global queue in topological (HLFET)
//    order and waits on per-group counters (acquire / release) -- no CTA
//    barrier anywhere, no grid barrier, no host round trip; deadlock-free
//    because a task only waits on tasks earlier in the queue, which running
//    warps own;
//  * multifrontal update vectors are summed by the consumer in fixed order
//    (gather form), so results are bitwise reproducible run to run.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>

#include "common.h"
#include "dag_solve.h"

#ifndef SFCDD_LEAN
#define SFCDD_LEAN 0  // experiment switches (tools/build_variants.sh): 1 no watchdog / diagnostics, 2 launch-bounds
#endif                // register cap, 4 specialised FRAG calls, 8 no syncwarp before the ROW front copy

#ifndef SFCDD_REGS4
#define SFCDD_REGS4 72  // registers per thread of the 4-worker kernel: 5 CTAs of 160 threads per SM
#endif

namespace sfcdd {

namespace {

constexpr unsigned FULL = 0xffffffffu;

struct DagArgs {
  const TaskDev* tasks;
  int32_t ntask;
  int32_t slot_bytes;  // per warp: blob area + scratch area
  int32_t blob_max;    // blob area bytes (scratch follows)
  const uint8_t* blobs;
  const FactorDev* factors;
  const double* rhs;
  double* xy;
  double* upd;
  int32_t* ctr;  // [0] unused | per group: fin, bdone, rdone (plan.h)
  int32_t* qhead;  // nq queue heads, one per 128-byte line: queue j holds tasks j, j+nq, ...
  int32_t nq;
  const int32_t* skip;  // optional: nonzero -> whole solve skipped (PCG done)
  unsigned long long* trace;  // optional: per task {sm, t_top, t_deps, t_data, t_end} (ns)
  unsigned long long* ptrace;  // optional: per task 16 clock64 stamps (FRAG phases)
  int32_t mode;  // tuning switches (SFCDD_DAG_MODE): 1 = acquire polling, 2 = workers release directly,
                 // 4 = blob copies without the L2 evict_first hint
  int32_t sig_ns;  // signaller idle sleep (ns, SFCDD_SIG_NS; mode bit 8)
  uint32_t sig_wait_ns;  // signaller suspend-time hint on the post barrier (SFCDD_SIG_WAIT_NS)
  int32_t* diag;  // mode bit 32 (SFCDD_DAG_MODE, debugging): a dependency wait that times out records
                  // {1, task, wait_idx, value, target, kind} here and every warp leaves at its next wait
                  // instead of trapping; the host reads it back after the launch
  unsigned long long watchdog_ns;
  int32_t pf_dist;  // > 0: the claimer of task t pulls the descriptor and blob of task t + pf_dist into L2
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

// arrive on a count-1 barrier (release.cta): one completed phase per post
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// suspend until the phase of this parity completes or ~ns elapse (the
// thread issues nothing meanwhile); true if the phase completed
__device__ __forceinline__ bool mbar_wait_timed(uint64_t* bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
      : "memory");
  return ok != 0;
}

// Watchdog (never fires in a correct run): a wait that exceeds this many
// ns traps the kernel -- a launch error for the caller instead of a hung GPU
constexpr unsigned long long DAG_WATCHDOG_NS = 20ull * 1000 * 1000 * 1000;  // bulk-copy waits

// mbarrier wait with the watchdog (1 us suspend hints per try)
// (the slow path is ONE out-of-line copy: the kernel is instruction-cache bound, code size is time)
__device__ __noinline__ void mbar_wait_slow(uint64_t* bar, uint32_t parity) {
  const unsigned long long t0 = gtimer();
  while (!mbar_wait_timed(bar, parity, 1000))
    if (gtimer() - t0 > DAG_WATCHDOG_NS) __trap();
}
__device__ __forceinline__ void mbar_wait_guard(uint64_t* bar, uint32_t parity) {
  if (mbar_wait_timed(bar, parity, 1000)) return;
  mbar_wait_slow(bar, parity);
}

// TMA bulk copy global -> shared, completion signalled on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// the same with an L2 cache policy (evict_first for the streamed factor blobs,
// so the work vectors the gathers read stay resident in L2)
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// generic-proxy global writes (other tasks' outputs, acquired through their
// counters) -> visible to this thread's async-proxy (bulk copy) reads
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

inline __device__ uint32_t bytes16(int n_doubles) { return (uint32_t)((8 * n_doubles + 15) & ~15); }

__device__ __forceinline__ int32_t ld_acquire(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int32_t ld_relaxed(const int32_t* p) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int32_t ld_acquire_cta(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.cta.shared::cta.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_cta(int32_t* p, int32_t v) {
  asm volatile("st.release.cta.shared::cta.s32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

__device__ __forceinline__ void st_relaxed_cta(int32_t* p, int32_t v) {
  asm volatile("st.relaxed.cta.shared::cta.s32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

__device__ __forceinline__ void red_relaxed_add(int32_t* p, int32_t v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void red_release_add(int32_t* p, int32_t v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int64_t gidx(const FactorDev& F, int32_t ro) {
  int64_t g = F.gstart + ro;
  return g >= F.gmod ? g - F.gmod : g;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

__device__ __forceinline__ int64_t coloff(int64_t s, int64_t m, int64_t k) { return k * (s + m) - k * (k - 1) / 2; }

__device__ __forceinline__ int lo16(int32_t v) { return (int)((uint32_t)v & 0xffffu); }
__device__ __forceinline__ int hi16(int32_t v) { return (int)((uint32_t)v >> 16); }

// Gather n values with all of a lane's global loads in flight before any
// store (8 per lane per round): one memory latency instead of one per element.
// (RB = 16 in the 128-register 2-worker kernel -- one round for the ~360 values a 3-D fragment
// gathers -- measured slower: C3 k_dag 1.79 -> 1.90 ms, C5 27.7 -> 30.5 ms)
template <int RB = 8, typename Load, typename Store>
__device__ __forceinline__ void warp_gather(int n, int lane, Load ld, Store st) {
  #pragma unroll 1
  for (int base = 0; base < n; base += RB * 32) {
    double v[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int c = base + lane + 32 * r;
      v[r] = c < n ? ld(c) : 0.0;
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int c = base + lane + 32 * r;
      if (c < n) st(c, v[r]);
    }
  }
}

// one gather-form assembly run: S[dst] + S[src_0] + S[src_1] + ... in fixed
// order.  Runs of <= 3 sources (nearly all) are straight-line: every load is
// unconditional (indices clamped into the run), the adds are selects.
__device__ __forceinline__ void run_apply(const int32_t* runs, const int32_t* gp, int r, double* S) {
  const int p0 = runs[r], p1 = runs[r + 1];
  const int n = p1 - p0;
  const int32_t g0 = gp[p0];
  const int32_t g1 = gp[p0 + (n > 1 ? 1 : 0)];
  const int32_t g2 = gp[p0 + (n > 2 ? 2 : 0)];
  const int dst = lo16(g0);
  const double d = S[dst], v0 = S[hi16(g0)], v1 = S[hi16(g1)], v2 = S[hi16(g2)];
  double acc = d + v0;
  acc = n > 1 ? acc + v1 : acc;
  acc = n > 2 ? acc + v2 : acc;
  #pragma unroll 1
  for (int p = p0 + 3; p < p1; ++p) acc += S[hi16(gp[p])];
  S[dst] = acc;
}

// gather-form assembly runs of one level; two runs per lane in flight
__device__ __forceinline__ void gather_runs(const int32_t* runs, const int32_t* gp, int r0, int r1, double* S,
                                            int lane) {
  // (one copy of run_apply: two runs per lane in flight measured no faster than the smaller code)
  #pragma unroll 1
  for (int r = r0 + lane; r < r1; r += 32) run_apply(runs, gp, r, S);
}

// ===================================================== FRAG (small subtree)
__device__ __forceinline__ int rec_s(const int4& r) { return r.x & 0xfff; }
__device__ __forceinline__ int rec_lp(const int4& r) { return (r.x >> 12) & 7; }
__device__ __forceinline__ int rec_m(const int4& r) { return (int)((unsigned)r.x >> 16); }

// forward row i of a supernode: y_i (i < s) or u_i = f_i - (W f_J)_i.
// M[k][i-k] sits at coloff(k) + i - k; successive k advance by s+m-1-k.
__device__ __forceinline__ void fwd_row(const int4 R, const double* vals, double* S, int i) {
  const int s = rec_s(R), m = rec_m(R);
  if (i >= s + m) return;
  double* f = S + R.y;
  const double* M = vals + R.z;
  const int kmax = i < s ? i : s - 1;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int idx = i, step = s + m - 1;
  int k = 0;
  #pragma unroll 1
  for (; k + 3 <= kmax; k += 4) {
    const int i1 = idx + step, i2 = i1 + step - 1, i3 = i2 + step - 2;
    a0 = fma(M[idx], f[k], a0);
    a1 = fma(M[i1], f[k + 1], a1);
    a2 = fma(M[i2], f[k + 2], a2);
    a3 = fma(M[i3], f[k + 3], a3);
    idx = i3 + step - 3;
    step -= 4;
  }
  #pragma unroll 1
  for (; k <= kmax; ++k) {
    a0 = fma(M[idx], f[k], a0);
    idx += step;
    --step;
  }
  const double acc = (a0 + a1) + (a2 + a3);
  if (i < s)
    S[R.w + i] = acc;  // y_J
  else
    f[i] -= acc;  // u = f_B - W f_J (only f[0:s) is read by other rows)
}

// the same for a supernode with s <= 4, straight-line and branch-free
// (predicated loads, selected store address): ~3x fewer cycles than the
// looped path for the tiny supernodes that dominate the leaves
__device__ __forceinline__ void fwd_tiny(const int4 R, const double* vals, double* S, int i, bool on) {
  const int s = rec_s(R), w = s + rec_m(R);
  const bool ok = on && i < w;
  const int kmax = i < s ? i : s - 1;
  double* f = S + R.y;
  const double* M = vals + R.z;
  const double m0 = ok ? M[i] : 0.0, f0 = ok ? f[0] : 0.0;
  const double m1 = ok && kmax >= 1 ? M[w + i - 1] : 0.0, f1 = ok && kmax >= 1 ? f[1] : 0.0;
  const double m2 = ok && kmax >= 2 ? M[2 * w + i - 3] : 0.0, f2 = ok && kmax >= 2 ? f[2] : 0.0;
  const double m3 = ok && kmax >= 3 ? M[3 * w + i - 6] : 0.0, f3 = ok && kmax >= 3 ? f[3] : 0.0;
  const double fi = ok && i >= s ? f[i] : 0.0;
  const double acc = fma(m1, f1, m0 * f0) + fma(m3, f3, m2 * f2);
  double* dst = i < s ? S + R.w + i : f + i;
  const double val = i < s ? acc : fi - acc;
  if (ok) *dst = val;
}

// backward columns [k0, k0+c) of a supernode (c <= 32): lanes = (column,
// row-phase), partial dot products reduced over the phases
__device__ __forceinline__ void bwd_cols(const int4 R, const double* vals, double* S, int k0, int c, int lane) {
  const int s = rec_s(R), m = rec_m(R);
  const double* v = S + R.y;
  const int CP = c <= 1 ? 1 : 1 << (32 - __clz(c - 1));  // lanes per phase
  const int P = 32 / CP;
  const int j = lane & (CP - 1), ph = lane / CP;
  const int k = k0 + j;
  double a0 = 0.0, a1 = 0.0;
  if (j < c) {
    const double* col = vals + R.z + coloff(s, m, k);
    const double* vk = v + k;
    const int len = s + m - k;
    int t = ph;
    #pragma unroll 1
    for (; t + P < len; t += 2 * P) {
      a0 = fma(col[t], vk[t], a0);
      a1 = fma(col[t + P], vk[t + P], a1);
    }
    if (t < len) a0 = fma(col[t], vk[t], a0);
  }
  double acc = a0 + a1;
  #pragma unroll 1
  for (int o = CP; o < 32; o <<= 1) acc += __shfl_xor_sync(FULL, acc, o);
  if (ph == 0 && j < c) S[R.w + k] = acc;
}

// backward of packed supernodes (s <= 32 each), lanes = (supernode, column
// k, row phase): 2^lp lanes per column each sum every 2^lp-th row of column
// k of M against v = [y_J ; -x_B], then a butterfly over the phases (groups
// are aligned to 2^lp).  Supernodes are in descending record order.
__device__ __forceinline__ void bwd_lanes(const int4* recs, const double* vals, double* S, int x, int cnt,
                                          unsigned mask, int lane) {
  const unsigned upto = mask & ((2u << lane) - 1u);
  const int seg = __popc(upto) - 1;
  const int seg_lo = 31 - __clz(upto);
  const bool on = seg < cnt;
  const int4 R = recs[x + cnt - 1 - (on ? seg : 0)];
  const int s = rec_s(R), m = rec_m(R), lp = rec_lp(R);
  const int local = lane - seg_lo;
  const int k = local >> lp, P = 1 << lp;
  const bool act = on && k < s;
  double a0 = 0.0, a1 = 0.0;
  if (act) {
    const double* col = vals + R.z + coloff(s, m, k);
    const double* v = S + R.y + k;
    const int len = s + m - k;
    int t = local & (P - 1);
    #pragma unroll 1
    for (; t + P < len; t += 2 * P) {
      a0 = fma(col[t], v[t], a0);
      a1 = fma(col[t + P], v[t + P], a1);
    }
    if (t < len) a0 = fma(col[t], v[t], a0);
  }
  double acc = a0 + a1;
  const int pmax = (int)__reduce_max_sync(FULL, act ? (unsigned)P : 1u);
  #pragma unroll 1
  for (int d = 1; d < pmax; d <<= 1) {
    const double o = __shfl_xor_sync(FULL, acc, d);
    if (d < P) acc += o;
  }
  if (act && (local & (P - 1)) == 0) S[R.w + k] = acc;
}

template <int RB, typename Ahead>
__device__ __forceinline__ void run_frag(const int32_t* h, bool fwd, double* S, const DagArgs& A, const FactorDev& F,
                                         int lane, unsigned long long* pt, Ahead ahead) {
  auto stamp = [&](int i) {
    if (pt && lane == 0 && i < 15) pt[i] = clock64();
  };
  const double* vals = reinterpret_cast<const double*>(reinterpret_cast<const uint8_t*>(h) + h[H_VAL_OFF]);
  const int nlev = h[H_NLEV];
  const int32_t* levtab = h + h[H_LEVELS];
  const int32_t* runs = h + h[H_RUNS];
  const int32_t* gp = h + h[H_GPAIRS];
  const int32_t* bp = h + h[H_BPAIRS];
  const int2* items = reinterpret_cast<const int2*>(h + h[H_ITEMS]);
  const int4* recs = reinterpret_cast<const int4*>(h + h[H_REC]);
  const int32_t* cols = h + h[H_COLS];
  const int32_t* colpos = h + h[H_COLPOS];
  const int ncol = h[H_NCOL];
  double* xy = A.xy + F.xy_off;
  if (fwd) {
    stamp(0);
    const int nzero = h[H_ZERO];
    #pragma unroll 1
    for (int i = lane; i < nzero; i += 32) S[i] = 0.0;
    __syncwarp();
    {  // one batched gather: right-hand side at the columns + external child updates
      const int32_t* eu = h + h[H_EXTU];
      const int nu = h[H_NEXTU], ub = h[H_EXTU_BASE];
      warp_gather<RB>(
          ncol + nu, lane,
          [&](int c) { return c < ncol ? __ldg(A.rhs + gidx(F, cols[c])) : __ldcg(A.upd + eu[c - ncol]); },
          [&](int c, double v) { S[c < ncol ? lo16(colpos[c]) : ub + (c - ncol)] = v; });
    }
    __syncwarp();
    stamp(1);
    #pragma unroll 1
    for (int lv = 0; lv < nlev; ++lv) {
      const int32_t* L = levtab + L_WORDS * lv;
      if (L[L_RUN1] > L[L_RUN0]) {  // multifrontal assembly, gather form
        gather_runs(runs, gp, L[L_RUN0], L[L_RUN1], S, lane);
        __syncwarp();
      }
      if (lv < 6) stamp(2 + 2 * lv);
      #pragma unroll 1
      for (int it = L[L_FI0]; it < L[L_FI1]; ++it) {  // rows of the level's supernodes
        const int2 item = items[it];
        const unsigned ix = (unsigned)item.x;
        const int cnt = (int)((ix >> 16) & 0x7fffu);
        // one row block of a tall front (cnt == 0: record ix, rows 32 item.y + lane) or
        // several small fronts packed into the lanes; ONE copy of fwd_row for both
        // (the kernel is instruction-cache bound: code size is time)
        const unsigned upto = cnt == 0 ? 1u : (unsigned)item.y & ((2u << lane) - 1u);
        const int seg = __popc(upto) - 1;
        const bool on = cnt == 0 || seg < cnt;
        const int4 R = recs[(ix & 0xffffu) + (on ? seg : 0)];
        const int i = cnt == 0 ? 32 * item.y + lane : lane - (31 - __clz(upto));
        if (ix & 0x80000000u)
          fwd_tiny(R, vals, S, i, on);
        else if (on)
          fwd_row(R, vals, S, i);
      }
      __syncwarp();
      if (lv < 6) stamp(3 + 2 * lv);
    }
    ahead();  // (the levels are done: only the result stores remain)
    #pragma unroll 1
    for (int c = lane; c < ncol; c += 32) __stcg(xy + cols[c], S[hi16(colpos[c])]);
    {  // update vectors of the tops (one per packed sibling subtree)
      const int32_t* tops = h + h[H_TOPS];
      #pragma unroll 1
      for (int tp = 0; tp < h[H_NTOP]; ++tp) {
        const int slot = tops[2 * tp + 1];
        if (slot < 0) continue;
        const int4 R = recs[tops[2 * tp]];
        const double* u = S + R.y + rec_s(R);
        #pragma unroll 1
        for (int a = lane; a < rec_m(R); a += 32) __stcg(A.upd + slot + a, u[a]);
      }
    }
    stamp(14);
    if (pt && lane == 0) pt[15] = nlev;
  } else {
    stamp(0);
    {  // one batched gather: y at the columns + x of the external ancestor rows
      const int32_t* ex = h + h[H_EXTX];
      const int nx = h[H_NEXTX], xb = h[H_EXTX_BASE];
      warp_gather<RB>(ncol + nx, lane, [&](int c) { return __ldcg(xy + (c < ncol ? cols[c] : ex[c - ncol])); },
                  [&](int c, double v) { S[c < ncol ? lo16(colpos[c]) : xb + (c - ncol)] = v; });
    }
    __syncwarp();
    stamp(1);
    #pragma unroll 1
    for (int lv = nlev - 1; lv >= 0; --lv) {
      const int32_t* L = levtab + L_WORDS * lv;
      if (L[L_BP1] > L[L_BP0]) {  // v_B = -x(rows)
        #pragma unroll 1
        for (int p = L[L_BP0] + lane; p < L[L_BP1]; p += 32) S[lo16(bp[p])] = -S[hi16(bp[p])];
        __syncwarp();
      }
      const int ls = nlev - 1 - lv;
      if (ls < 4) stamp(2 + 2 * ls);
      #pragma unroll 1
      for (int it = L[L_BI0]; it < L[L_BI1]; ++it) {  // columns / packed small supernodes
        const int2 item = items[it];
        const unsigned ix = (unsigned)item.x;
        const int cnt = (int)((ix >> 16) & 0x7fffu);
        // (FRAG supernodes have s <= 32 = SMALL_MAX_S: every backward item is a packed
        // column-lane item; the wide-supernode column blocks (bwd_cols) are gone)
        bwd_lanes(recs, vals, S, ix & 0xffffu, cnt, (unsigned)item.y, lane);
      }
      __syncwarp();
      if (ls < 4) stamp(3 + 2 * ls);
    }
    ahead();
    #pragma unroll 1
    for (int c = lane; c < ncol; c += 32) __stcg(xy + cols[c], S[hi16(colpos[c])]);
    stamp(14);
    if (pt && lane == 0) pt[15] = nlev;
  }
}

// ====================================================== ASM (big forward)
// front positions [q0, q0+nq) of J: f[q] = (q < s ? rhs[col] : 0) + child
// updates in fixed order; 2 positions per lane, their first 3 update loads
// all in flight (nearly every position has <= 3 contributions)
__device__ __noinline__ void run_asm(const int32_t* h, const DagArgs& A, const FactorDev& F, int lane) {
  const int s = h[AS_S], q0 = h[AS_Q0], nq = h[AS_NQ];
  const int32_t* cols = h + h[AS_COLS];
  const int32_t* ptr = h + h[AS_PTR];
  const int32_t* src = h + h[AS_SRC];
  double* f = A.upd + h[AS_FOFF] + q0;
  constexpr int U = 2;
  #pragma unroll 1
  for (int base = 0; base < nq; base += 32 * U) {
    double acc[U], v0[U], v1[U], v2[U];
    int e0[U], e1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + lane + 32 * u;
      const bool ok = i < nq;
      e0[u] = ok ? ptr[i] : 0;
      e1[u] = ok ? ptr[i + 1] : 0;
      const int n = e1[u] - e0[u];
      acc[u] = (ok && q0 + i < s) ? __ldg(A.rhs + gidx(F, cols[i])) : 0.0;
      v0[u] = n > 0 ? __ldcg(A.upd + src[e0[u]]) : 0.0;
      v1[u] = n > 1 ? __ldcg(A.upd + src[e0[u] + 1]) : 0.0;
      v2[u] = n > 2 ? __ldcg(A.upd + src[e0[u] + 2]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + lane + 32 * u;
      if (i >= nq) continue;
      const int n = e1[u] - e0[u];
      double a = acc[u];
      if (n > 0) a += v0[u];
      if (n > 1) a += v1[u];
      if (n > 2) a += v2[u];
      #pragma unroll 1
      for (int e = e0[u] + 3; e < e1[u]; ++e) a += __ldcg(A.upd + src[e]);
      __stcg(f + i, a);
    }
  }
}

// ======================================================= XB (big backward)
// vb[a] = -x(rows[a]) for J's below rows [a0, a0+na)
__device__ __noinline__ void run_xb(const int32_t* h, const DagArgs& A, const FactorDev& F, int lane) {
  const int a0 = h[XB_A0], na = h[XB_NA];
  const int32_t* rows = h + h[XB_ROWS];
  const double* xy = A.xy + F.xy_off;
  double* vb = A.upd + h[XB_XOFF] + a0;
  warp_gather(na, lane, [&](int q) { return -__ldcg(xy + rows[q]); }, [&](int q, double v) { __stcg(vb + q, v); });
}

// ================================================= BLOB ROW (big forward)
// values in the slot: rows [r0, r0+R) of out = M f_J; lanes = (row, k-phase)
// when R < 32; the assembled front f = [f_J ; f_B] is read contiguously (ASM tasks)
template <bool SPLIT, bool WIDE>
__device__ __forceinline__ void run_row_blob(const int32_t* h, double* S, const DagArgs& A, const FactorDev& F,
                                             int lane, uint64_t* bar, uint32_t& phase, unsigned long long* pt) {
  if (pt && lane == 0) pt[0] = clock64();  // trace stamps: start, front in the slot, products done, stored
  const int s = h[RW_S], R = h[RW_R], C = h[RW_C], r0 = h[RW_R0], NB = h[RW_NB];
  const double* V = reinterpret_cast<const double*>(reinterpret_cast<const uint8_t*>(h) + h[RW_VAL_OFF]);
  int boff = C;  // S index of the first update-row value f_B[r0 - s + i]
  if (SPLIT && h[RW_FOFF] >= 0) {
    // front assembled by J's ASM tasks, contiguous and 16-byte aligned in
    // upd: bulk-copy f_J[0:C) and the update rows f[r0 : r0+NB) (one TMA
    // round trip instead of gather rounds)
    const double* f = A.upd + h[RW_FOFF];
    const int c2 = (C + 1) & ~1;
    boff = c2 + (r0 & 1);
    if (!(SFCDD_LEAN & 8)) __syncwarp();  // every lane has observed the blob copy's phase before the barrier is armed again
    if (lane == 0) {
      fence_proxy_async_global();
      const uint32_t ba = bytes16(C), bb = NB > 0 ? bytes16(NB + (r0 & 1)) : 0u;
      mbar_expect_tx(bar, ba + bb);
      bulk_g2s(S, f, ba, bar);
      if (NB > 0) bulk_g2s(S + c2, f + (r0 & ~1), bb, bar);
    }
    __syncwarp();
    mbar_wait(bar, phase);
    phase ^= 1u;
  } else if (h[RW_ASM_HI] >= 0) {
    // huge s: J's assembly record in global memory [s, m] cols ptr src
    const int64_t o16 = (int64_t)(uint32_t)h[RW_ASM16] | ((int64_t)h[RW_ASM_HI] << 32);
    const int32_t* am = reinterpret_cast<const int32_t*>(A.blobs + 16 * o16);
    const int32_t* cols = am + 2;
    const int32_t* ptr = cols + s;
    const int32_t* src = ptr + s + __ldg(am + 1) + 1;
    #pragma unroll 1
    for (int q = lane; q < C + NB; q += 32) {
      const int p = q < C ? q : r0 + (q - C);
      const int e0 = __ldg(ptr + p), e1 = __ldg(ptr + p + 1);
      double acc = q < C ? __ldg(A.rhs + gidx(F, __ldg(cols + q))) : 0.0;
      #pragma unroll 1
      for (int e = e0; e < e1; ++e) acc += __ldcg(A.upd + __ldg(src + e));
      S[q] = acc;
    }
  } else {
    // f = base + child updates in fixed order (base 0 for update rows); the
    // metadata is in the slot, so every load below is one global round trip
    // U front positions per lane, their right-hand side and first three update
    // loads all in flight (nearly every position has <= 3 contributions): one
    // global round trip per batch instead of one per pair of contributions
    // (traced on C3: the gather was half of a ROW task); same summation order
    const int32_t* cols = h + h[RW_COLS];
    const int32_t* ptr = h + h[RW_PTR];
    const int32_t* src = h + h[RW_SRC];
    constexpr int U = WIDE ? 4 : 2;
    #pragma unroll 1
    for (int base = 0; base < C + NB; base += 32 * U) {
      int e0[U], cn[U];
      double acc[U], v0[U], v1[U], v2[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = base + lane + 32 * u;
        const bool ok = q < C + NB;
        e0[u] = ok ? ptr[q] : 0;
        cn[u] = ok ? ptr[q + 1] - e0[u] : 0;
        acc[u] = (ok && q < C) ? __ldg(A.rhs + gidx(F, cols[q])) : 0.0;
        v0[u] = cn[u] > 0 ? __ldcg(A.upd + src[e0[u]]) : 0.0;
        v1[u] = cn[u] > 1 ? __ldcg(A.upd + src[e0[u] + 1]) : 0.0;
        v2[u] = cn[u] > 2 ? __ldcg(A.upd + src[e0[u] + 2]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = base + lane + 32 * u;
        if (q >= C + NB) continue;
        double a = acc[u];
        if (cn[u] > 0) a += v0[u];
        if (cn[u] > 1) a += v1[u];
        if (cn[u] > 2) a += v2[u];
        #pragma unroll 1
        for (int e = e0[u] + 3; e < e0[u] + cn[u]; ++e) a += __ldcg(A.upd + src[e]);
        S[q] = a;
      }
    }
  }
  __syncwarp();
  if (pt && lane == 0) pt[1] = clock64();
  // (per-pass lane phases for a ragged last pass -- 40 rows as 32 + 8 x 4 phases -- measured slower: C3 +1.3 %)
  const int RP = R >= 32 ? 32 : (R <= 1 ? 1 : 1 << (32 - __clz(R - 1)));  // lanes per phase
  const int P = 32 / RP;
  const int il = lane & (RP - 1), ph = lane / RP;
  double* yo = A.upd + h[RW_YOFF];
  double* uo = A.upd + h[RW_UOFF];
  #pragma unroll 1
  for (int rb = 0; rb < R; rb += RP) {
    const int i = rb + il;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (i < R) {
      // WIDE (16 KB blobs, 2-worker CTAs: long rows): four independent (value, f)
      // load pairs in flight per step -- the loop is bound by the shared-memory
      // latency of a step, not by its FMAs (C3 k_dag -3 %).  The 8 KB kernel keeps
      // two: the larger code costs it more than the loop gains (C2 +2.5 %)
      const double* v = V + i;
      int k = ph;
      #pragma unroll 1
      for (; WIDE && k + 3 * P < C; k += 4 * P) {
        const double m0 = v[k * R], m1 = v[(k + P) * R], m2 = v[(k + 2 * P) * R], m3 = v[(k + 3 * P) * R];
        const double f0 = S[k], f1 = S[k + P], f2 = S[k + 2 * P], f3 = S[k + 3 * P];
        a0 = fma(m0, f0, a0);
        a1 = fma(m1, f1, a1);
        a2 = fma(m2, f2, a2);
        a3 = fma(m3, f3, a3);
      }
      #pragma unroll 1
      for (; !WIDE && k + P < C; k += 2 * P) {
        a0 = fma(v[k * R], S[k], a0);
        a1 = fma(v[(k + P) * R], S[k + P], a1);
      }
      #pragma unroll 1
      for (; k < C; k += P) a0 = fma(v[k * R], S[k], a0);
    }
    double acc = (a0 + a1) + (a2 + a3);
    #pragma unroll 1
    for (int o = RP; o < 32; o <<= 1) acc += __shfl_xor_sync(FULL, acc, o);
    if (ph == 0 && i < R) {
      const int row = r0 + i;
      if (row < s)
        __stcg(yo + row, acc);
      else
        __stcg(uo + (row - s), S[boff + i] - acc);
    }
  }
  if (pt && lane == 0) {
    pt[2] = clock64();
    pt[15] = 100 + R;  // (marks a ROW record for tools/analyze_trace.py)
  }
}

// ================================================ BLOB COL (big backward)
// columns [k0, k0+c): x_j = sum_r M[k0+r, k0+j] v[r]; lanes = (column, row-phase)
template <bool SPLIT, bool WIDE>
__device__ __forceinline__ void run_col_blob(const int32_t* h, double* S, const DagArgs& A, const FactorDev& F,
                                             int lane, uint64_t* bar, uint32_t& phase) {
  const int s = h[CL_S], m = h[CL_M], k0 = h[CL_K0], c = h[CL_C];
  const double* V = reinterpret_cast<const double*>(reinterpret_cast<const uint8_t*>(h) + h[CL_VAL_OFF]);
  const int32_t* cols = h + h[CL_COLS];
  double* xy = A.xy + F.xy_off;
  const int ny = s - k0, L = ny + m;
  const double* yv = A.upd + h[CL_YOFF] + k0;
  const double* Sv = S;  // v[r] = Sv[r]
  if (SPLIT && h[CL_XOFF] >= 0) {
    // -x_B (XB tasks) follows y_J in upd: v = [y_J[k0:s) ; -x_B] is one
    // contiguous range (plan.cpp), bulk-copied from its 16-byte aligned start
    const int sh = (int)((h[CL_YOFF] + k0) & 1);
    Sv = S + sh;
    __syncwarp();  // every lane has observed the blob copy's phase before the barrier is armed again
    if (lane == 0) {
      fence_proxy_async_global();
      mbar_expect_tx(bar, bytes16(L + sh));
      bulk_g2s(S, yv - sh, bytes16(L + sh), bar);
    }
    __syncwarp();
    mbar_wait(bar, phase);
    phase ^= 1u;
  } else {
    const int32_t* rows = h + h[CL_ROWS];
    warp_gather(
        L, lane, [&](int q) { return q < ny ? __ldcg(yv + q) : -__ldcg(xy + rows[q - ny]); },
        [&](int q, double v) { S[q] = v; });
  }
  __syncwarp();
  const int CP = c >= 32 ? 32 : (c <= 1 ? 1 : 1 << (32 - __clz(c - 1)));  // lanes per phase
  const int P = 32 / CP;
  const int j = lane & (CP - 1), ph = lane / CP;
  #pragma unroll 1
  for (int jb = 0; jb < c; jb += CP) {
    const int jj = jb + j;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (jj < c) {
      const double* v = V + jj;
      int r = ph;
      #pragma unroll 1
      for (; WIDE && r + 3 * P < L; r += 4 * P) {
        const double m0 = v[r * c], m1 = v[(r + P) * c], m2 = v[(r + 2 * P) * c], m3 = v[(r + 3 * P) * c];
        const double f0 = Sv[r], f1 = Sv[r + P], f2 = Sv[r + 2 * P], f3 = Sv[r + 3 * P];
        a0 = fma(m0, f0, a0);
        a1 = fma(m1, f1, a1);
        a2 = fma(m2, f2, a2);
        a3 = fma(m3, f3, a3);
      }
      #pragma unroll 1
      for (; !WIDE && r + P < L; r += 2 * P) {
        a0 = fma(v[r * c], Sv[r], a0);
        a1 = fma(v[(r + P) * c], Sv[r + P], a1);
      }
      #pragma unroll 1
      for (; r < L; r += P) a0 = fma(v[r * c], Sv[r], a0);
    }
    double acc = (a0 + a1) + (a2 + a3);
    #pragma unroll 1
    for (int o = CP; o < 32; o <<= 1) acc += __shfl_xor_sync(FULL, acc, o);
    if (ph == 0 && jj < c) __stcg(xy + cols[jj], acc);
  }
}

// ================================================ dense blocks (ROW / COL)
// DIRECT blocks: the dense ROW / COL blocks of wide separators stay in HBM
// and are streamed into registers -- any size, every factor value is used
// exactly once -- where a BLOB block (above) arrives in the slot with its
// metadata in one bulk copy, the lowest-latency form for small blocks.
//
// dense_dot: lane (il, ph) accumulates sum_k V[k W + il] vec[k] over
// k = ph, ph + P, ... (W <= 32 lanes per vector entry, P = 32 / pow2(W) entry
// phases), DU loads per lane in flight ahead of the FMAs (two register
// groups), then a butterfly over the phases.  ROW: W = R rows, k = columns of
// the R x C column-major block, vec = f_J.  COL: W = c columns, k = rows of
// the L x c row-major block, vec = [y_J[k0:s) ; -x_B].
//  * RING = false: vec sits in the slot scratch (gathered by the task);
//  * RING = true: vec is contiguous in the update buffer (ASM / XB tasks
//    wrote it) and travels through a two-slot ring of RING_CHUNK doubles by
//    bulk copies on the warp's mbarrier, the next chunk in flight while the
//    current one is consumed: vec[k] = gvec[k + sh], gvec 16-byte aligned.

// (ONE inlined copy in the kernel: run_dense below is the only caller; the
// kernel's code size matters -- every resident warp runs a different path)
template <int DU>
__device__ __forceinline__ double dense_dot(const double* __restrict__ V, bool ring, int W, int Len, double* S,
                                            const double* gvec, int sh, uint64_t* bar, uint32_t& phase, int lane) {
  static_assert(RING_CHUNK % DU == 0 && RING_CHUNK / DU <= 32, "a ring chunk holds whole groups");
  constexpr int WPMIN = 32 / (RING_CHUNK / DU);  // phases P <= RING_CHUNK / DU: groups never straddle ring chunks
  const int WP = W >= 32 ? 32 : (W <= WPMIN ? WPMIN : 1 << (32 - __clz(W - 1)));  // lanes per phase
  const int P = 32 / WP;
  const int ph = lane / WP;
  const int il = min(lane & (WP - 1), W - 1);  // lanes >= W repeat the last one (result unused)
  const int nj = (Len - ph + P - 1) / P;       // vector entries of this lane's phase (>= 0)
  const int ng = ((Len + P - 1) / P + DU - 1) / DU;
  const double* q = V + (size_t)ph * W + il;   // this lane's next value
  const int vs = P * W;                        // value stride per vector entry of the phase
  if (ring) {
    // every lane has observed the barrier phase of the task's blob copy before
    // the barrier is armed again (a lane still polling the old parity would
    // see two completed phases as none)
    __syncwarp();
    if (lane == 0) {
      fence_proxy_async_global();  // the producers' generic-proxy writes -> this bulk read
      fence_proxy_async();         // earlier generic reads of the ring slot -> async write
      const uint32_t nb = bytes16(min(RING_CHUNK, Len) + sh);
      mbar_expect_tx(bar, nb);
      bulk_g2s(S, gvec, nb, bar);
    }
  }
  double d[DU];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const int GPC = ring ? RING_CHUNK / (P * DU) : ng;  // groups per ring chunk (>= 1)
  const double* fq = S + ph;  // vec entry of this lane's next value (no ring)
  #pragma unroll 1
  for (int g = 0; g < ng; ++g) {
    // DU independent loads per lane in flight (the only latency the loop pays)
    const int left = nj - g * DU;  // entries of this lane still to do
#pragma unroll
    for (int u = 0; u < DU; ++u) d[u] = u < left ? __ldcs(q + u * vs) : 0.0;  // streamed from HBM, evict-first
    q += (size_t)DU * vs;
    if (ring && g % GPC == 0) {
      const int c = g / GPC;
      mbar_wait_guard(bar, phase);
      phase ^= 1u;
      // every lane has consumed chunk c - 1 (its slot may be refilled) and has
      // observed chunk c's phase (the barrier may be armed again)
      __syncwarp();
      if (lane == 0 && RING_CHUNK * (c + 1) < Len) {
        fence_proxy_async();
        const uint32_t nb = bytes16(min(RING_CHUNK, Len - RING_CHUNK * (c + 1)) + sh);
        mbar_expect_tx(bar, nb);
        bulk_g2s(S + ((c + 1) & 1) * RING_STRIDE, gvec + RING_CHUNK * (c + 1), nb, bar);
      }
      fq = S + (c & 1) * RING_STRIDE + sh + ph;
    }
#pragma unroll
    for (int u = 0; u < DU; u += 4) {
      a0 = fma(d[u], u < left ? fq[P * u] : 0.0, a0);
      a1 = fma(d[u + 1], u + 1 < left ? fq[P * (u + 1)] : 0.0, a1);
      a2 = fma(d[u + 2], u + 2 < left ? fq[P * (u + 2)] : 0.0, a2);
      a3 = fma(d[u + 3], u + 3 < left ? fq[P * (u + 3)] : 0.0, a3);
    }
    fq += P * DU;
  }
  double acc = (a0 + a1) + (a2 + a3);
  #pragma unroll 1
  for (int o = WP; o < 32; o <<= 1) acc += __shfl_xor_sync(FULL, acc, o);
  return acc;
}

// The same dot product with the VALUES travelling through a ring of VST
// shared-memory stages filled by bulk copies (one mbarrier per stage): up to
// VST * 4 KB of a task's value stream in flight instead of the DU loads per
// lane of dense_dot (4 KB per warp, one memory latency per group), and no
// registers held by loads in flight.  Used where the slot has room for >= 2
// stages behind the task's scratch (wide slots of the 2-worker kernel); the
// stage area is free shared memory of the slot, the planner reserves nothing.
// A stage holds kc = min(RING_CHUNK, 512 / WP) vector entries (kc W values,
// <= 4 KB; kc divides RING_CHUNK, so a stage never straddles a vector chunk).
constexpr int VST = 4;             // value stages per worker (mbarriers)
constexpr int VSTAGE_DOUBLES = 512;

__device__ __forceinline__ double dense_dot_tma(const double* __restrict__ V, bool ring, int W, int Len, double* S,
                                                const double* gvec, int sh, uint64_t* bar, uint32_t& phase,
                                                uint64_t* vbar, uint32_t& vph, double* stage, int nst, int lane) {
  const int WP = W >= 32 ? 32 : (W <= 1 ? 1 : 1 << (32 - __clz(W - 1)));  // lanes per phase
  const int P = 32 / WP;
  const int ph = lane / WP;
  const int il = min(lane & (WP - 1), W - 1);  // lanes >= W repeat the last one (result unused)
  const int kc = min(RING_CHUNK, VSTAGE_DOUBLES / WP);
  const int nch = (Len + kc - 1) / kc;
  const uint64_t pol = policy_evict_first();
  // every lane has observed the barrier phase of the task's blob copy before
  // the barrier is armed again, and is done with the slot's previous contents
  __syncwarp();
  auto issue = [&](int c, int st) {  // lane 0: values of vector entries [c kc, (c + 1) kc) -> stage st
    const int k0 = c * kc, nk = min(kc, Len - k0);
    const uint32_t nb = (uint32_t)((8 * nk * W + 15) & ~15);
    mbar_expect_tx(vbar + st, nb);
    bulk_g2s_hint(stage + st * VSTAGE_DOUBLES, V + (size_t)k0 * W, nb, vbar + st, pol);
  };
  if (lane == 0) {
    fence_proxy_async();  // earlier generic accesses of the ring slots / stages -> async writes
    if (ring) {
      fence_proxy_async_global();  // the producers' generic-proxy writes -> this bulk read
      const uint32_t nb = bytes16(min(RING_CHUNK, Len) + sh);
      mbar_expect_tx(bar, nb);
      bulk_g2s(S, gvec, nb, bar);
    }
    #pragma unroll 1
    for (int c = 0; c < nst && c < nch; ++c) issue(c, c);
  }
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int st = 0;
  #pragma unroll 1
  for (int c = 0; c < nch; ++c) {
    const int k0 = c * kc, nk = min(kc, Len - k0);
    const int rc = k0 / RING_CHUNK;
    if (ring && k0 == rc * RING_CHUNK) {
      mbar_wait_guard(bar, phase);
      phase ^= 1u;
      // every lane has consumed vector chunk rc - 1 (its slot may be refilled)
      // and has observed chunk rc's phase (the barrier may be armed again)
      __syncwarp();
      if (lane == 0 && RING_CHUNK * (rc + 1) < Len) {
        fence_proxy_async();
        const uint32_t nb = bytes16(min(RING_CHUNK, Len - RING_CHUNK * (rc + 1)) + sh);
        mbar_expect_tx(bar, nb);
        bulk_g2s(S + ((rc + 1) & 1) * RING_STRIDE, gvec + RING_CHUNK * (rc + 1), nb, bar);
      }
    }
    const double* vec = ring ? S + (rc & 1) * RING_STRIDE + sh + (k0 - rc * RING_CHUNK) : S + k0;
    mbar_wait_guard(vbar + st, (vph >> st) & 1u);
    vph ^= 1u << st;
    const double* v = stage + st * VSTAGE_DOUBLES + il;
    int k = ph;
    #pragma unroll 1
    for (; k + 3 * P < nk; k += 4 * P) {
      const double m0 = v[k * W], m1 = v[(k + P) * W], m2 = v[(k + 2 * P) * W], m3 = v[(k + 3 * P) * W];
      const double f0 = vec[k], f1 = vec[k + P], f2 = vec[k + 2 * P], f3 = vec[k + 3 * P];
      a0 = fma(m0, f0, a0);
      a1 = fma(m1, f1, a1);
      a2 = fma(m2, f2, a2);
      a3 = fma(m3, f3, a3);
    }
    #pragma unroll 1
    for (; k < nk; k += P) a0 = fma(v[k * W], vec[k], a0);
    // every lane is done with stage st and has observed its phase: refill it
    __syncwarp();
    if (lane == 0 && c + nst < nch) {
      fence_proxy_async();
      issue(c + nst, st);
    }
    st = st + 1 == nst ? 0 : st + 1;
  }
  double acc = (a0 + a1) + (a2 + a3);
  #pragma unroll 1
  for (int o = WP; o < 32; o <<= 1) acc += __shfl_xor_sync(FULL, acc, o);
  return acc;
}

// MROW (plan.h): update rows [r0, r0 + rows) of a narrow supernode (C = s <=
// RING_CHUNK) as ONE value stream of nb blocks of Rb rows; lanes = rows of the
// block, f_J and the task's f_B rows sit in the two ring slots (one bulk-copy
// round trip), u = f_B - W f_J stored block by block.
template <int DU, bool PIPE>
__device__ __forceinline__ uint32_t run_mrow(const int32_t* h, double* S, const DagArgs& A, const uint8_t* gblob,
                                             int lane, uint64_t* bar, uint32_t phase) {
  const int s = h[RW_S], Rb = h[RW_R], C = h[RW_C], r0 = h[RW_R0], rows = h[RW_NB], nb = h[RW_NBLK];
  const double* f = A.upd + h[RW_FOFF];
  __syncwarp();  // every lane has observed the blob copy's phase before the barrier is armed again
  if (lane == 0) {
    fence_proxy_async_global();
    fence_proxy_async();
    const uint32_t ba = bytes16(C), bb = bytes16(rows + (r0 & 1));
    mbar_expect_tx(bar, ba + bb);
    bulk_g2s(S, f, ba, bar);
    bulk_g2s(S + RING_STRIDE, f + (r0 & ~1), bb, bar);
  }
  const double* fB = S + RING_STRIDE + (r0 & 1);
  double* uo = A.upd + h[RW_UOFF] + (r0 - s);
  const double* V = reinterpret_cast<const double*>(gblob + h[RW_VAL_OFF]) + min(lane, Rb - 1);
  // units = (block, group of <= DU columns of the block); PIPE: the next
  // unit's loads are in flight while this one is consumed (two register sets)
  const int gpb = (C + DU - 1) / DU;  // groups per block
  const int nu = nb * gpb;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int lb = 0, lg = 0;  // (block, group) of the next unit to load
  auto load_unit = [&](double (&d)[DU]) {
    const int k0 = lg * DU, n = min(DU, C - k0);
    const double* q = V + ((size_t)lb * C + k0) * Rb;
#pragma unroll
    for (int u = 0; u < DU; ++u) d[u] = u < n ? __ldcs(q + u * Rb) : 0.0;
    if (++lg == gpb) {
      lg = 0;
      ++lb;
    }
  };
  int cb = 0, cg = 0;  // (block, group) of the next unit to consume
  auto fma_unit = [&](const double (&d)[DU]) {
    const int k0 = cg * DU, n = min(DU, C - k0);
    const double* fq = S + k0;
#pragma unroll
    for (int u = 0; u < DU; u += 4) {
      a0 = fma(d[u], u < n ? fq[u] : 0.0, a0);
      a1 = fma(d[u + 1], u + 1 < n ? fq[u + 1] : 0.0, a1);
      a2 = fma(d[u + 2], u + 2 < n ? fq[u + 2] : 0.0, a2);
      a3 = fma(d[u + 3], u + 3 < n ? fq[u + 3] : 0.0, a3);
    }
    if (++cg == gpb) {  // block cb done: u = f_B - W f_J
      const int row = cb * Rb + lane;
      if (lane < Rb && row < rows) __stcg(uo + row, fB[row] - ((a0 + a1) + (a2 + a3)));
      a0 = a1 = a2 = a3 = 0.0;
      cg = 0;
      ++cb;
    }
  };
  double d0[DU];
  if (PIPE) {
    double d1[DU];
    load_unit(d0);
    if (nu > 1) load_unit(d1);
    mbar_wait_guard(bar, phase);
    phase ^= 1u;
    for (int i = 0; i < nu; i += 2) {
      fma_unit(d0);
      if (i + 2 < nu) load_unit(d0);
      if (i + 1 < nu) {
        fma_unit(d1);
        if (i + 3 < nu) load_unit(d1);
      }
    }
  } else {
    load_unit(d0);
    mbar_wait_guard(bar, phase);
    phase ^= 1u;
    for (int i = 0; i < nu; ++i) {
      fma_unit(d0);
      if (i + 1 < nu) load_unit(d0);
    }
  }
  return phase;
}

// DIRECT ROW (big forward): rows [r0, r0+R) of out = M f_J: y rows (< s) or update
// rows u = f_B - out.  DIRECT COL (big backward): columns [k0, k0+c):
// x_j = sum_r M[k0+r, k0+j] v[r], v = [y_J[k0:s) ; -x_B].
template <bool SPLIT, int DU>
__device__ __forceinline__ uint32_t run_dense(bool is_row, const int32_t* h, double* S, const DagArgs& A,
                                              const FactorDev& F, const uint8_t* gblob, int lane, uint64_t* bar,
                                              uint32_t phase, uint64_t* vbar, uint32_t& vph, const uint8_t* slot_end,
                                              const bool allow_stages) {
  double* xy = A.xy + F.xy_off;
  const double* V;
  const double* gvec = nullptr;
  bool ring = false;
  int W, Len, sh = 0;
  double fb = 0.0;
  if (is_row) {
    const int s = h[RW_S], R = h[RW_R], C = h[RW_C], r0 = h[RW_R0], NB = h[RW_NB];
    V = reinterpret_cast<const double*>(gblob + h[RW_VAL_OFF]);
    W = R;
    Len = C;
    if (SPLIT && h[RW_FOFF] >= 0) {
      // front assembled by J's ASM tasks, contiguous and 16-byte aligned in upd
      gvec = A.upd + h[RW_FOFF];
      ring = true;
      if (NB > 0 && lane < R) fb = __ldcg(gvec + r0 + lane);
    } else {
      // f = base + child updates in fixed order (base 0 for update rows), from
      // the metadata in the slot or from J's global assembly record
      // [s, m] cols ptr src over front positions (every load one global round trip)
      const bool ga = h[RW_ASM_HI] >= 0;
      const int64_t o16 = (int64_t)(uint32_t)h[RW_ASM16] | ((int64_t)h[RW_ASM_HI] << 32);
      const int32_t* am = reinterpret_cast<const int32_t*>(A.blobs + 16 * o16);
      const int32_t* cols = ga ? am + 2 : h + h[RW_COLS];
      const int32_t* ptr = ga ? cols + s : h + h[RW_PTR];
      const int32_t* src = ga ? ptr + s + __ldg(am + 1) + 1 : h + h[RW_SRC];
      #pragma unroll 1
      for (int q = lane; q < C + NB; q += 32) {
        const int p = ga && q >= C ? r0 + (q - C) : q;
        const int e0 = ptr[p], e1 = ptr[p + 1];
        double a = q < C ? __ldg(A.rhs + gidx(F, cols[q])) : 0.0;
        int e = e0;
        #pragma unroll 1
        for (; e + 2 <= e1; e += 2) {
          const double u0 = __ldcg(A.upd + src[e]), u1 = __ldcg(A.upd + src[e + 1]);
          a += u0;
          a += u1;
        }
        if (e < e1) a += __ldcg(A.upd + src[e]);
        S[q] = a;
      }
      __syncwarp();
      if (NB > 0 && lane < R) fb = S[C + lane];
    }
  } else {
    const int s = h[CL_S], m = h[CL_M], k0 = h[CL_K0];
    V = reinterpret_cast<const double*>(gblob + h[CL_VAL_OFF]);
    W = h[CL_C];
    const int ny = s - k0;
    Len = ny + m;
    const double* yv = A.upd + h[CL_YOFF] + k0;
    if (SPLIT && h[CL_XOFF] >= 0) {
      // -x_B (XB tasks) follows y_J in upd: v is one contiguous range (plan.cpp)
      sh = (int)((h[CL_YOFF] + k0) & 1);
      gvec = yv - sh;
      ring = true;
    } else {
      const int32_t* rows = h + h[CL_ROWS];
      warp_gather(
          Len, lane, [&](int q) { return q < ny ? __ldcg(yv + q) : -__ldcg(xy + rows[q - ny]); },
          [&](int q, double v) { S[q] = v; });
      __syncwarp();
    }
  }
  // value stages behind the task's scratch, if the slot has room for two or more (and the block is
  // worth a pipeline: at least two stages of values)
  double* stage = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(S + (is_row ? h[RW_SCRATCH] : h[CL_SCRATCH])) + 127) & ~(uintptr_t)127);
  const int nst = min(VST, (int)((slot_end - reinterpret_cast<const uint8_t*>(stage)) / (8 * VSTAGE_DOUBLES)));
  const bool staged = allow_stages && nst >= 2 && (int64_t)W * Len >= 2 * VSTAGE_DOUBLES;
  const double acc = staged ? dense_dot_tma(V, SPLIT && ring, W, Len, S, gvec, sh, bar, phase, vbar, vph, stage, nst, lane)
                            : dense_dot<DU>(V, SPLIT && ring, W, Len, S, gvec, sh, bar, phase, lane);
  // after the butterfly every phase holds the sum: lane i (< W <= lanes per phase) owns row / column i
  if (lane < W) {
    if (is_row) {
      const int row = h[RW_R0] + lane, s = h[RW_S];
      if (row < s)
        __stcg(A.upd + h[RW_YOFF] + row, acc);
      else
        __stcg(A.upd + h[RW_UOFF] + (row - s), fb - acc);
    } else {
      __stcg(xy + (h + h[CL_COLS])[lane], acc);
    }
  }
  return phase;
}

// ================================================================ kernel
// Completion signaller (one thread per CTA, in an extra warp): workers post
// the counter index of a finished task to their mailbox (st.release.cta) and
// move on; the signaller acquires the mailboxes, issues ONE gpu-scope fence
// for everything collected (cumulative over the workers' writes, which
// happen-before it through the CTA-scope release/acquire) and then bumps the
// counters.  The workers never stall on the ~1 us release fence.
template <int WPB>
__device__ __forceinline__ void signaller(const DagArgs& A, const int mode, int32_t* mbox, int32_t* nexit,
                                          uint64_t* sigbar) {
  int32_t v[WPB];
  uint32_t par = 0;
  for (;;) {
    int np = 0;
#pragma unroll
    for (int w = 0; w < WPB; ++w) {
      v[w] = ld_acquire_cta(mbox + w);
      np += v[w] >= 0;
    }
    if (np == 0) {
      if (ld_acquire_cta(nexit) == WPB) {  // workers done: drain once more
        np = 0;
#pragma unroll
        for (int w = 0; w < WPB; ++w) {
          v[w] = ld_acquire_cta(mbox + w);
          np += v[w] >= 0;
        }
        if (np == 0) return;
      } else {
        // idle: sleep on the post barrier (every mailbox post and every
        // worker exit arrives on it) instead of spinning; the scan above
        // decides, the barrier only wakes (a stale parity costs one extra
        // scan and resynchronises)
        if (mode & 8)
          __nanosleep(A.sig_ns);
        else if (mbar_wait_timed(sigbar, par, A.sig_wait_ns))
          par ^= 1u;
        continue;
      }
    }
    __threadfence();
#pragma unroll
    for (int w = 0; w < WPB; ++w)
      if (v[w] >= 0) {
        red_relaxed_add(A.ctr + v[w], 1);
        st_relaxed_cta(mbox + w, -1);
      }
  }
}

// SPLIT: the plan has ASM / XB tasks (many-subdomain configurations); the
// kernel without them keeps the smaller code of the common case
// DIRECT: the plan has ROW / COL blocks streamed from HBM (wide separators)
// TRACE: the instantiation sfcdd_op_trace launches (per-task time stamps); the
// production kernel carries none of that code
template <int WPB, bool SPLIT, bool DIRECT, bool TRACE>
#if SFCDD_LEAN & 2
__global__ void __launch_bounds__((WPB + 1) * 32, 20 / WPB) k_dag(DagArgs A) {
#else
__global__ void __launch_bounds__((WPB + 1) * 32) __maxnreg__(WPB == 4 ? SFCDD_REGS4 : WPB == 2 ? 128 : 96) k_dag(DagArgs A) {
#endif
  // values in flight per lane of a DIRECT block: 2-worker CTAs (big slots, few warps per SM) have the
  // registers for 32 (8 KB per warp), the others 16
  constexpr int DU = 16;  // (32 with 128 registers measured no better)
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[WPB];
  __shared__ __align__(8) uint64_t vbars[DIRECT ? WPB * VST : 1];  // value-stage barriers of the DIRECT blocks
  __shared__ int32_t mbox[WPB];
  __shared__ int32_t nexit;
  __shared__ __align__(8) uint64_t sigbar;
  if (A.skip && *A.skip) return;
  // the tuning / diagnostic switches (SFCDD_DAG_MODE) exist in the TRACE instantiation only: the
  // production kernel carries none of their code (C2 k_dag -6 % without the trace and mode paths)
  const int mode = TRACE ? A.mode : 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < WPB) mbox[threadIdx.x] = -1;
  if (threadIdx.x == 0) {
    nexit = 0;
    mbar_init(&sigbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == WPB) {
    if (lane == 0) signaller<WPB>(A, mode, mbox, &nexit, &sigbar);
    return;
  }
  uint64_t* bar = &bars[warp];
  if (lane == 0) {
    mbar_init(bar, 1);
    if (DIRECT)
      for (int i = 0; i < VST; ++i) mbar_init(&vbars[warp * VST + i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t phase = 0;
  uint32_t vph = 0;  // parity of each value-stage barrier's next phase (bit i: stage i)
  // queue of this warp (interleaved split of the global order: spreads the
  // claim atomics over nq lines; deadlock-free, the smallest unfinished task
  // is always claimable)
  const int q = (int)((blockIdx.x * WPB + warp) % (unsigned)A.nq);
  int32_t* qh = A.qhead + 32 * q;
  // static mode (mode bit 16, experimental): worker w runs tasks w, w + W,
  // w + 2W, ... of the queue order (W = resident workers).  Deadlock-free for
  // the same reason as claiming (each worker's list follows one topological
  // order) provided every CTA is resident -- the kernel must run alone.  No
  // claim atomic, and the next descriptor is loaded (one word per lane)
  // while the current task runs.
  const bool stat = (mode & 16) != 0;
  // hook at a FRAG task's tail, after its last level: the claim atomic of the
  // NEXT task is issued before the result stores and the completion post, so
  // its L2 round trip (~0.8 us between a worker's tasks) overlaps them.  The
  // claimed task is held for the stores only (claiming a whole level earlier
  // was measured slower: a held task delays its dependents); deadlock-free as
  // before -- this task is past its waits and completes unconditionally.
  int tnext = -1;
  auto ahead = [&]() {
    if ((mode & 64) && !stat && lane == 0) tnext = q + A.nq * atomicAdd(qh, 1);
  };
  const int nw = (int)gridDim.x * WPB;
  int ts = (int)blockIdx.x * WPB + warp;
  constexpr int TW = (int)(sizeof(TaskDev) / 4);
  static_assert(sizeof(TaskDev) % 4 == 0 && TW <= 32, "TaskDev words");
  int32_t pw = (stat && lane < TW && ts < A.ntask) ? __ldg(reinterpret_cast<const int32_t*>(A.tasks + ts) + lane) : 0;
  int dead = 0;
  for (;;) {
    int t = 0;
    if (stat) {
      t = ts;
    } else {
      if (lane == 0) {
        t = tnext >= 0 ? tnext : q + A.nq * atomicAdd(qh, 1);
        tnext = -1;
      }
      t = __shfl_sync(FULL, t, 0);
    }
    if (t >= A.ntask) {
      if (lane == 0) {  // release: ordered after this warp's last mailbox post
        asm volatile("red.release.cta.shared::cta.add.s32 [%0], 1;" ::"r"(smem_u32(&nexit)) : "memory");
        mbar_arrive(&sigbar);
      }
      break;
    }
    TaskDev T;
    if (stat) {
      static_assert(offsetof(TaskDev, copy_bytes) == 8 && offsetof(TaskDev, signal_idx) == 32, "TaskDev layout");
      T.blob_off = (int64_t)(uint32_t)__shfl_sync(FULL, pw, 0) | ((int64_t)__shfl_sync(FULL, pw, 1) << 32);
      T.copy_bytes = __shfl_sync(FULL, pw, 2);
      T.kind = __shfl_sync(FULL, pw, 3);
      T.factor = __shfl_sync(FULL, pw, 4);
      T.group = 0;
      T.wait_idx = __shfl_sync(FULL, pw, 6);
      T.wait_target = __shfl_sync(FULL, pw, 7);
      T.signal_idx = __shfl_sync(FULL, pw, 8);
      T.values = 0;
      ts += nw;
      pw = (lane < TW && ts < A.ntask) ? __ldg(reinterpret_cast<const int32_t*>(A.tasks + ts) + lane) : 0;
    } else {
      T = A.tasks[t];
    }
    // L2 prefetch of a task about one task duration ahead in the queue order
    // (whoever claims it then finds its descriptor and blob in L2, not DRAM):
    // lane 1 loads that descriptor now and issues the blob prefetch once this
    // task's own blob has arrived -- nothing on this task's chain waits for it
    int64_t pf_off = 0;
    int32_t pf_bytes = 0;
    if (A.pf_dist > 0 && lane == 1 && t + A.pf_dist < A.ntask) {
      pf_off = __ldg(&A.tasks[t + A.pf_dist].blob_off);
      pf_bytes = __ldg(&A.tasks[t + A.pf_dist].copy_bytes);
    }
    // issued now, consumed after the blob / dependency waits (off the claim chain)
    const FactorDev F = A.factors[T.factor];
    // slot addresses computed from the shared base so the compiler keeps the
    // shared state space (LDS, not generic loads) for every blob/scratch access
    const int32_t* h = reinterpret_cast<const int32_t*>(smem + (size_t)warp * A.slot_bytes);
    // the scratch follows the task's own blob (128-byte aligned): blob and
    // scratch share the slot, so small-scratch tasks carry larger blobs
    double* S = reinterpret_cast<double*>(smem + (size_t)warp * A.slot_bytes + ((T.copy_bytes + 127) & ~127));
    unsigned long long* tr = TRACE && A.trace ? A.trace + 5 * (size_t)t : nullptr;
    if (lane == 0) {
      if (tr) {
        tr[0] = smid() | ((unsigned long long)(blockIdx.x * WPB + warp) << 16);  // sm | worker id << 16
        tr[1] = gtimer();
      }
      // the blob does not depend on other tasks: copy it while waiting
      fence_proxy_async();
      mbar_expect_tx(bar, (uint32_t)T.copy_bytes);
      if (mode & 4)
        bulk_g2s(smem + (size_t)warp * A.slot_bytes, A.blobs + T.blob_off, (uint32_t)T.copy_bytes, bar);
      else
        bulk_g2s_hint(smem + (size_t)warp * A.slot_bytes, A.blobs + T.blob_off, (uint32_t)T.copy_bytes, bar,
                      policy_evict_first());
      if (T.wait_idx >= 0) {
        // relaxed polling (no L1 invalidation per poll), one acquire at the end
        unsigned ns = 32;
        unsigned polls = 0;
        unsigned long long t0 = 0;
        auto watchdog = [&]() {  // a dependency that never completes traps instead of hanging the GPU
          if (SFCDD_LEAN & 1) return;
          if ((++polls & 4095u) == 0) {
            if (t0 == 0) t0 = gtimer();
            if (mode & 32) {  // diagnostic mode: record the stuck wait, let every warp leave
              if (ld_relaxed(A.diag) != 0) dead = 1;
              else if (gtimer() - t0 > A.watchdog_ns && atomicCAS(A.diag, 0, 1) == 0) {
                A.diag[1] = t;
                A.diag[2] = T.wait_idx;
                A.diag[3] = ld_relaxed(A.ctr + T.wait_idx);
                A.diag[4] = T.wait_target;
                A.diag[5] = T.kind;
                A.diag[6] = T.group;
                dead = 1;
              }
            } else if (gtimer() - t0 > A.watchdog_ns) {
              __trap();
            }
          }
        };
        if (mode & 1) {
          while (!((SFCDD_LEAN & 16) ? 0 : dead) && ld_acquire(A.ctr + T.wait_idx) < T.wait_target) {
            __nanosleep(ns);
            ns = ns < 256 ? 2 * ns : 256;
            watchdog();
          }
        } else {
          while (!((SFCDD_LEAN & 16) ? 0 : dead) && ld_relaxed(A.ctr + T.wait_idx) < T.wait_target) {
            __nanosleep(ns);
            ns = ns < 256 ? 2 * ns : 256;
            watchdog();
          }
          (void)ld_acquire(A.ctr + T.wait_idx);
        }
      }
      if (tr) tr[2] = gtimer();
    }
    __syncwarp();
    if (SFCDD_LEAN & 1)
      mbar_wait(bar, phase);
    else
      mbar_wait_guard(bar, phase);
    phase ^= 1u;
    if (!(SFCDD_LEAN & 1) && (mode & 32)) {  // diagnostic mode: leave once a stuck wait was recorded
      dead = __shfl_sync(FULL, dead, 0);
      if (dead) {
        if (lane == 0) {
          asm volatile("red.release.cta.shared::cta.add.s32 [%0], 1;" ::"r"(smem_u32(&nexit)) : "memory");
          mbar_arrive(&sigbar);
        }
        break;
      }
    }
    if (tr && lane == 0) tr[3] = gtimer();
    if (pf_bytes > 0)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.blobs + pf_off), "r"(pf_bytes) : "memory");
#if !(SFCDD_LEAN & 32)  // (the if-chain measured 3 % faster than the switch below on C2: code layout)
    if ((SFCDD_LEAN & 4) && T.kind == TK_FRAG_FWD) {
      run_frag<8>(h, true, S, A, F, lane, TRACE && A.ptrace ? A.ptrace + 16 * (size_t)t : nullptr, ahead);
    } else if ((SFCDD_LEAN & 4) && T.kind == TK_FRAG_BWD) {
      run_frag<8>(h, false, S, A, F, lane, TRACE && A.ptrace ? A.ptrace + 16 * (size_t)t : nullptr, ahead);
    } else if (T.kind == TK_FRAG_FWD || T.kind == TK_FRAG_BWD) {
      run_frag<8>(h, T.kind == TK_FRAG_FWD, S, A, F, lane, TRACE && A.ptrace ? A.ptrace + 16 * (size_t)t : nullptr, ahead);
    } else if (SPLIT && T.kind == TK_ASM_FWD) {
      run_asm(h, A, F, lane);
    } else if (SPLIT && T.kind == TK_XB_BWD) {
      run_xb(h, A, F, lane);
    } else if (T.kind == TK_ROW_FWD && (!DIRECT || h[RW_INBLOB])) {
      run_row_blob<SPLIT, WPB == 2>(h, S, A, F, lane, bar, phase, TRACE && A.ptrace ? A.ptrace + 16 * (size_t)t : nullptr);
    } else if (T.kind == TK_COL_BWD && (!DIRECT || h[CL_INBLOB])) {
      run_col_blob<SPLIT, WPB == 2>(h, S, A, F, lane, bar, phase);
    } else if constexpr (DIRECT) {
      if (TRACE && SPLIT && T.kind == TK_ROW_FWD && h[RW_NBLK] > 1)  // (MROW tasks: opt-in plans, TRACE instantiation)
        phase = run_mrow<16, WPB == 2>(h, S, A, A.blobs + T.blob_off, lane, bar, phase);
      else
        phase = run_dense<SPLIT, DU>(T.kind == TK_ROW_FWD, h, S, A, F, A.blobs + T.blob_off, lane, bar, phase,
                                     &vbars[DIRECT ? warp * VST : 0], vph,
                                     smem + (size_t)(warp + 1) * A.slot_bytes, !(mode & 128));
    } else {
      __trap();  // a DIRECT block in a plan built without them
    }
#else
    switch (T.kind) {
      case TK_FRAG_FWD:
        run_frag<8>(h, true, S, A, F, lane, TRACE && A.ptrace ? A.ptrace + 16 * (size_t)t : nullptr, ahead);
        break;
      case TK_FRAG_BWD:
        run_frag<8>(h, false, S, A, F, lane, TRACE && A.ptrace ? A.ptrace + 16 * (size_t)t : nullptr, ahead);
        break;
      case TK_ROW_FWD:
        if (!DIRECT || h[RW_INBLOB]) {
          run_row_blob<SPLIT, WPB == 2>(h, S, A, F, lane, bar, phase, TRACE && A.ptrace ? A.ptrace + 16 * (size_t)t : nullptr);
          break;
        }
        [[fallthrough]];
      default:
        if constexpr (SPLIT) {
          if (T.kind == TK_ASM_FWD) {
            run_asm(h, A, F, lane);
            break;
          }
          if (T.kind == TK_XB_BWD) {
            run_xb(h, A, F, lane);
            break;
          }
        }
        if (T.kind == TK_COL_BWD && (!DIRECT || h[CL_INBLOB])) {
          run_col_blob<SPLIT, WPB == 2>(h, S, A, F, lane, bar, phase);
          break;
        }
        if constexpr (DIRECT) {  // ROW or COL block streamed from HBM
          if (TRACE && SPLIT && T.kind == TK_ROW_FWD && h[RW_NBLK] > 1)  // (MROW tasks: opt-in plans, TRACE instantiation)
            phase = run_mrow<16, WPB == 2>(h, S, A, A.blobs + T.blob_off, lane, bar, phase);
          else
            phase = run_dense<SPLIT, DU>(T.kind == TK_ROW_FWD, h, S, A, F, A.blobs + T.blob_off, lane, bar, phase,
                                     &vbars[DIRECT ? warp * VST : 0], vph,
                                     smem + (size_t)(warp + 1) * A.slot_bytes, !(mode & 128));
        }
        break;
    }
#endif
    __syncwarp();
    if (lane == 0) {
      // release: cumulative over the warp's writes (ordered before it by __syncwarp)
      if (mode & 2) {  // direct release by the worker (old path)
        red_release_add(A.ctr + T.signal_idx, 1);
      } else {
        while (ld_acquire_cta(&mbox[warp]) >= 0) __nanosleep(20);  // signaller still busy with the last one
        st_release_cta(&mbox[warp], T.signal_idx);
        mbar_arrive(&sigbar);
      }
      if (tr) tr[4] = gtimer();
    }
  }
}

inline int32_t round128(int64_t x) { return (int32_t)((x + 127) / 128 * 128); }

// deferred-value plans: metadata segments (16-byte multiples) -> blob buffer
__global__ void k_meta_scatter(const MetaSeg* __restrict__ segs, int64_t nseg, const uint8_t* __restrict__ img,
                               uint8_t* __restrict__ blobs) {
  for (int64_t sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
    const MetaSeg S = segs[sg];
    const int4* src = reinterpret_cast<const int4*>(img + S.host_off);
    int4* dst = reinterpret_cast<int4*>(blobs + S.dev_off);
    for (int64_t i = threadIdx.x; i < S.bytes / 16; i += blockDim.x) dst[i] = src[i];
  }
}

// value placement (plan.h ValDesc, host twin place_values in plan.cpp): one
// warp per descriptor; src = the factor's packed values (HostFactor::val layout)
__global__ void k_place_values(const ValDesc* __restrict__ vd, int64_t nvd, const double* __restrict__ vals,
                               const int64_t* __restrict__ fbase, int32_t f0, uint8_t* __restrict__ blobs) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = w0; q < nvd; q += nw) {
    const ValDesc d = vd[q];
    const double* M = vals + fbase[d.factor - f0] + d.src;
    double* out = reinterpret_cast<double*>(blobs + d.dst);
    if (d.kind == VD_COPY) {
      for (int32_t i = lane; i < d.len; i += 32) out[i] = M[i];
    } else if (d.kind == VD_ROW) {
      const int32_t nr = d.rows > 0 ? d.rows : d.w;
      for (int32_t k = 0; k < d.len; ++k) {
        const double* col = M + packed_col_off(d.s, d.m, k);
        for (int32_t i = max(0, k - d.p0) + lane; i < nr; i += 32) out[(int64_t)k * d.w + i] = col[d.p0 + i - k];
      }
    } else {
      for (int32_t j = 0; j < d.w; ++j) {
        const double* col = M + packed_col_off(d.s, d.m, d.p0 + j);
        for (int32_t r = j + lane; r < d.len; r += 32) out[(int64_t)r * d.w + j] = col[r - j];
      }
    }
  }
}

}  // namespace

void DagSolver::place_values(int32_t f0, int32_t f1, const double* vals_dev, const int64_t* fbase_host,
                             cudaStream_t st) {
  SFCDD_REQUIRE(f0 >= 0 && f1 <= (int32_t)vd_ptr_.size() - 1 && f0 <= f1, SFCDD_EINTERNAL, "factor range");
  const int64_t q0 = vd_ptr_[f0], q1 = vd_ptr_[f1];
  if (q1 == q0) return;
  ValDesc* dvd = nullptr;
  int64_t* dfb = nullptr;
  CUDA_CHECK(cudaMallocAsync(&dvd, (q1 - q0) * sizeof(ValDesc), st));
  CUDA_CHECK(cudaMallocAsync(&dfb, (f1 - f0) * sizeof(int64_t), st));
  CUDA_CHECK(cudaMemcpyAsync(dvd, vdesc_.data() + q0, (q1 - q0) * sizeof(ValDesc), cudaMemcpyHostToDevice, st));
  CUDA_CHECK(cudaMemcpyAsync(dfb, fbase_host, (f1 - f0) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  const int64_t blocks = std::min<int64_t>((q1 - q0 + 7) / 8, 148 * 16);
  k_place_values<<<(unsigned)blocks, 256, 0, st>>>(dvd, q1 - q0, vals_dev, dfb, f0, blobs_);
  CUDA_CHECK(cudaGetLastError());
  CUDA_CHECK(cudaFreeAsync(dvd, st));
  CUDA_CHECK(cudaFreeAsync(dfb, st));
}

DagSolver::DagSolver(const DevicePlan& plan, int device, int64_t extra_xy) : device_(device) {
  CUDA_CHECK(cudaSetDevice(device));
  ngroups_ = plan.ngroups;
  ntask_ = (int32_t)plan.tasks.size();
  host_tasks = plan.tasks;
  blob_max_ = round128(plan.blob_max);
  slot_bytes_ = round128(std::max<int64_t>(plan.slot_need, 256));
  // worker warps per CTA: the plan's choice (plan.h choose_blob_shape, SFCDD_WPB)
  wpb_ = plan.wpb;
  SFCDD_REQUIRE(wpb_ == 2 || wpb_ == 4 || wpb_ == 8, SFCDD_EVALUE, "worker warps per CTA must be 2, 4 or 8");
  bool split = false;
  for (const TaskDev& T : plan.tasks) split = split || T.kind == TK_ASM_FWD || T.kind == TK_XB_BWD;
  auto pick = [&](auto sp, auto dr, auto tr) -> const void* {
    constexpr bool SP = decltype(sp)::value, DR = decltype(dr)::value, TR = decltype(tr)::value;
    return wpb_ == 2   ? (const void*)k_dag<2, SP, DR, TR>
           : wpb_ == 4 ? (const void*)k_dag<4, SP, DR, TR>
                       : (const void*)k_dag<8, SP, DR, TR>;
  };
  using T_ = std::true_type;
  using F_ = std::false_type;
  kern_ = split ? (plan.has_direct ? pick(T_{}, T_{}, F_{}) : pick(T_{}, F_{}, F_{}))
                : (plan.has_direct ? pick(F_{}, T_{}, F_{}) : pick(F_{}, F_{}, F_{}));
  kern_trace_ = split ? (plan.has_direct ? pick(T_{}, T_{}, T_{}) : pick(T_{}, F_{}, T_{}))
                      : (plan.has_direct ? pick(F_{}, T_{}, T_{}) : pick(F_{}, F_{}, T_{}));
  split_ = split;
  has_mrow_ = plan.has_mrow;
  if (const char* e = std::getenv("SFCDD_DAG_MODE")) mode_ = std::atoi(e);
  if (const char* e = std::getenv("SFCDD_SIG_NS")) sig_ns_ = std::atoi(e);
  if (const char* e = std::getenv("SFCDD_SIG_WAIT_NS")) sig_wait_ns_ = std::atoi(e);
  // L2 prefetch-ahead where the blobs of one launch are many times the L2 (measured with the
  // final kernel: C3 4.7 GB -0.8 %, C4 15 GB -3 %, C5 92 GB -1.8 %; C2 0.9 GB +1.1 %: off)
  pf_dist_ = plan.blob_bytes > (2ll << 30) ? 1536 : 0;
  if (const char* e = std::getenv("SFCDD_PF_DIST")) pf_dist_ = std::max(0, std::atoi(e));
  for (const FactorDev& F : plan.factors) rhs_doubles_ = std::max<int64_t>(rhs_doubles_, F.gmod);
  if (const char* e = std::getenv("SFCDD_L2_PERSIST")) l2_persist_ = std::atoi(e);
  if (l2_persist_) CUDA_CHECK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 48u << 20));
  smem_ = wpb_ * slot_bytes_;
  SFCDD_REQUIRE(smem_ <= 227 * 1024, SFCDD_EINTERNAL, "DAG shared-memory footprint exceeds 227 KB");
  auto up = [&](void** dst, const void* src, size_t bytes) {
    CUDA_CHECK(cudaMalloc(dst, std::max<size_t>(bytes, 16) + 16));  // (+16: 16-byte rounded tails of bulk copies)
    if (bytes) CUDA_CHECK(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
    bytes_ += std::max<size_t>(bytes, 16);
  };
  if (!plan.deferred) {
    SFCDD_REQUIRE((int64_t)plan.blobs.size() == plan.blob_bytes, SFCDD_EINTERNAL, "blob image size");
    up((void**)&blobs_, plan.blobs.data(), plan.blobs.size());
  } else {
    // metadata now (staged image + segment scatter), values later (place_values)
    CUDA_CHECK(cudaMalloc(&blobs_, std::max<int64_t>(plan.blob_bytes, 16) + 16));  // (+16: a value stage's 16-byte rounded tail)
    bytes_ += std::max<int64_t>(plan.blob_bytes, 16);
    CUDA_CHECK(cudaMemset(blobs_, 0, std::max<int64_t>(plan.blob_bytes, 16)));
    uint8_t* img = nullptr;
    MetaSeg* sg = nullptr;
    CUDA_CHECK(cudaMalloc(&img, std::max<size_t>(plan.blobs.size(), 16)));
    CUDA_CHECK(cudaMalloc(&sg, std::max<size_t>(plan.segs.size() * sizeof(MetaSeg), 16)));
    CUDA_CHECK(cudaMemcpy(img, plan.blobs.data(), plan.blobs.size(), cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(sg, plan.segs.data(), plan.segs.size() * sizeof(MetaSeg), cudaMemcpyHostToDevice));
    if (!plan.segs.empty()) {
      k_meta_scatter<<<(unsigned)std::min<size_t>(plan.segs.size(), 148 * 64), 128>>>(
          sg, (int64_t)plan.segs.size(), img, blobs_);
      CUDA_CHECK(cudaGetLastError());
    }
    CUDA_CHECK(cudaDeviceSynchronize());
    CUDA_CHECK(cudaFree(img));
    CUDA_CHECK(cudaFree(sg));
  }
  // value descriptors grouped by factor (deferred plans: filled by place_values)
  if (plan.deferred) vdesc_ = plan.vdesc;
  vd_ptr_.assign(plan.factors.size() + 1, 0);
  {
    std::vector<int64_t> cnt(plan.factors.size() + 1, 0);
    for (const ValDesc& d : plan.vdesc) cnt[d.factor + 1]++;
    for (size_t f = 0; f < plan.factors.size(); ++f) vd_ptr_[f + 1] = vd_ptr_[f] + cnt[f + 1];
  }
  up((void**)&tasks_, plan.tasks.data(), plan.tasks.size() * sizeof(TaskDev));
  up((void**)&factors_, plan.factors.data(), plan.factors.size() * sizeof(FactorDev));
  // (+8: the 16-byte rounded bulk copies of run_row / run_col may read a
  // few doubles past the last slot)
  CUDA_CHECK(cudaMalloc(&upd_, (std::max<int64_t>(plan.upd_doubles, 2) + 8) * 8));
  CUDA_CHECK(cudaMemset(upd_, 0, (std::max<int64_t>(plan.upd_doubles, 2) + 8) * 8));
  CUDA_CHECK(cudaMalloc(&xy_, std::max<int64_t>(plan.xy_doubles + extra_xy, 2) * 8));
  xy_doubles_ = plan.xy_doubles + extra_xy;
  // counters (plan.h) then nq queue heads, one per 128-byte line; one memset per solve
  nq_ = 16;
  if (const char* e = std::getenv("SFCDD_QUEUES")) nq_ = std::max(1, std::atoi(e));
  const int64_t cw = (1 + CTR_PER_GROUP * (int64_t)ngroups_ + 31) / 32 * 32;
  ctr_words_ = cw + 32 * (int64_t)nq_ + 32;  // + one line of diagnostics (mode bit 32)
  CUDA_CHECK(cudaMalloc(&ctr_, ctr_words_ * 4));
  qhead_ = ctr_ + cw;
  if (const char* e = std::getenv("SFCDD_WATCHDOG_MS")) watchdog_ms_ = std::max(1, std::atoi(e));
  bytes_ += std::max<int64_t>(plan.upd_doubles, 2) * 8 + std::max<int64_t>(xy_doubles_, 2) * 8 + ctr_words_ * 4;
  {
    // the attribute is per function: only ever raise it, so every live
    // solver (several handles per process in shard emulation) can launch
    // (the attribute is per device: the cache is keyed by device and kernel)
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> max_smem;
    std::lock_guard<std::mutex> g(mu);
    for (const void* k : {kern_, kern_trace_}) {
      int& cur = max_smem[{device, k}];
      if (smem_ > cur) {
        CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_));
        cur = smem_;
      }
    }
  }
  int per_sm = 0, sms = 0;
  CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern_, (wpb_ + 1) * 32, smem_));
  CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  SFCDD_REQUIRE(per_sm >= 1, SFCDD_EINTERNAL, "DAG kernel cannot be resident");
  if (const char* e = std::getenv("SFCDD_CTAS_PER_SM")) per_sm = std::max(1, std::min(per_sm, std::atoi(e)));
  grid_ = std::max(1, std::min(per_sm * sms, (ntask_ + wpb_ - 1) / wpb_));
  if (std::getenv("SFCDD_PLAN_DEBUG"))
    std::fprintf(stderr, "[dag] %d tasks, %d-worker CTAs, slot %d B (blob %d), %d B smem per CTA, %d CTAs per SM, grid %d\n",
                 ntask_, wpb_, slot_bytes_, blob_max_, smem_, per_sm, grid_);
}

DagSolver::~DagSolver() {
  cudaFree(blobs_);
  cudaFree(tasks_);
  cudaFree(factors_);
  cudaFree(upd_);
  cudaFree(xy_);
  cudaFree(ctr_);
}

void DagSolver::solve(const double* rhs, cudaStream_t st, const int32_t* skip) {
  if (ntask_ == 0) return;
  CUDA_CHECK(cudaMemsetAsync(ctr_, 0, ctr_words_ * 4, st));
  DagArgs a;
  a.tasks = tasks_;
  a.ntask = ntask_;
  a.slot_bytes = slot_bytes_;
  a.blob_max = blob_max_;
  a.blobs = blobs_;
  a.factors = factors_;
  a.rhs = rhs;
  a.xy = xy_;
  a.upd = upd_;
  a.ctr = ctr_;
  a.qhead = qhead_;
  a.nq = nq_;
  a.skip = skip;
  a.trace = trace_;
  a.ptrace = trace_ ? trace_ + 5 * (size_t)ntask_ : nullptr;
  a.mode = mode_;
  a.sig_ns = sig_ns_;
  a.sig_wait_ns = (uint32_t)sig_wait_ns_;
  a.diag = qhead_ + 32 * (int64_t)nq_;
  a.watchdog_ns = 1000000ull * (unsigned long long)watchdog_ms_;
  a.pf_dist = pf_dist_;
  void* params[] = {&a};
  // (mode switches and MROW tasks: TRACE instantiation only)
  const void* kern = (trace_ || mode_ != 0 || has_mrow_) ? kern_trace_ : kern_;
  if (l2_persist_) {  // experiment: keep the gathered vector resident in L2 while the blobs stream through
    cudaStreamAttrValue av{};
    av.accessPolicyWindow.base_ptr = l2_persist_ == 2 ? (void*)xy_ : (void*)rhs;
    av.accessPolicyWindow.num_bytes =
        (size_t)std::min<int64_t>(8 * (l2_persist_ == 2 ? xy_doubles_ : rhs_doubles_), 32ll << 20);
    av.accessPolicyWindow.hitRatio = 1.0f;
    av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    CUDA_CHECK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
  }
  if (mode_ & 16)  // static worker lists need every CTA resident: cooperative launch guarantees it (or fails)
    CUDA_CHECK(cudaLaunchCooperativeKernel(kern, dim3(grid_), dim3((wpb_ + 1) * 32), params, smem_, st));
  else
    CUDA_CHECK(cudaLaunchKernel(kern, dim3(grid_), dim3((wpb_ + 1) * 32), params, smem_, st));
  if (l2_persist_) {
    cudaStreamAttrValue av{};
    av.accessPolicyWindow.num_bytes = 0;
    CUDA_CHECK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
  }
  if (mode_ & 32) {  // diagnostic mode (not capturable): report a stuck dependency wait
    int32_t d[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    CUDA_CHECK(cudaMemcpyAsync(d, a.diag, sizeof(d), cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    if (d[0] != 0)
      throw Error(SFCDD_EINTERNAL, "DAG dependency wait timed out: task " + std::to_string(d[1]) + " (kind " +
                                       std::to_string(d[5]) + ", group " + std::to_string(d[6]) + ") waits on counter " +
                                       std::to_string(d[2]) + " = " + std::to_string(d[3]) + " < " +
                                       std::to_string(d[4]) + " of " + std::to_string(ngroups_) + " groups, " +
                                       std::to_string(ntask_) + " tasks");
  }
}

void DagSolver::set_trace(unsigned long long* dev_buf) { trace_ = dev_buf; }

}  // namespace sfcdd
