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
//    cp.async.bulk (TMA bulk copy) completing on an mbarrier; the copy is
//    issued before the task's dependencies are awaited, so the factor
//    stream overlaps the dataflow waits;
//  * CTAs pull tasks from a global queue in topological order and wait on
//    per-fragment counters (acquire/release) -- no grid barrier, no host
//    round trip, deadlock-free because a task only waits on earlier tasks;
//  * multifrontal update vectors between fragments live in a global slot
//    buffer and are summed by the parent in fixed child order, so results
//    are bitwise reproducible run to run.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"
#include "dag_solve.h"

namespace sfcdd {

namespace {

constexpr int DAG_THREADS = 256;
constexpr int NWARP = DAG_THREADS / 32;

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
  const int32_t* skip;  // optional: nonzero -> whole solve skipped (PCG done)
};

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

// ---------------------------------------------------------------- forward
// f = [rhs(cols) ; 0] + sum_children extend(u_K); then out = M f[:s];
// y = out[:s] -> xy;  u = f[s:] - out[s:] (kept in f[s:])
__device__ void assemble_front(const int32_t* h, const int32_t* R, double* f, double* scratch,
                               const DagArgs& A, const FactorDev& F, int i0, int stride,
                               bool warp_scope) {
  const int s = R[R_S], m = R[R_M];
  const int32_t* ro = h + R[R_IDX];
  for (int i = i0; i < s + m; i += stride) f[i] = i < s ? __ldg(A.rhs + gidx(F, ro[i])) : 0.0;
  if (warp_scope)
    __syncwarp();
  else
    __syncthreads();
  const int32_t* recs = h + h[H_REC];
  for (int q = 0; q < R[R_NCH]; ++q) {
    const int32_t* cr = h + R[R_CH] + CH_WORDS * q;
    const int mk = cr[1];
    const int32_t* rel = h + cr[2];
    if (cr[0] >= 0) {
      const int32_t* RC = recs + R_WORDS * cr[0];
      const double* src = scratch + RC[R_SCR] + RC[R_S];
      for (int a = i0; a < mk; a += stride) f[rel[a]] += src[a];
    } else {
      const double* src = A.upd + cr[3];
      for (int a = i0; a < mk; a += stride) f[rel[a]] += __ldcg(src + a);
    }
    if (warp_scope)
      __syncwarp();
    else
      __syncthreads();
  }
}

__device__ void fwd_sn_warp(const int32_t* h, const int32_t* R, const double* vals, double* scratch,
                            const DagArgs& A, const FactorDev& F, int lane) {
  const int s = R[R_S], m = R[R_M];
  double* f = scratch + R[R_SCR];
  const int32_t* ro = h + R[R_IDX];
  assemble_front(h, R, f, scratch, A, F, lane, 32, true);
  const double* M = vals + R[R_VAL];
  for (int i = lane; i < s + m; i += 32) {
    const int kmax = i < s ? i : s - 1;
    double acc = 0.0;
    int idx = i, step = s + m - 1;
    for (int k = 0; k <= kmax; ++k) {
      acc = fma(M[idx], f[k], acc);
      idx += step;
      --step;
    }
    if (i < s)
      A.xy[F.xy_off + ro[i]] = acc;
    else
      f[i] -= acc;
  }
  __syncwarp();
  if (R[R_PARENT] < 0 && h[H_TOP_UPD] >= 0)
    for (int a = lane; a < m; a += 32) A.upd[h[H_TOP_UPD] + a] = f[s + a];
}

// single big supernode, values streamed from global (read-only path)
__device__ void fwd_big(const int32_t* h, const double* Mg, double* scratch, const DagArgs& A,
                        const FactorDev& F) {
  const int32_t* R = h + h[H_REC];
  const int s = R[R_S], m = R[R_M];
  double* f = scratch + R[R_SCR];
  const int32_t* ro = h + R[R_IDX];
  assemble_front(h, R, f, scratch, A, F, threadIdx.x, DAG_THREADS, false);
  const double* M = Mg + R[R_VAL];
  for (int i0 = 0; i0 < s + m; i0 += DAG_THREADS) {
    const int i = i0 + threadIdx.x;
    if (i < s + m) {
      const int kmax = i < s ? i : s - 1;
      double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
      int64_t idx = i;
      int step = s + m - 1;
      int k = 0;
      for (; k + 3 <= kmax; k += 4) {
        const int64_t i1 = idx + step, i2 = i1 + step - 1, i3 = i2 + step - 2;
        const double m0 = __ldg(M + idx), m1 = __ldg(M + i1), m2 = __ldg(M + i2), m3 = __ldg(M + i3);
        acc0 = fma(m0, f[k], acc0);
        acc1 = fma(m1, f[k + 1], acc1);
        acc2 = fma(m2, f[k + 2], acc2);
        acc3 = fma(m3, f[k + 3], acc3);
        idx = i3 + step - 3;
        step -= 4;
      }
      for (; k <= kmax; ++k) {
        acc0 = fma(__ldg(M + idx), f[k], acc0);
        idx += step;
        --step;
      }
      const double acc = (acc0 + acc1) + (acc2 + acc3);
      if (i < s)
        A.xy[F.xy_off + ro[i]] = acc;
      else
        f[i] -= acc;  // only f[0:s) is read by other threads
    }
  }
  __syncthreads();
  if (h[H_TOP_UPD] >= 0)
    for (int a = threadIdx.x; a < m; a += DAG_THREADS) A.upd[h[H_TOP_UPD] + a] = f[s + a];
}

// --------------------------------------------------------------- backward
// x_J = M^T [y_J ; -x_B]
__device__ void bwd_sn_warp(const int32_t* h, const int32_t* R, const double* vals, double* scratch,
                            const DagArgs& A, const FactorDev& F, int lane) {
  const int s = R[R_S], m = R[R_M];
  double* v = scratch + R[R_SCR];
  const int32_t* ro = h + R[R_IDX];
  double* xy = A.xy + F.xy_off;
  for (int i = lane; i < s + m; i += 32) {
    const double t = __ldcg(xy + ro[i]);
    v[i] = i < s ? t : -t;
  }
  __syncwarp();
  const double* M = vals + R[R_VAL];
  int64_t coff = 0;
  for (int k = 0; k < s; ++k) {
    const int len = s + m - k;
    const double* col = M + coff;
    double acc = 0.0;
    for (int t = lane; t < len; t += 32) acc = fma(col[t], v[k + t], acc);
    acc = warp_sum(acc);
    if (lane == 0) xy[ro[k]] = acc;
    coff += len;
  }
}

__device__ void bwd_big(const int32_t* h, const double* Mg, double* scratch, const DagArgs& A,
                        const FactorDev& F, int lane, int warp) {
  const int32_t* R = h + h[H_REC];
  const int s = R[R_S], m = R[R_M];
  double* v = scratch + R[R_SCR];
  const int32_t* ro = h + R[R_IDX];
  double* xy = A.xy + F.xy_off;
  for (int i = threadIdx.x; i < s + m; i += DAG_THREADS) {
    const double t = __ldcg(xy + ro[i]);
    v[i] = i < s ? t : -t;
  }
  __syncthreads();
  const double* M = Mg + R[R_VAL];
  for (int k = warp; k < s; k += NWARP) {
    const int len = s + m - k;
    const double* col = M + packed_col_off(s, m, k);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int t = lane;
    for (; t + 96 < len; t += 128) {
      a0 = fma(__ldg(col + t), v[k + t], a0);
      a1 = fma(__ldg(col + t + 32), v[k + t + 32], a1);
      a2 = fma(__ldg(col + t + 64), v[k + t + 64], a2);
      a3 = fma(__ldg(col + t + 96), v[k + t + 96], a3);
    }
    for (; t < len; t += 32) a0 = fma(__ldg(col + t), v[k + t], a0);
    const double acc = warp_sum((a0 + a1) + (a2 + a3));
    if (lane == 0) xy[ro[k]] = acc;
  }
}

__global__ void __launch_bounds__(DAG_THREADS, 2) k_dag(DagArgs A) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ int32_t s_task;
  uint8_t* blob = smem;
  double* scratch = reinterpret_cast<double*>(smem + A.blob_max);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (A.skip && *A.skip) return;
  int32_t* fwd_cnt = A.ctr + 1;
  int32_t* fwd_done = fwd_cnt + A.nfrag;
  int32_t* bwd_done = fwd_done + A.nfrag;
  if (tid == 0) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase = 0;
  for (;;) {
    if (tid == 0) s_task = atomicAdd(A.ctr, 1);
    __syncthreads();
    const int32_t t = s_task;
    if (t >= A.ntask) break;
    const TaskDev T = A.tasks[t];
    const bool fwd = t < A.nfrag;
    if (tid == 0) {
      fence_proxy_async();
      mbar_expect_tx(&mbar, (uint32_t)T.copy_bytes);
      bulk_g2s(blob, A.blobs + T.blob_off, (uint32_t)T.copy_bytes, &mbar);
      if (fwd) {
        if (T.wait_on > 0)
          while (ld_acquire(fwd_cnt + T.frag) < T.wait_on) __nanosleep(32);
      } else {
        const int32_t* flag = T.wait_on >= 0 ? bwd_done + T.wait_on : fwd_done + T.frag;
        while (ld_acquire(flag) == 0) __nanosleep(32);
      }
    }
    mbar_wait(&mbar, phase);
    phase ^= 1u;
    __syncthreads();
    const int32_t* h = reinterpret_cast<const int32_t*>(blob);
    const FactorDev F = A.factors[T.factor];
    if (T.big) {
      const double* Mg = reinterpret_cast<const double*>(A.blobs + T.blob_off + h[H_VAL_OFF]);
      if (fwd)
        fwd_big(h, Mg, scratch, A, F);
      else
        bwd_big(h, Mg, scratch, A, F, lane, warp);
    } else {
      const double* vals = reinterpret_cast<const double*>(blob + h[H_VAL_OFF]);
      const int32_t nlev = h[H_NLEV];
      const int32_t* lev_ptr = h + h[H_LEV_PTR];
      const int32_t* lev_list = h + h[H_LEV_LIST];
      const int32_t* recs = h + h[H_REC];
      if (fwd) {
        for (int lv = 0; lv < nlev; ++lv) {
          for (int j = lev_ptr[lv] + warp; j < lev_ptr[lv + 1]; j += NWARP)
            fwd_sn_warp(h, recs + R_WORDS * lev_list[j], vals, scratch, A, F, lane);
          __syncthreads();
        }
      } else {
        for (int lv = nlev - 1; lv >= 0; --lv) {
          for (int j = lev_ptr[lv] + warp; j < lev_ptr[lv + 1]; j += NWARP)
            bwd_sn_warp(h, recs + R_WORDS * lev_list[j], vals, scratch, A, F, lane);
          __syncthreads();
        }
      }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      if (fwd) {
        if (T.signal >= 0) atomicAdd(fwd_cnt + T.signal, 1);
        st_release(fwd_done + T.frag, 1);
      } else {
        st_release(bwd_done + T.frag, 1);
      }
    }
  }
}

}  // namespace

DagSolver::DagSolver(const DevicePlan& plan, int device) : device_(device) {
  CUDA_CHECK(cudaSetDevice(device));
  nfrag_ = plan.nfrag;
  ntask_ = (int32_t)plan.tasks.size();
  xy_doubles_ = plan.xy_doubles;
  blob_max_ = (int32_t)((std::max(plan.max_copy, 16) + 127) / 128 * 128);
  smem_ = blob_max_ + 8 * std::max(plan.max_scratch, 2);
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
  CUDA_CHECK(cudaMalloc(&xy_, std::max<int64_t>(plan.xy_doubles, 2) * 8));
  ctr_words_ = 1 + 3 * nfrag_;
  CUDA_CHECK(cudaMalloc(&ctr_, ctr_words_ * 4));
  bytes_ += std::max<int64_t>(plan.upd_doubles, 2) * 8 + std::max<int64_t>(plan.xy_doubles, 2) * 8 + ctr_words_ * 4;
  CUDA_CHECK(cudaFuncSetAttribute(k_dag, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_));
  int per_sm = 0, sms = 0;
  CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dag, DAG_THREADS, smem_));
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
  a.skip = skip;
  k_dag<<<grid_, DAG_THREADS, smem_, st>>>(a);
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace sfcdd
