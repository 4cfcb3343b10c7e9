// Batched multifrontal numeric Cholesky on the device.
//
// Replaces the per-subdomain factorizations of the reference
// (linalg.Factorization -> scipy splu / cho_factor, linalg.py:40-65, called
// for every subdomain block in schwarz.py:58-61) with one device pass over a
// batch of blocks.  Input: the symbolic factors of the host analysis
// (ordering, supernodes, update row maps: chol.cpp analyze_host) and each
// block's matrix entries scattered to front positions.  Output: the
// block-inverse values M_J = [L_JJ^-1 ; L_BJ L_JJ^-1] of every supernode in the
// HostFactor::val layout, which DagSolver::place_values moves into the DAG
// blobs -- no factor value ever touches host memory.
//
// Schedule: level-synchronous over the supernodal trees of all blocks of the
// batch (level = height above the leaves, so every child is finished before
// its parent's level starts), one CTA per front, three shapes:
//   tier 1  nf <= 32: 32-thread CTA, front in shared memory;
//   tier 2  nf <= 96: 128-thread CTA, front in shared memory;
//   tier 3  larger:   256-thread CTA, front in a global workspace, blocked
//           right-looking Cholesky (unblocked 32-column panels, 64x64
//           shared-memory-tiled trailing updates), L_BJ L_JJ^-1 as a tiled
//           product.
// Per front: zero, add the matrix entries, extend-add the children's update
// matrices (children in fixed order: bitwise reproducible), partial Cholesky
// of the s pivot columns (nonpositive pivot -> FactorizationError, as
// linalg.py:51-52/62-63), in-place inverse of L_JJ, M_J packed column-major
// (col k = rows k..s+m-1), update matrix F22 - L_BJ L_BJ^T packed lower for
// the parent.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.h"
#include "gpu_factor.h"

namespace sfcdd {

namespace {

// column-major front, element (i, j) at F[j * ld + i]
__device__ __forceinline__ int64_t at(int ld, int i, int j) { return (int64_t)j * ld + i; }

template <int T>
__device__ void assemble(double* F, int nf, const FItem& it, const FChild* __restrict__ ch,
                         const int32_t* __restrict__ rel, const FAent* __restrict__ ae, const double* __restrict__ upd) {
  const int tid = threadIdx.x;
  for (int64_t e = tid; e < (int64_t)nf * nf; e += T) F[e] = 0.0;
  __syncthreads();
  for (int e = tid; e < it.a_cnt; e += T) {
    const FAent a = ae[it.a_off + e];
    F[a.idx] += a.val;  // positions are distinct within one front
  }
  __syncthreads();
  constexpr int W = T / 32;
  const int warp = tid >> 5, lane = tid & 31;
  for (int c = 0; c < it.c_cnt; ++c) {  // fixed child order
    const FChild C = ch[it.c_off + c];
    const double* U = upd + C.upd_off;
    const int32_t* r = rel + C.rel_off;
    for (int b = warp; b < C.m; b += W) {
      const double* col = U + packed_col_off(C.m, 0, b);
      const int rb = r[b];
      for (int a = b + lane; a < C.m; a += 32) F[at(nf, r[a], rb)] += col[a - b];
    }
    __syncthreads();
  }
}

// unblocked right-looking partial Cholesky of columns [k0, k1) over rows
// [k0, nf), updating only columns < kend (trailing columns >= kend are
// updated by the caller, blocked)
template <int T>
__device__ void chol_cols(double* F, int nf, int k0, int k1, int kend, int* err) {
  const int tid = threadIdx.x;
  for (int k = k0; k < k1; ++k) {
    __syncthreads();
    double d = F[at(nf, k, k)];
    if (!(d > 0.0)) {
      if (tid == 0) atomicExch(err, 1);
      d = 1.0;
    }
    d = sqrt(d);
    const double inv = 1.0 / d;
    __syncthreads();
    if (tid == 0) F[at(nf, k, k)] = d;
    for (int i = k + 1 + tid; i < nf; i += T) F[at(nf, i, k)] *= inv;
    __syncthreads();
    const int nc = kend - (k + 1);   // columns to update
    const int nr = nf - (k + 1);     // rows below the pivot
    if (nc <= 0) continue;
    for (int64_t e = tid; e < (int64_t)nc * nr; e += T) {
      const int jj = (int)(e / nr), ii = (int)(e % nr);
      if (ii < jj) continue;  // lower part only
      const int j = k + 1 + jj, i = k + 1 + ii;
      F[at(nf, i, j)] -= F[at(nf, i, k)] * F[at(nf, j, k)];
    }
  }
  __syncthreads();
}

// In-place inverse of the lower triangle L = F[0:s, 0:s] (dtrti2 order:
// columns right to left, each from the already inverted trailing block).
// tmp: s doubles of scratch.
template <int T>
__device__ void trtri_lower(double* F, int ld, int s, double* tmp) {
  const int tid = threadIdx.x;
  for (int j = s - 1; j >= 0; --j) {
    __syncthreads();
    const double wjj = 1.0 / F[at(ld, j, j)];
    // x = L[j+1:, j];  new column = -wjj * W22 x  (W22 lower, already inverted)
    for (int i = j + 1 + tid; i < s; i += T) {
      double acc = 0.0;
      for (int t = j + 1; t <= i; ++t) acc = fma(F[at(ld, i, t)], F[at(ld, t, j)], acc);
      tmp[i] = acc;
    }
    __syncthreads();
    for (int i = j + 1 + tid; i < s; i += T) F[at(ld, i, j)] = -wjj * tmp[i];
    if (tid == 0) F[at(ld, j, j)] = wjj;
  }
  __syncthreads();
}

// packed M = [W ; L21 W] (small fronts: direct dots) and the packed update
template <int T>
__device__ void write_outputs_direct(const double* F, int nf, int s, int m, double* M, double* U) {
  const int tid = threadIdx.x;
  // M_top: column k rows k..s-1
  for (int64_t e = tid; e < (int64_t)s * s; e += T) {
    const int k = (int)(e / s), i = (int)(e % s);
    if (i >= k) M[packed_col_off(s, m, k) + (i - k)] = F[at(nf, i, k)];
  }
  // M_bot(a, k) = sum_{t=k}^{s-1} L21(a, t) W(t, k)
  for (int64_t e = tid; e < (int64_t)s * m; e += T) {
    const int k = (int)(e / m), a = (int)(e % m);
    double acc = 0.0;
    for (int t = k; t < s; ++t) acc = fma(F[at(nf, s + a, t)], F[at(nf, t, k)], acc);
    M[packed_col_off(s, m, k) + (s - k) + a] = acc;
  }
  if (U) {
    for (int b = tid >> 5; b < m; b += T / 32)
      for (int a = b + (tid & 31); a < m; a += 32) U[packed_col_off(m, 0, b) + (a - b)] = F[at(nf, s + a, s + b)];
  }
}

template <int T, int NFMAX>
__global__ void __launch_bounds__(T) k_front_smem(const FItem* __restrict__ items, const int32_t* __restrict__ list,
                                                  const FChild* __restrict__ ch, const int32_t* __restrict__ rel,
                                                  const FAent* __restrict__ ae, double* __restrict__ vals,
                                                  double* __restrict__ upd, int* err) {
  extern __shared__ double sm[];
  const FItem it = items[list[blockIdx.x]];
  const int s = it.s, m = it.m, nf = s + m;
  double* F = sm;
  double* tmp = sm + NFMAX * NFMAX;
  assemble<T>(F, nf, it, ch, rel, ae, upd);
  chol_cols<T>(F, nf, 0, s, nf, err);
  trtri_lower<T>(F, nf, s, tmp);
  write_outputs_direct<T>(F, nf, s, m, vals + it.val_off, it.upd_off >= 0 ? upd + it.upd_off : nullptr);
}

// ---------------------------------------------------------------- tier 3
constexpr int T3 = 256;
constexpr int NB = 32;  // panel width
constexpr int TM = 64;  // output tile
constexpr int KC = 16;  // k chunk staged in shared memory

// acc(4x4 per thread) = sum_l A(i0 + i, l) B(l, j0 + j), l in [0, K); 256
// threads, thread (tx, ty) owns rows ty + 16u, columns tx + 16v
template <class FA, class FB>
__device__ void tile_mm(double (&acc)[4][4], FA A, FB B, int i0, int j0, int K, int mrows, int ncols,
                        double (*As)[TM + 1], double (*Bs)[TM + 1]) {
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
  for (int l0 = 0; l0 < K; l0 += KC) {
    __syncthreads();
    for (int e = tid; e < KC * TM; e += T3) {
      const int i = e % TM, l = e / TM;
      As[l][i] = (l0 + l < K && i0 + i < mrows) ? A(i0 + i, l0 + l) : 0.0;
      Bs[l][i] = (l0 + l < K && j0 + i < ncols) ? B(l0 + l, j0 + i) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int l = 0; l < KC; ++l) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = As[l][ty + 16 * u];
#pragma unroll
      for (int v = 0; v < 4; ++v) b[v] = Bs[l][tx + 16 * v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
  }
}

// all 64x64 tiles of an M x N product C = A B (K terms); epi(i, j, c) per
// entry inside [0, M) x [0, N)
template <class FA, class FB, class FE>
__device__ void cta_gemm(int M, int N, int K, FA A, FB B, FE epi, double (*As)[TM + 1], double (*Bs)[TM + 1]) {
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  for (int i0 = 0; i0 < M; i0 += TM)
    for (int j0 = 0; j0 < N; j0 += TM) {
      double acc[4][4];
      tile_mm(acc, A, B, i0, j0, K, M, N, As, Bs);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int i = i0 + ty + 16 * u, j = j0 + tx + 16 * v;
          if (i < M && j < N) epi(i, j, acc[u][v]);
        }
    }
  __syncthreads();
}

// Blocked in-place inverse of the lower triangle L = F[0:s, 0:s] (ld = nf):
// column blocks right to left; W_jj = inv(L_jj) unblocked, then
// W[je:, jb:je] = -(W[je:, je:] L[je:, jb:je]) W_jj as two tiled products
// (tmp: (s - je) x NB doubles, column-major, ld = s; sc: NB doubles)
__device__ void trtri_blocked(double* F, int nf, int s, double* tmp, double* sc, double (*As)[TM + 1],
                              double (*Bs)[TM + 1]) {
  const int nblk = (s + NB - 1) / NB;
  for (int b = nblk - 1; b >= 0; --b) {
    const int jb = b * NB, je = min(s, jb + NB), nb = je - jb;
    double* D = F + at(nf, jb, jb);  // the diagonal block, ld = nf
    trtri_lower<T3>(D, nf, nb, sc);
    const int R = s - je;
    if (R == 0) continue;
    // tmp(i, c) = sum_{t <= i} W(je + i, je + t) L(je + t, jb + c)
    cta_gemm(
        R, nb, R, [&](int i, int t) { return t <= i ? F[at(nf, je + i, je + t)] : 0.0; },
        [&](int t, int c) { return F[at(nf, je + t, jb + c)]; },
        [&](int i, int c, double v) { tmp[(int64_t)c * s + i] = v; }, As, Bs);
    // W(je + i, jb + c) = -sum_{k >= c} tmp(i, k) W_jj(k, c)
    cta_gemm(
        R, nb, nb, [&](int i, int k) { return tmp[(int64_t)k * s + i]; },
        [&](int k, int c) { return k >= c ? D[at(nf, k, c)] : 0.0; },
        [&](int i, int c, double v) { F[at(nf, je + i, jb + c)] = -v; }, As, Bs);
  }
}

__global__ void __launch_bounds__(T3) k_front_global(const FItem* __restrict__ items, const int32_t* __restrict__ list,
                                                     const FChild* __restrict__ ch, const int32_t* __restrict__ rel,
                                                     const FAent* __restrict__ ae, double* __restrict__ vals,
                                                     double* __restrict__ upd, double* __restrict__ work, int* err) {
  __shared__ double As[KC][TM + 1], Bs[KC][TM + 1];
  const FItem it = items[list[blockIdx.x]];
  const int s = it.s, m = it.m, nf = s + m;
  double* F = work + it.front_off;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  assemble<T3>(F, nf, it, ch, rel, ae, upd);
  // blocked partial Cholesky over the s pivot columns
  for (int kb = 0; kb < s; kb += NB) {
    const int ke = min(s, kb + NB);
    chol_cols<T3>(F, nf, kb, ke, ke, err);  // the panel (all rows, panel columns)
    // trailing update F[i][j] -= sum_{l in panel} F[i][l] F[j][l], ke <= j <= i < nf
    const int r0 = ke, nr = nf - ke;
    const int nt = (nr + TM - 1) / TM;
    for (int tj = 0; tj < nt; ++tj)
      for (int ti = tj; ti < nt; ++ti) {
        const int i0 = r0 + ti * TM, j0 = r0 + tj * TM;
        double acc[4][4];
        tile_mm(
            acc, [&](int i, int l) { return F[at(nf, i, kb + l)]; },
            [&](int l, int j) { return F[at(nf, j, kb + l)]; }, i0, j0, ke - kb, nf, nf, As, Bs);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int i = i0 + ty + 16 * u, j = j0 + tx + 16 * v;
            if (i < nf && j < nf && i >= j) F[at(nf, i, j)] -= acc[u][v];
          }
      }
    __syncthreads();
  }
  // W = L11^{-1} in place, blocked (scratch after the front: NB doubles,
  // then an s x NB panel)
  trtri_blocked(F, nf, s, F + (int64_t)nf * nf + NB, F + (int64_t)nf * nf, As, Bs);
  double* M = vals + it.val_off;
  // M_top
  for (int64_t e = tid; e < (int64_t)s * s; e += T3) {
    const int k = (int)(e / s), i = (int)(e % s);
    if (i >= k) M[packed_col_off(s, m, k) + (i - k)] = F[at(nf, i, k)];
  }
  // M_bot = L21 W (m x s, W lower): tiled
  if (m > 0) {
    const int ntr = (m + TM - 1) / TM, ntc = (s + TM - 1) / TM;
    for (int tr = 0; tr < ntr; ++tr)
      for (int tc = 0; tc < ntc; ++tc) {
        const int i0 = tr * TM, j0 = tc * TM;
        double acc[4][4];
        tile_mm(
            acc, [&](int a, int t) { return F[at(nf, s + a, t)]; },
            [&](int t, int k) { return t >= k ? F[at(nf, t, k)] : 0.0; }, i0, j0, s, m, s, As, Bs);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int a = i0 + ty + 16 * u, k = j0 + tx + 16 * v;
            if (a < m && k < s) M[packed_col_off(s, m, k) + (s - k) + a] = acc[u][v];
          }
      }
  }
  // update matrix for the parent
  if (it.upd_off >= 0) {
    double* U = upd + it.upd_off;
    for (int b = tid >> 5; b < m; b += T3 / 32)
      for (int a = b + (tid & 31); a < m; a += 32) U[packed_col_off(m, 0, b) + (a - b)] = F[at(nf, s + a, s + b)];
  }
}

template <class V>
V* upload(const std::vector<V>& h, cudaStream_t st, std::vector<void*>& owned) {
  V* d = nullptr;
  CUDA_CHECK(cudaMallocAsync(&d, std::max<size_t>(h.size() * sizeof(V), 16), st));
  if (!h.empty()) CUDA_CHECK(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(V), cudaMemcpyHostToDevice, st));
  owned.push_back(d);
  return d;
}

}  // namespace

void gpu_factor_prepare(const HostFactor& F, const CsrMatrix& A, GpuFactorInput& out) {
  const int64_t n = F.n;
  out.n = n;
  out.aent_ptr.assign(F.sn.size() + 1, 0);
  out.aent.clear();
  std::vector<int32_t> iperm(n), pos(n, -1);
  for (int64_t k = 0; k < n; ++k) iperm[F.perm[k]] = (int32_t)k;
  for (size_t k = 0; k < F.sn.size(); ++k) {
    const Supernode& S = F.sn[k];
    const int64_t s = S.s, m = S.m, nf = s + m;
    for (int64_t t = 0; t < s; ++t) pos[S.col0 + t] = (int32_t)t;
    for (int64_t a = 0; a < m; ++a) pos[F.rows[S.rows_off + a]] = (int32_t)(s + a);
    for (int64_t t = 0; t < s; ++t) {
      const int64_t c = S.col0 + t;
      const int32_t o = F.perm[c];
      for (int64_t p = A.indptr[o]; p < A.indptr[o + 1]; ++p) {
        const int32_t r = iperm[A.indices[p]];
        if (r < c) continue;
        const int32_t ps = pos[r];
        SFCDD_REQUIRE(ps >= 0, SFCDD_EINTERNAL, "matrix entry outside front");
        SFCDD_REQUIRE(nf * nf < (int64_t(1) << 31), SFCDD_EINTERNAL, "front too large");
        out.aent.push_back(FAent{(int32_t)(t * nf + ps), 0, A.data[p]});
      }
    }
    for (int64_t t = 0; t < s; ++t) pos[S.col0 + t] = -1;
    for (int64_t a = 0; a < m; ++a) pos[F.rows[S.rows_off + a]] = -1;
    out.aent_ptr[k + 1] = (int64_t)out.aent.size();
  }
}

int64_t gpu_factor_work_bound(const HostFactor& F) {
  int64_t w = 0;
  for (const Supernode& S : F.sn) {
    const int64_t nf = S.s + S.m;
    if (nf > 96) w += nf * nf + (int64_t)(NB + 1) * nf;
  }
  return w;
}

int64_t gpu_factor_update_doubles(const HostFactor& F) {
  int64_t u = 0;
  for (const Supernode& S : F.sn)
    if (S.parent >= 0) u += (int64_t)S.m * (S.m + 1) / 2;
  return u;
}

void gpu_factor_batch(const std::vector<const HostFactor*>& fs, const std::vector<const GpuFactorInput*>& in,
                      double* vals_dev, const std::vector<int64_t>& val_base, cudaStream_t st, double* seconds) {
  std::vector<void*> owned;
  auto free_all = [&]() {
    for (void* p : owned) cudaFreeAsync(p, st);
    owned.clear();
  };
  try {
    // item / child / rel / entry tables of the whole batch
    std::vector<FItem> items;
    std::vector<FChild> childs;
    std::vector<int32_t> rel;
    std::vector<FAent> aent;
    std::vector<int32_t> level;
    std::vector<int32_t> nfv;
    int64_t upd_tot = 0;
    int32_t maxlev = 0;
    for (size_t f = 0; f < fs.size(); ++f) {
      const HostFactor& F = *fs[f];
      const GpuFactorInput& G = *in[f];
      const int64_t ibase = (int64_t)items.size();
      const int64_t rbase = (int64_t)rel.size();
      const int64_t abase = (int64_t)aent.size();
      rel.insert(rel.end(), F.rel.begin(), F.rel.end());
      aent.insert(aent.end(), G.aent.begin(), G.aent.end());
      for (size_t k = 0; k < F.sn.size(); ++k) {
        const Supernode& S = F.sn[k];
        FItem it{};
        it.val_off = val_base[f] + S.val_off;
        if (S.parent >= 0) {
          it.upd_off = upd_tot;
          upd_tot += (int64_t)S.m * (S.m + 1) / 2;
        } else {
          it.upd_off = -1;
        }
        it.a_off = abase + G.aent_ptr[k];
        it.a_cnt = (int32_t)(G.aent_ptr[k + 1] - G.aent_ptr[k]);
        it.c_off = (int32_t)childs.size();
        it.c_cnt = F.child_ptr[k + 1] - F.child_ptr[k];
        it.s = S.s;
        it.m = S.m;
        for (int32_t q = F.child_ptr[k]; q < F.child_ptr[k + 1]; ++q) {
          const int32_t c = F.child_list[q];
          FChild C{};
          C.upd_off = items[ibase + c].upd_off;  // children precede parents (postorder)
          C.rel_off = rbase + F.sn[c].rel_off;
          C.m = F.sn[c].m;
          childs.push_back(C);
        }
        items.push_back(it);
        level.push_back(S.level);
        nfv.push_back(S.s + S.m);
        maxlev = std::max(maxlev, S.level);
      }
    }
    // per level: item lists of the three tiers, tier-3 workspace offsets
    std::vector<std::vector<int32_t>> l1(maxlev + 1), l2(maxlev + 1), l3(maxlev + 1);
    std::vector<int64_t> ws(maxlev + 1, 0);
    for (size_t i = 0; i < items.size(); ++i) {
      const int lv = level[i], nf = nfv[i];
      if (nf <= 32) {
        l1[lv].push_back((int32_t)i);
      } else if (nf <= 96) {
        l2[lv].push_back((int32_t)i);
      } else {
        items[i].front_off = ws[lv];
        ws[lv] += (int64_t)nf * nf + (int64_t)(NB + 1) * nf;
        l3[lv].push_back((int32_t)i);
      }
    }
    const int64_t ws_max = *std::max_element(ws.begin(), ws.end());
    cudaEvent_t e0, e1;
    CUDA_CHECK(cudaEventCreate(&e0));
    CUDA_CHECK(cudaEventCreate(&e1));
    CUDA_CHECK(cudaEventRecord(e0, st));
    FItem* d_items = upload(items, st, owned);
    FChild* d_ch = upload(childs, st, owned);
    int32_t* d_rel = upload(rel, st, owned);
    FAent* d_ae = upload(aent, st, owned);
    double* d_upd = nullptr;
    double* d_work = nullptr;
    int* d_err = nullptr;
    CUDA_CHECK(cudaMallocAsync(&d_upd, std::max<int64_t>(upd_tot, 2) * 8, st));
    owned.push_back(d_upd);
    CUDA_CHECK(cudaMallocAsync(&d_work, std::max<int64_t>(ws_max, 2) * 8, st));
    owned.push_back(d_work);
    CUDA_CHECK(cudaMallocAsync(&d_err, 4, st));
    owned.push_back(d_err);
    CUDA_CHECK(cudaMemsetAsync(d_err, 0, 4, st));
    std::vector<int32_t> lists;
    std::vector<int64_t> loff;
    for (int lv = 0; lv <= maxlev; ++lv)
      for (auto* L : {&l1[lv], &l2[lv], &l3[lv]}) {
        loff.push_back((int64_t)lists.size());
        lists.insert(lists.end(), L->begin(), L->end());
      }
    loff.push_back((int64_t)lists.size());
    int32_t* d_lists = upload(lists, st, owned);
    const int smem1 = (32 * 32 + 32) * 8, smem2 = (96 * 96 + 96) * 8;
    CUDA_CHECK(cudaFuncSetAttribute(k_front_smem<128, 96>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
    // SFCDD_FACTOR_DEBUG: device time per tier (events around every launch)
    const bool dbg = std::getenv("SFCDD_FACTOR_DEBUG") != nullptr;
    double tier_ms[3] = {0, 0, 0};
    int64_t tier_n[3] = {0, 0, 0};
    cudaEvent_t ta, tb;
    if (dbg) {
      CUDA_CHECK(cudaEventCreate(&ta));
      CUDA_CHECK(cudaEventCreate(&tb));
    }
    auto timed = [&](int tier, int64_t cnt, auto&& launch) {
      if (cnt <= 0) return;
      if (!dbg) {
        launch();
        return;
      }
      CUDA_CHECK(cudaEventRecord(ta, st));
      launch();
      CUDA_CHECK(cudaEventRecord(tb, st));
      CUDA_CHECK(cudaEventSynchronize(tb));
      float t = 0.f;
      CUDA_CHECK(cudaEventElapsedTime(&t, ta, tb));
      tier_ms[tier] += t;
      tier_n[tier] += cnt;
    };
    for (int lv = 0; lv <= maxlev; ++lv) {
      const int64_t* o = &loff[3 * lv];
      timed(0, o[1] - o[0], [&]() {
        k_front_smem<32, 32><<<(unsigned)(o[1] - o[0]), 32, smem1, st>>>(d_items, d_lists + o[0], d_ch, d_rel, d_ae,
                                                                         vals_dev, d_upd, d_err);
      });
      timed(1, o[2] - o[1], [&]() {
        k_front_smem<128, 96><<<(unsigned)(o[2] - o[1]), 128, smem2, st>>>(d_items, d_lists + o[1], d_ch, d_rel,
                                                                           d_ae, vals_dev, d_upd, d_err);
      });
      timed(2, o[3] - o[2], [&]() {
        k_front_global<<<(unsigned)(o[3] - o[2]), T3, 0, st>>>(d_items, d_lists + o[2], d_ch, d_rel, d_ae, vals_dev,
                                                               d_upd, d_work, d_err);
      });
      CUDA_CHECK(cudaGetLastError());
    }
    if (dbg) {
      std::fprintf(stderr, "[factor] batch of %zu blocks, %d levels: tier1 %lld fronts %.1f ms, tier2 %lld %.1f ms, "
                   "tier3 %lld %.1f ms\n", fs.size(), maxlev + 1, (long long)tier_n[0], tier_ms[0],
                   (long long)tier_n[1], tier_ms[1], (long long)tier_n[2], tier_ms[2]);
      cudaEventDestroy(ta);
      cudaEventDestroy(tb);
    }
    int herr = 0;
    CUDA_CHECK(cudaMemcpyAsync(&herr, d_err, 4, cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaEventRecord(e1, st));
    free_all();
    CUDA_CHECK(cudaStreamSynchronize(st));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (seconds) *seconds += 1e-3 * ms;
    if (herr) throw Error(SFCDD_EFACTOR, "nonpositive pivot, matrix is not SPD");
  } catch (...) {
    free_all();
    throw;
  }
}

}  // namespace sfcdd
