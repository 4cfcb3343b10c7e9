// The Schwarz operator handle (sfcdd_op) and its device kernels.
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <mutex>
#include <vector>

#include "common.h"
#include "dag_solve.h"
#include "host.h"
#include "sfc.h"

namespace sfcdd {

struct ShardRuntime;
void destroy_shard_runtime(ShardRuntime* r);

constexpr int VEC_THREADS = 256;
constexpr int CHUNK = 2048;
constexpr int COARSE_DENSE_MAX = 8192;  // coarse DOFs up to which A0^{-1} is held dense (GEMV solve)  // points per reduction chunk (never crosses an aggregate)

struct Stencil {
  int d;
  int64_t n;
  double dhat;
  double off[MAX_GRID_DIM];
  const int32_t* nbr;  // [2d][n] SFC rank of the -/+ neighbour per axis, -1 outside
};

// device-resident solver state (PCG scalars, reduction tickets, counters)
struct DevState {
  double tol, hist0, rz, beta, pap, alpha;
  int32_t k, converged, breakdown, exhausted, have_rz, max_iters, done, stop_pending;
  uint32_t ticket[8];
  long long apply_calls;
  long long fault_index;
  double ehist0;         // energy error at k = 0 (energy tracking)
  int32_t track_energy;  // an exact solution was given: record energy errors
  int32_t energy_mode;   // the energy error decides convergence (else ||r||)
};

// index-free stencil tiles (tiles.h), device copy
struct Tiles {
  int d;
  int32_t ntiles;
  const int32_t* r0;        // ntiles + 1
  const int32_t* dims;      // 3 per tile
  const int32_t* tab_off;   // ntiles
  const uint16_t* tab;
  const int32_t* halo_off;  // ntiles + 1
  const int32_t* halo;
  const int32_t* slot0;     // ntiles + 1: first R0 Â w partial slot of each tile (one per aggregate met)
  const int32_t* sptr;      // n0 + 1: slots of each aggregate (contiguous, tile order)
  int32_t max_points;       // points of the largest tile (box area in shared memory)
  int32_t smem_doubles;     // box + halo doubles of the largest tile
};
constexpr int TILE_MAX_SEGS = 4;  // aggregates one tile may meet for the tiled R0 Â w

struct Chunks {
  const int64_t* start;       // nch + 1
  const int32_t* agg;         // aggregate of each chunk (or -1)
  const int32_t* agg_ptr;     // first chunk of each aggregate (n0 + 1)
  int32_t nch;
};

}  // namespace sfcdd

struct sfcdd_op {
  int device = 0;
  int d = 0;
  int32_t levels[8] = {0};
  int64_t n = 0;
  int32_t p = 0, q = 0, variant = 3, weighting = 1, threads = 0;
  int32_t shard_first = 0, shard_count = 0;  // shard mode (multi-GPU): owned subdomains
  int32_t curve = 0;                         // SFC: 0 Hilbert, 1 Lebesgue
  int32_t raw = 0;                           // 1: unscaled A (grid.py:91-114), 0: Â = T A T
  int64_t own_g0 = 0, own_g1 = 0;            // owned SFC segment [own_g0, own_g1)
  std::vector<int64_t> xy_off_host;          // per subdomain slot in the xy buffer (-1 none)
  int32_t n0 = 0;
  std::vector<int64_t> ov_start, ov_len, dj_start, dj_len, agg_start;
  std::vector<double> omega;
  double dhat = 0, off[16] = {0}, tscale = 0;
  bool ready = false;
  // device
  int32_t* nbr = nullptr;
  int32_t* agg = nullptr;
  int64_t* chunk_start = nullptr;
  int32_t* chunk_agg = nullptr;
  int32_t* agg_ptr = nullptr;
  int32_t nch = 0;
  double* ainv = nullptr;
  int64_t* d_ov_start = nullptr;
  int64_t* d_ov_len = nullptr;
  int64_t* d_xy_off = nullptr;
  int64_t* d_dj_start = nullptr;  // p + 1
  int32_t* cand_ptr = nullptr;
  int32_t* cand = nullptr;
  bool tiled = false;             // stencils run on SFC tiles (2-D / 3-D, single GPU)
  bool tile_agg = false;          // ... including R0 Â w (every tile meets <= TILE_MAX_SEGS aggregates)
  sfcdd::Tiles tiles{};
  double* part_t = nullptr;       // per-tile partials (p.Ap; R0 Â w slots)
  double* cvec = nullptr;         // n0: R0 Â w summed per aggregate
  int64_t* d_agg_start = nullptr; // n0 + 1 (tiled R0 Â w)
  int32_t* ccand_ptr = nullptr;  // per reduction chunk (nch + 1)
  int32_t* ccand = nullptr;
  double* d_wgt = nullptr;     // per subdomain weight (omega / 1)
  int32_t* d_count = nullptr;  // per point cover count (d_matrix weighting)
  int8_t* d_fault = nullptr;   // per subdomain fault mask
  sfcdd::DevState* st = nullptr;
  double* hist = nullptr;
  int32_t hist_cap = 0;
  double *t = nullptr, *w = nullptr, *y0 = nullptr, *y0b = nullptr;
  double *part_a = nullptr, *part_b = nullptr, *part_c = nullptr;
  double *r = nullptr, *z = nullptr, *p0 = nullptr, *p1 = nullptr, *ap = nullptr;
  double *aex = nullptr, *part_e = nullptr, *ehist = nullptr;  // energy tracking (A x*, partials, history)
  const double* pcg_b = nullptr;                                // b / x* the captured graph reads
  const double* pcg_exact = nullptr;
  std::unique_ptr<sfcdd::DagSolver> dag;
  sfcdd::CsrMatrix a0;           // host copy of A0 (diagnostics)
  std::unique_ptr<sfcdd::DagSolver> coarse_dag;  // sparse A0 factor (n0 > COARSE_DENSE_MAX)
  double* cvec0 = nullptr;       // n0: coarse right-hand side of the sparse path
  sfcdd_stats stats{};
  int64_t dev_bytes = 0;
  cudaStream_t own_stream = nullptr;
  cudaGraphExec_t pcg_graph = nullptr;
  cudaStream_t pcg_graph_stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // re-entrancy (test_schwarz.py:208-222, linalg.py:7-8): every call that
  // touches the handle's scratch runs on own_stream, entered and left through
  // events on the caller's stream, with the host-side enqueue under `mu`; two
  // threads applying one operator therefore serialize on the device
  std::mutex mu;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  sfcdd::ShardRuntime* srt = nullptr;  // device-driven sharded PCG (NCCL), shard mode only
};

namespace sfcdd {
class OpScope {
 public:
  OpScope(sfcdd_op* op, cudaStream_t caller);
  ~OpScope() noexcept(false);
  cudaStream_t stream() const { return op_->own_stream; }

 private:
  sfcdd_op* op_;
  cudaStream_t caller_;
  std::unique_lock<std::mutex> lk_;
};
}  // namespace sfcdd
