// Batched multifrontal numeric Cholesky on the device (gpu_factor.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "host.h"

namespace sfcdd {

// one supernode (front) of a batch
struct FItem {
  int64_t val_off;    // its packed M in the batch value buffer
  int64_t upd_off;    // its packed lower update matrix (m (m+1) / 2), -1: root
  int64_t a_off;      // matrix entries [a_off, a_off + a_cnt)
  int64_t front_off;  // tier 3: front workspace (nf * nf + nf doubles)
  int32_t a_cnt;
  int32_t c_off, c_cnt;  // children (FChild table)
  int32_t s, m;
  int32_t pad;
};
struct FChild {
  int64_t upd_off;  // the child's update matrix
  int64_t rel_off;  // its m positions in the parent front (HostFactor::rel)
  int32_t m;
  int32_t pad;
};
// a matrix entry at column-major front position idx = t * nf + pos
struct FAent {
  int32_t idx;
  int32_t pad;
  double val;
};

// per-block host input: the block's entries scattered to front positions
struct GpuFactorInput {
  int64_t n = 0;
  std::vector<int64_t> aent_ptr;  // per supernode
  std::vector<FAent> aent;
};
void gpu_factor_prepare(const HostFactor& F, const CsrMatrix& A, GpuFactorInput& out);
// device memory the batch needs besides the values: update matrices, and an
// upper bound of the tier-3 front workspace
int64_t gpu_factor_update_doubles(const HostFactor& F);
int64_t gpu_factor_work_bound(const HostFactor& F);
// values of block f -> vals_dev + val_base[f] (HostFactor::val layout);
// throws Error(SFCDD_EFACTOR) for a nonpositive pivot; *seconds += device time
void gpu_factor_batch(const std::vector<const HostFactor*>& fs, const std::vector<const GpuFactorInput*>& in,
                      double* vals_dev, const std::vector<int64_t>& val_base, cudaStream_t st, double* seconds);

}  // namespace sfcdd
