// Device-resident batch of block-inverse factors + the dataflow solve kernel.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "plan.h"

namespace sfcdd {

class DagSolver {
 public:
  // extra_xy: doubles appended to the xy work buffer (shard mode: slots for
  // foreign subdomains' solutions received from other ranks)
  DagSolver(const DevicePlan& plan, int device, int64_t extra_xy = 0);
  ~DagSolver();
  DagSolver(const DagSolver&) = delete;
  DagSolver& operator=(const DagSolver&) = delete;

  // xy[factor i][ro] = A_i^{-1} rhs[(gstart_i + ro) mod gmod_i]
  void solve(const double* rhs, cudaStream_t st, const int32_t* skip = nullptr);
  double* xy() const { return xy_; }
  int64_t xy_doubles() const { return xy_doubles_; }
  int64_t device_bytes() const { return bytes_; }
  int32_t grid() const { return grid_; }
  int32_t ngroups() const { return ngroups_; }
  // diagnostics: per-task timestamps {sm, top, deps ok, data ok, end} (5 x u64 per task)
  void set_trace(unsigned long long* dev_buf);
  int32_t ntask() const { return ntask_; }
  // deferred-value plans: place the packed values of factors [f0, f1) into
  // the blobs; vals_dev + fbase_host[f - f0] = factor f's HostFactor::val
  void place_values(int32_t f0, int32_t f1, const double* vals_dev, const int64_t* fbase_host, cudaStream_t st);

 private:
  int device_;
  int32_t ngroups_ = 0, ntask_ = 0, grid_ = 1, blob_max_ = 0, slot_bytes_ = 0, smem_ = 0, wpb_ = 4, mode_ = 0, sig_ns_ = 20,
          sig_wait_ns_ = 1000;
  bool split_ = false;  // kernel variant with ASM / XB tasks
  bool has_mrow_ = false;  // the plan holds MROW tasks (opt-in): needs the full kernel
  const void* kern_ = nullptr;
  const void* kern_trace_ = nullptr;  // the same kernel with per-task time stamps (sfcdd_op_trace)
  int64_t xy_doubles_ = 0, ctr_words_ = 0, bytes_ = 0;
  int64_t rhs_doubles_ = 0;  // length of the gathered right-hand side (max gmod of the factors)
  int32_t l2_persist_ = 0;   // SFCDD_L2_PERSIST: 1 = rhs, 2 = xy as a persisting L2 window of the launch (experiment)
  int32_t watchdog_ms_ = 20000;  // dependency-wait watchdog (SFCDD_WATCHDOG_MS)
  int32_t pf_dist_ = 0;          // L2 prefetch distance in queue positions (SFCDD_PF_DIST; set per plan in the
                                 // constructor: about one task duration of claims ahead, or 0)
  uint8_t* blobs_ = nullptr;
  TaskDev* tasks_ = nullptr;
  FactorDev* factors_ = nullptr;
  double* upd_ = nullptr;
  double* xy_ = nullptr;
  int32_t* ctr_ = nullptr;
  int32_t* qhead_ = nullptr;
  int32_t nq_ = 16;
  unsigned long long* trace_ = nullptr;
  std::vector<ValDesc> vdesc_;   // deferred plans only
  std::vector<int64_t> vd_ptr_;  // descriptor range per factor

 public:
  std::vector<TaskDev> host_tasks;
};

}  // namespace sfcdd
