// Device execution plan for a batch of block-inverse factors: the factor
// trees are cut into fragments (connected subtrees whose factor bytes and
// metadata fit one shared-memory blob, or a single big supernode streamed
// from HBM), and each fragment becomes one forward and one backward task of
// the dataflow kernel in dag_solve.cu.
#pragma once
#include <cstdint>
#include <vector>

#include "host.h"

namespace sfcdd {

// per-factor addressing of the global vectors
struct FactorDev {
  int64_t gstart;  // gather source: rhs[(gstart + ro) mod gmod]
  int64_t gmod;
  int64_t xy_off;  // work vector xy[xy_off + ro]
  int64_t n;
};

// one DAG task; tasks [0, nfrag) are forward sweeps (bottom-up order),
// tasks [nfrag, 2 nfrag) backward sweeps (top-down order)
struct TaskDev {
  int64_t blob_off;    // byte offset of the fragment blob
  int32_t copy_bytes;  // bytes bulk-copied into shared memory
  int32_t frag;        // fragment id
  int32_t factor;      // factor id
  int32_t wait_on;     // forward: #child fragments; backward: fragment to wait on (-1 = own fwd)
  int32_t signal;      // forward: parent fragment (-1 none)
  int32_t big;         // 1 = single supernode, values streamed from global
};

// blob header (int32 words)
enum BlobHdr {
  H_NSN = 0,
  H_NLEV,
  H_SCRATCH,   // doubles of frontal scratch
  H_VAL_OFF,   // byte offset of the value area within the blob
  H_TOP,       // local id of the fragment's top supernode
  H_TOP_UPD,   // global update slot of the top supernode (-1 none)
  H_LEV_PTR,   // int offset of lev_ptr[nlev+1]
  H_LEV_LIST,  // int offset of level-ordered local ids [nsn]
  H_REC,       // int offset of SnRec[nsn]
  H_WORDS = 12
};
// per-supernode record (int32 words)
enum SnRecField { R_S = 0, R_M, R_VAL, R_SCR, R_IDX, R_NCH, R_CH, R_PARENT, R_WORDS };
// child record: {loc (>=0 local id, -1 external), m, rel int offset, upd slot}
constexpr int CH_WORDS = 4;

struct PlanOptions {
  int32_t blob_max = 64 * 1024;     // bytes per small fragment (meta + values)
  int32_t scratch_max = 2048;       // doubles of frontal scratch per fragment
  int32_t big_meta_max = 48 * 1024; // meta bytes of a big supernode (must fit)
};

struct DevicePlan {
  std::vector<uint8_t> blobs;
  std::vector<TaskDev> tasks;    // 2 * nfrag
  std::vector<FactorDev> factors;
  int32_t nfrag = 0;
  int64_t upd_doubles = 0;
  int64_t xy_doubles = 0;
  int64_t num_supernodes = 0;
  int64_t stored = 0, nnz_l = 0;
  int32_t max_scratch = 0;  // doubles
  int32_t max_copy = 0;     // bytes
};

// factors[i] with gather start/modulus gstart[i], gmod[i]
DevicePlan build_plan(const std::vector<const HostFactor*>& factors, const std::vector<int64_t>& gstart,
                      const std::vector<int64_t>& gmod, const PlanOptions& opt);

}  // namespace sfcdd
