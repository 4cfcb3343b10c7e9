// Device execution plan for a batch of block-inverse factors: the factor
// trees are cut into fragments (connected subtrees whose factor bytes and
// metadata fit one shared-memory blob, or a single big supernode streamed
// from HBM in chunks), and each fragment becomes one forward and one
// backward task of the dataflow kernel in dag_solve.cu.
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

// One DAG task (forward or backward sweep of one fragment).  The queue holds
// the 2 nfrag tasks in decreasing critical-path rank (longest weighted path
// to the end of the solve), which is a topological order: every task waits
// only on tasks earlier in the queue.
struct TaskDev {
  int64_t blob_off;    // byte offset of the fragment blob
  int32_t copy_bytes;  // bytes bulk-copied into shared memory (0 for big)
  int32_t frag;        // fragment id
  int32_t factor;      // factor id
  int32_t wait_on;     // forward: #child fragments; backward: fragment to wait on (-1 = own fwd)
  int32_t signal;      // forward: parent fragment (-1 none)
  int32_t flags;       // TASK_BIG | TASK_BWD
};
constexpr int32_t TASK_BIG = 1;  // single supernode, values streamed from HBM in chunks
constexpr int32_t TASK_BWD = 2;  // backward sweep

// Blob = [int32 meta | pad16 | fp64 packed M blocks].
//
// SMALL fragment (whole blob copied to shared memory).  Supernodes are
// numbered in level order (level 0 = fragment leaves).  Shared scratch
// (doubles):  [frontal slots (s+m each)] [column values (sum s)]
//             [ext_x staging] [ext_u staging]
// Frontal slot of J: f = [b_J + child updates ; f_B] (forward) or
// v = [y_J ; -x_B] (backward).  Column values receive y_J (forward) or
// x_J (backward).  Per level l the meta holds
//   * gather runs (forward assembly, gather form, fixed child order):
//     pairs (dst | src << 16) sorted by dst; run r = pairs [run[r], run[r+1])
//     all with the same dst: S[dst] += sum S[src];
//   * backward row pairs: S[dst] = -S[src]  (dst = v_B slot, src = x slot);
//   * forward / backward warp items (int2) {x, y}:
//     x < 65536: row block y (forward) / column y (backward) of supernode x;
//     x = j | cnt << 16: cnt consecutive small supernodes j.. packed into the
//     32 lanes, y = bit mask of the lanes where each one starts (+ end lane).
//
// BIG fragment (one supernode): meta read from global, values streamed in
// column chunks; rows hold range offsets (ro) and child records reference
// global update slots.
enum BlobHdr {
  H_NSN = 0,
  H_NLEV,
  H_SCRATCH,   // doubles of scratch used
  H_VAL_OFF,   // byte offset of the value area within the blob
  H_TOP,       // local id of the fragment's top supernode
  H_TOP_UPD,   // global update slot of the top supernode (-1 none)
  H_NCOL,      // number of fragment columns
  H_COLS,      // int offset: ro[ncol]
  H_COLPOS,    // int offset: (fpos | cpos << 16)[ncol]
  H_NEXTX,     // number of external rows (staged contiguously from H_EXTX_BASE)
  H_EXTX,      // int offset of their ro[nextx]
  H_NEXTU,     // number of staged external update doubles (contiguous from H_EXTU_BASE)
  H_EXTU,      // int offset of their global update indices [nextu]
  H_BIG,       // 1 = big fragment
  H_REC,       // int offset of SnRec[nsn] (level order)
  H_LEVELS,    // int offset of the per-level table (L_WORDS per level)
  H_RUNS,      // int offset of gather run starts (int32, absolute pair index)
  H_GPAIRS,    // int offset of forward gather pairs (uint32)
  H_BPAIRS,    // int offset of backward row pairs (uint32)
  H_ITEMS,     // int offset of items (int2)
  H_EXTX_BASE, // scratch position of the first ext_x slot
  H_EXTU_BASE, // scratch position of the first ext_u slot
  H_WORDS = 22
};
// per-level table: [rec0, rec1, run0, run1, bpair0, bpair1,
//   fwarp[NWARP_PLAN+1], bwarp[NWARP_PLAN+1]]  -- the level's forward /
// backward items are pre-assigned to the compute warps (longest-processing-
// time first by an item cost model): warp w runs items [fwarp[w], fwarp[w+1]).
constexpr int NWARP_PLAN = 8;
enum LevField { L_REC0 = 0, L_REC1, L_RUN0, L_RUN1, L_BP0, L_BP1, L_FW, L_BW = L_FW + NWARP_PLAN + 1,
                L_WORDS = L_BW + NWARP_PLAN + 1 };
// per-supernode record (int32 words).  Small: S, M, VAL, SCR, CPOS used.
// Big: S, M, VAL, ROWS (ro of the m rows), NCH, CH (child records).
enum SnRecField { R_S = 0, R_M, R_VAL, R_SCR, R_ROWS, R_NCH, R_CH, R_CPOS, R_WORDS };
// big-fragment child record: {global update slot, m, rel int offset}
constexpr int CH_WORDS = 3;
constexpr int SMALL_MAX_S = 128;  // supernodes wider than this are "big"

struct PlanOptions {
  int32_t blob_max = 46 * 1024;     // bytes per small fragment (meta + values)
  int32_t scratch_max = 2048;       // doubles of shared scratch per fragment (< 65536)
  int32_t big_front_max = 1950;     // s+m limit of a streamed big supernode (DagSolver::big_front_max)
};

struct DevicePlan {
  std::vector<uint8_t> blobs;
  std::vector<TaskDev> tasks;  // 2 * nfrag
  std::vector<FactorDev> factors;
  int32_t nfrag = 0;
  int32_t nbig = 0;
  int64_t upd_doubles = 0;
  int64_t xy_doubles = 0;
  int64_t num_supernodes = 0;
  int64_t stored = 0, nnz_l = 0;
  int32_t max_scratch = 0;  // doubles
  int32_t max_copy = 0;     // bytes
  int32_t blob_max = 0;
};

DevicePlan build_plan(const std::vector<const HostFactor*>& factors, const std::vector<int64_t>& gstart,
                      const std::vector<int64_t>& gmod, const PlanOptions& opt);

}  // namespace sfcdd
