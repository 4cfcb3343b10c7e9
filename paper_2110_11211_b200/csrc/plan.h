// Device execution plan for a batch of block-inverse factors (v4, warp
// tasks).  Every task is executed by ONE warp out of a per-warp shared-memory
// slot (blob area + scratch area); a task's blob (int32 metadata + fp64 factor
// values) is moved HBM -> slot by one cp.async.bulk.
//
// Work units ("groups"):
//  * FRAG: a connected subtree of small supernodes, or several sibling
//    subtrees (roots with the same parent supernode) packed together.  One
//    forward task and one backward task share the blob; the warp runs the
//    subtrees level by level entirely in its slot.
//  * BIG: one supernode J too large for a slot.  Forward = ROW tasks (blocks
//    of rows of M = [L_JJ^-1 ; L_BJ L_JJ^-1], each re-assembling f_J from the
//    children's update vectors), backward = COL tasks (blocks of columns of M).
//    y_J travels from the ROW to the COL tasks through a global y slot.
// Dependencies are per-group counters (see TaskDev).
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

enum TaskKind : int32_t {
  TK_FRAG_FWD = 0,
  TK_FRAG_BWD = 1,
  TK_ROW_FWD = 2,
  TK_COL_BWD = 3,
  TK_ASM_FWD = 4,  // BIG forward assembly: f = [f_J ; f_B] once per supernode
  TK_XB_BWD = 5,   // BIG backward gather: -x_B once per supernode
  TK_KINDS = 6
};

// One warp task.  The queue holds all tasks in decreasing critical-path rank
// (HLFET), a topological order: a task only waits on tasks earlier in the
// queue.  Counters (int32, zeroed per solve): ctr[0] = queue head; per group
// g of G: fin = 1+g (forward arrivals of g's children), bdone = 1+G+g
// (g's backward tasks done), rdone = 1+2G+g (a root group's forward done),
// adone = 1+3G+g (BIG: assembly tasks done), xdone = 1+4G+g (BIG: -x_B
// gathered).
constexpr int CTR_PER_GROUP = 5;
struct TaskDev {
  int64_t blob_off;     // byte offset of the task blob (16-byte aligned)
  int32_t copy_bytes;   // bytes bulk-copied into the slot (multiple of 16)
  int32_t kind;         // TaskKind
  int32_t factor;       // factor id
  int32_t group;        // group id (diagnostics)
  int32_t wait_idx;     // counter to wait on (-1: none)
  int32_t wait_target;  // wait until ctr[wait_idx] >= wait_target
  int32_t signal_idx;   // counter incremented on completion
  int32_t values;       // factor values touched (diagnostics)
};

// ---------------------------------------------------------------- FRAG blob
// Blob = [int32 meta | pad16 | fp64 packed M blocks].  Supernodes are
// numbered in level order (level 0 = fragment leaves).  Shared scratch
// (doubles): [frontal slots (s+m each)] [column values (sum s)]
//            [ext_x staging] [ext_u staging]
// Frontal slot of J: f = [b_J + child updates ; f_B] (forward) or
// v = [y_J ; -x_B] (backward).  Column values receive y_J (forward) or x_J
// (backward).  Per level l the meta holds
//   * gather runs (forward assembly, gather form, fixed child order):
//     pairs (dst | src << 16) sorted by dst; run r = pairs [run[r], run[r+1])
//     all with the same dst: S[dst] += sum S[src];
//   * backward row pairs: S[dst] = -S[src]  (dst = v_B slot, src = x slot);
//   * forward / backward warp items (int2) {x, y}:
//     x < 65536: row block y (forward) / column block y = k0 | c << 16
//     (backward) of supernode x;
//     forward x = j | cnt << 16 (| 1 << 31 when the packed supernodes all
//     have s <= 4: straight-line paths): cnt consecutive small supernodes
//     j.. packed into the 32 lanes (lanes = rows), y = bit mask of the lanes
//     where each one starts (+ end lane);
//     backward x = j | cnt << 16: supernodes j..j+cnt-1 (s <= 32) packed in
//     DESCENDING order, lanes = (column, row phase), 2^lp phases (record),
//     segment starts aligned to 2^lp, y = start mask (+ end lane).
enum FragHdr {
  H_NSN = 0,
  H_NLEV,
  H_SCRATCH,    // doubles of scratch used
  H_VAL_OFF,    // byte offset of the value area within the blob
  H_NTOP,       // number of top supernodes (roots of the fragment's subtrees: siblings below one parent)
  H_TOPS,       // int offset of their pairs {local id, global update slot (-1 none)}
  H_NCOL,       // number of fragment columns
  H_COLS,       // int offset: ro[ncol]
  H_COLPOS,     // int offset: (fpos | cpos << 16)[ncol]
  H_NEXTX,      // number of external rows (staged contiguously from H_EXTX_BASE)
  H_EXTX,       // int offset of their ro[nextx]
  H_NEXTU,      // number of staged external update doubles (contiguous from H_EXTU_BASE)
  H_EXTU,       // int offset of their global update indices [nextu]
  H_REC,        // int offset (16-aligned) of the int4 supernode records (level order)
  H_LEVELS,     // int offset of the per-level table (L_WORDS per level)
  H_RUNS,       // int offset of gather run starts (int32, absolute pair index)
  H_GPAIRS,     // int offset of forward gather pairs (uint32)
  H_BPAIRS,     // int offset of backward row pairs (uint32)
  H_ITEMS,      // int offset of items (int2)
  H_EXTX_BASE,  // scratch position of the first ext_x slot
  H_EXTU_BASE,  // scratch position of the first ext_u slot
  H_ZERO,       // doubles zeroed before the forward gather: the frontal slots
                // (their f_B rows accumulate child updates); the rest is written
  H_WORDS
};
// per-level table: record range, forward gather runs, backward row pairs,
// forward items, backward items
enum LevField { L_REC0 = 0, L_REC1, L_RUN0, L_RUN1, L_BP0, L_BP1, L_FI0, L_FI1, L_BI0, L_BI1, L_WORDS };
// per-supernode record: int4 {s | lp << 12 | m << 16, scratch slot, value
// offset, column slot}; lp = log2 of the row phases per column in the
// supernode's backward column-lane item (s < 4096)
enum SnRecField { R_SM = 0, R_SCR, R_VAL, R_CPOS, R_WORDS };

// ---------------------------------------------------------- BIG blobs
// A BIG group is one supernode J too large for a slot.  Its dense block
// M = [L_JJ^-1 ; L_BJ L_JJ^-1] is cut into ROW tasks (forward) and COL tasks
// (backward); the gathers of the sweeps are done ONCE per supernode by
// ASM / XB tasks into contiguous global vectors (update buffer):
//   f  [s+m] at AS_FOFF: f_J = rhs + child updates, f_B = child updates
//   vb [m]   at XB_XOFF: -x_B
// so ROW / COL blobs carry values only (plus the column ids COL stores to).
// The split costs one dependency hop, so it is used in many-factor plans
// (PlanOptions::split_min_factors) and wherever a task could not hold its
// input vector in the slot; otherwise ROW / COL tasks gather for themselves.
//
// ASM blob: front positions [q0, q0+nq) of J: cols (ro of the positions < s),
// ptr[nq+1] / src[nnz] = CSR of the child update indices summed into each
// position (fixed order: children, then rows).
enum AsmHdr { AS_S = 0, AS_Q0, AS_NQ, AS_FOFF, AS_COLS, AS_PTR, AS_SRC, AS_WORDS };
// XB blob: rows [a0, a0+na) of J's m below-rows: vb[a] = -x(rows[a]).
enum XbHdr { XB_A0 = 0, XB_NA, XB_XOFF, XB_ROWS, XB_WORDS };
// ROW blob: forward rows [r0, r0+R) of J (all < s: y rows, or all >= s:
// update rows).  Values: R x C dense column-major (leading dim R), entry
// (i, k) = M[r0+i, k] (zero where k > r0+i), C = min(r0+R, s); they follow
// the metadata in the blob buffer (copied with it: BLOB, or not: DIRECT).  Scratch:
// ASM mode: a two-chunk ring of f_J pieces; inline mode: [f_J[0:C) ;
// f_B[r0 : r0+NB)] assembled by the task.
// MROW task (DIRECT, ASM mode, update rows of a supernode with s <= RING_CHUNK):
// RW_NBLK consecutive blocks of RW_R rows each -- block b holds rows
// [r0 + b R, r0 + (b+1) R) as R x C column-major, C = s, the last block padded
// with zero rows; RW_NB = rows of the whole task.  One contiguous value
// stream per task: the tall, narrow fronts of 3-D subdomains (s ~ 20,
// m ~ 500) become one task instead of m / 32.
enum RowHdr {
  RW_S = 0,
  RW_R,        // rows in the block
  RW_C,        // columns
  RW_R0,       // first front row
  RW_NB,       // block rows >= s (0 or R)
  RW_YOFF,     // global y slot of J (upd buffer)
  RW_UOFF,     // global update slot of J (-1: root)
  RW_FOFF,     // f slot of J (ASM mode), or -1: the task assembles f itself from
  RW_COLS,     //   int offset: ro[C] (rhs gather)
  RW_PTR,      //   int offset: ptr[C+NB+1] / src[nnz]: CSR over the task's front
  RW_SRC,      //   positions (f_J[0:C), then its NB update rows) of child update indices
  RW_ASM16,    // or (huge s): byte offset / 16 of J's global assembly record, low 32 bits
  RW_ASM_HI,   //   ... high bits (-1: no record); record = [s, m] [cols (s)] [ptr (s+m+1)] [src]
               //   over FRONT positions
  RW_VAL_OFF,  // byte offset of the values
  RW_SCRATCH,  // doubles of scratch used
  RW_INBLOB,   // 1: the values follow the metadata in the slot (BLOB block); 0: they stay in HBM (DIRECT)
  RW_NBLK,     // row blocks of the task (1; > 1: MROW task, see below)
  RW_WORDS
};
// COL blob: backward columns [k0, k0+c) of J.  Values: L x c dense row-major
// block of M (L = s+m-k0 rows starting at row k0), entry (r, j) =
// M[k0+r, k0+j] (zero where r < j), streamed from HBM like the ROW values.
// Scratch: XB mode: a two-chunk ring of v pieces; inline mode:
// v = [y_J[k0:s) ; -x_B] (L) gathered by the task.
enum ColHdr {
  CL_S = 0,
  CL_M,
  CL_K0,
  CL_C,        // columns in the block
  CL_YOFF,     // global y slot of J
  CL_XOFF,     // vb slot of J (-x_B, XB mode), or -1: the task gathers -x_B itself
  CL_COLS,     // int offset: ro of the c columns
  CL_ROWS,     // (CL_XOFF < 0) int offset: ro of the m below rows
  CL_VAL_OFF,  // byte offset of the values
  CL_SCRATCH,
  CL_INBLOB,   // 1: values in the slot (BLOB block); 0: in HBM (DIRECT)
  CL_WORDS
};

// Vector ring of the ROW / COL tasks whose input vector is contiguous in the
// update buffer (ASM / XB mode): chunks of RING_CHUNK doubles are bulk-copied
// into two alternating scratch slots of RING_STRIDE doubles (one leading
// double for a misaligned start + padding to 16 bytes), so the scratch need
// does not grow with the separator size (BASELINE C5: s ~ 2300).
constexpr int RING_CHUNK = 256;
constexpr int RING_STRIDE = RING_CHUNK + 2;

constexpr int SMALL_MAX_S = 32;  // wider supernodes are always BIG (a FRAG backward item packs whole supernodes
                                  // into the 32 lanes: dag_solve.cu bwd_lanes)

// ------------------------------------------------ factor value placement
// Where a factor's packed block-inverse values (HostFactor::val layout:
// supernode J's M at val_off, column-major packed trapezoid) land in the
// blob buffer.  One descriptor per FRAG supernode and per ROW / COL task;
// the same descriptors fill the blobs on the host (from HostFactor::val) or
// on the device (from values a device factorization produced), so plans can
// be built before any numeric factorization (PlanOptions::defer_values).
enum ValDescKind : int32_t {
  VD_COPY = 0,  // len consecutive values (a whole packed M block)
  VD_ROW = 1,   // ROW blob: R x C column-major, (i, k) = M[r0 + i, k], k <= r0 + i
  VD_COL = 2,   // COL blob: L x c row-major, (r, j) = M[k0 + r, k0 + j], j <= r
};
struct ValDesc {
  int64_t dst;     // byte offset in the blob buffer
  int64_t src;     // offset of J's packed M in its factor's values (Supernode::val_off)
  int32_t factor;  // factor id within the plan
  int32_t kind;    // ValDescKind
  int32_t s, m;    // supernode shape
  int32_t p0;      // ROW: r0; COL: k0
  int32_t w;       // ROW: R; COL: c
  int32_t len;     // COPY: count; ROW: C; COL: L
  int32_t rows;    // ROW: rows present (<= w; the rest of the block stays zero), 0: w
};
static_assert(sizeof(ValDesc) == 48, "ValDesc layout");
// metadata segment of a deferred-value plan: host bytes [host_off, +bytes)
// go to blob byte offset dev_off
struct MetaSeg {
  int64_t dev_off;
  int64_t host_off;
  int64_t bytes;
};
// host version of the placement (the device kernel follows it exactly)
void place_values(const ValDesc& d, const double* M /* J's packed block */, uint8_t* blob_buffer);

struct PlanOptions {
  int32_t blob_max = 8 * 1024;   // bytes of a task blob (slot blob area): FRAG blobs, BIG metadata
  int32_t scratch_max = 512;     // doubles of FRAG scratch (< 65536)
  int32_t big_scratch_max = 8192;  // doubles of scratch a BIG task may use
  int32_t workers = 0;             // warps assumed by the queue-order simulation (0: from the slot size; SFCDD_WORKERS)
  int32_t sms = 148;               // SMs of the target device (set by the caller)
  int32_t row_max = 128;           // rows per BLOB ROW task (SFCDD_ROW_MAX; latency vs task count), <= 128;
                                   // DIRECT ROW blocks hold <= 32 rows (one lane per row)
  int32_t col_max = 16;            // columns per COL task (SFCDD_COL_MAX), <= 32
  int32_t asm_max = 256;           // front positions per ASM task (SFCDD_ASM_MAX)
  double asm_redundancy = 4.0;     // BLOB supernodes: ASM when the ROW tasks would gather the front >= this often (SFCDD_ASM_RED)
  int32_t xb_min_tasks = 4;        // BLOB supernodes: XB when J has >= this many COL tasks (SFCDD_XB_MIN)
  int32_t direct_min_rows = -1;    // a supernode whose blob would hold fewer full-width rows streams DIRECT ROW blocks
                                   // (SFCDD_DIRECT_ROWS; 0: never, 1 << 20: always; -1: 8 in plans that hold a
                                   // supernode too wide for any BLOB block, else 0 -- measured)
  int32_t direct_min_cols = -1;    // ... fewer full-height columns: DIRECT COL blocks (SFCDD_DIRECT_COLS; -1: 4 / 0)
  int32_t mrow_rows = 0;           // rows per MROW task (<= RING_CHUNK; SFCDD_MROW_ROWS); 0: no MROW tasks, the
                                   // default -- measured slower than the BLOB row blocks they replace (C5 38.8 vs
                                   // 35.0 ms, C3 2.45 vs 2.26 ms: a warp streams ~1.5-3 GB/s)
  int32_t mrow_min_bytes = 32768;  // update rows of fewer value bytes stay ROW blocks (SFCDD_MROW_MIN)
  bool pack_siblings = true;       // FRAG groups may hold several sibling subtrees (SFCDD_PACK=0: one subtree each)
  int32_t pack_max = 64;           // ... at most this many (SFCDD_PACK_MAX)
  int32_t split_min_factors = 256; // ASM / XB only in plans of >= this many factors: with few
                                   // subdomains the top of the trees is latency bound and the
                                   // extra dependency hop costs more than it saves (SFCDD_SPLIT_MIN)
  double slack_us = 4.0;           // queue-order simulation: dependents become ready this late (SFCDD_SLACK_US)
  int32_t wpb = 4;                 // worker warps per DAG CTA: 2, 4 or 8 (SFCDD_WPB)
  int32_t slot_max = 0;            // > 0: ONE byte budget for a task's blob + scratch (the scratch follows the
                                   // task's own blob in the slot); 0: set by choose_blob_shape to the largest
                                   // slot that keeps 5 CTAs per SM; -1: separate blob_max / scratch_max budgets
                                   // (SFCDD_SLOT_MAX)
  bool tuned = false;              // blob_max / wpb fixed by the environment (no automatic choice)
  bool defer_values = false;       // build the plan from symbolic factors: blobs hold metadata only
                                   // (DevicePlan::segs), values are placed later by the descriptors
  int32_t threads = 0;             // host threads for the per-factor blob emission (0: hardware)
  PlanOptions();                 // environment overrides SFCDD_BLOB_MAX, SFCDD_SCRATCH_MAX, ...
};

// Blob size and CTA shape for a set of factors (unless set by the
// environment): plans whose values sit mostly in big supernodes (3-D
// subdomains) use 16 KB blobs with 2-worker CTAs, FRAG-heavy plans (2-D) keep
// 8 KB blobs and 4-worker CTAs (measured).
void choose_blob_shape(const std::vector<const HostFactor*>& factors, PlanOptions& opt);

struct DevicePlan {
  // the blob buffer's host image: every byte (values included), or with
  // `deferred` only the metadata, laid out by `segs`
  std::vector<uint8_t> blobs;
  bool deferred = false;
  int64_t blob_bytes = 0;        // device size of the blob buffer
  std::vector<MetaSeg> segs;     // deferred: metadata placement
  std::vector<ValDesc> vdesc;    // value placement, grouped by factor (ascending)
  std::vector<TaskDev> tasks;
  std::vector<FactorDev> factors;
  int32_t ngroups = 0;
  int32_t nfrag = 0;      // FRAG groups
  int32_t nbig = 0;       // BIG groups
  int64_t upd_doubles = 0;
  int64_t xy_doubles = 0;
  int64_t num_supernodes = 0;
  int64_t stored = 0, nnz_l = 0;
  bool has_direct = false;  // some ROW / COL task streams its values from HBM (selects the kernel variant)
  bool has_mrow = false;    // some ROW task is an MROW task (opt-in, PlanOptions::mrow_rows)
  int32_t wpb = 4;          // worker warps per DAG CTA the plan was simulated for
  int32_t max_scratch = 0;  // doubles, over all tasks
  int64_t slot_need = 0;    // bytes of shared memory a worker needs: max over tasks of align128(blob) + scratch
  int32_t max_copy = 0;     // bytes
  int32_t blob_max = 0;
  double sim_us = 0.0;  // makespan of the simulated schedule (model time)
  int32_t workers = 0;  // warps the schedule was simulated on
  double crit_us = 0.0; // critical path of the task graph (model time)
};

DevicePlan build_plan(const std::vector<const HostFactor*>& factors, const std::vector<int64_t>& gstart,
                      const std::vector<int64_t>& gmod, const PlanOptions& opt);

// host interpreter of the plan (test hook): same blob semantics as the kernel
void plan_exec_host(const DevicePlan& P, const double* rhs, double* xy);

}  // namespace sfcdd
