// program.hpp — the compiled form of an ExecutionGraph that the replay kernel
// walks.  Shared by the host compiler (compile.cpp) and the device code
// (replay.cu).
//
// A graph is split into independent components (weakly connected pieces of
// the dependency graph; in a merged multi-rank replay graph every rank is one,
// because merge_ranks adds no cross-rank edges, build.hpp:113-115).  Each
// component becomes a straight-line *program*: one op per task in a
// topological order, each op reading its predecessors' finish times from
// numbered *slots* and writing its own finish time to a slot.  Slots are
// allocated by liveness, so a scenario's whole replay state fits in a few
// dozen int64 words of shared memory no matter how many tasks the graph has.
//
// The op semantics restate the reference replay on the chained-lane class
// (simulate.cpp:145-337; every build_graph lane is chained, build.cpp:375-386):
//   start(v) = max(W, finish(p) for p in preds(v)),  finish(v) = start(v) + d(v)
// with W = iteration_window.start (simulate.cpp:172).  Stream/DeviceSync rules
// (simulate.cpp:210-216) compile to static predecessor edges plus a per-
// scenario certificate (OP_SYNC + OpExt) that proves the static binding equals
// the reference's first-quiescent-instant rule, see compile.cpp.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define LUMOS_HD __host__ __device__
#else
#define LUMOS_HD
#endif

namespace lumos {

constexpr uint16_t kNoSlot = 0xFFFF;
constexpr int kMaxClasses = 4;
constexpr int kCertPerExt = 4;
// Reserved slots: slot 0 always holds W (the replay origin) and is what unused
// predecessor fields point at, so every op reads exactly four slots with no
// branch on the fan-in; slot 1 is a write-only sink for results nobody reads;
// slot 2 holds +inf, the coverage source of an F_TRACK1 op without one.
constexpr uint16_t kSlotOrigin = 0;
constexpr uint16_t kSlotTrash = 1;
constexpr uint16_t kSlotInf = 2;
constexpr int kFirstSlot = 3;
// Programs are streamed through shared memory in chunks of kChunk records; no
// op group (an op plus its auxiliary records) straddles a chunk boundary.
constexpr int kChunk = 64;
// Each walk thread replays kScenPerThread adjacent scenarios.  The slot table
// is [slot][T] of int64 x kScenPerThread (16 bytes) for a CTA of T threads
// (128, 64 or 32, chosen at launch from the slot count), so slot s of a thread
// lives s * T * 16 bytes past slot 0.  Records store s * kWalkThreads (16-bit,
// up to 511 slots); the kernel shifts by log2(T) - 3 to get the byte offset.
constexpr int kWalkThreads = 128;
constexpr int kScenPerThread = 2;
constexpr int kSlotStride = kWalkThreads * 8 * kScenPerThread;
constexpr int kMaxSlots = 65535 / kWalkThreads;
LUMOS_HD constexpr uint16_t slot_off(int s) {
  return static_cast<uint16_t>(s * kWalkThreads);
}

enum OpKind : uint8_t {
  // kinds 0..3 take start = max(W, preds) (the walk tests kind <= OP_ACC)
  OP_NODE = 0,    // start = max(W, preds); fin = start + d
  OP_SYNC = 1,    // OP_NODE over fixed preds, then static sync edges + certificate
  OP_START = 2,   // start = max(W, preds) -> dst (first half of a collective member)
  OP_ACC = 3,     // dst = max(preds)  (fan-in > 4 folding; no task)
  OP_FINISH = 4,  // start = slot[pred0]; fin = max(start, preds[1..)) + d
  OP_GATED = 5,   // start = max(W, preds[0..nfixed)); fin = max(start, preds[nfixed..)) + d
  OP_NOP = 6,     // padding to a chunk boundary
  // cooperative multi-rank walks (one warp per rank of a component):
  OP_POST = 7,    // mailbox[x1] = slot[pred0], then its ready flag
  OP_WAIT = 8,    // wait for mailbox[x1]'s flag, slot[dst] = mailbox[x1]
};

enum OpFlags : uint8_t {
  F_TRACK = 1,        // followed by an OpCov record: maintain coverage values
  F_STORE_START = 2,  // also store start into slot x2
  F_BUSY = 4,         // kernel on the compute stream of a fused component: the
                      // walk adds finish - start to the rank's busy sum |A|
  F_COMM = 8,         // OpClass::Communication
  F_NO_OUT = 16,      // helper op, produces no SimEntry
  F_TRACK1 = 32,      // compact coverage: cov = pred0 >= start ? min(start, slot x0) : start -> x1
  F_SINK = 64,        // finish read by no other op: candidate for the makespan
  F_RT = 128,         // task carries what-if retime metadata (GEMM, optimizer,
                      // allreduce, p2p send): a retime walk looks its duration up
                      // through CompiledGraph::rt_rec_of
};

// 32-byte op record.  cls: low nibble = scenario class, high nibble = nfixed
// (OP_GATED).  For OP_SYNC, x0 = number of OpExt records that follow; a
// F_TRACK op is followed by exactly one OpCov record; a F_TRACK1 op keeps its
// single coverage source / destination in x0 / x1.
struct alignas(16) Op {
  int64_t base;      // base duration (us)
  int32_t node;      // task id relative to the component's node_base
  uint8_t kind;
  uint8_t npred;
  uint8_t cls;
  uint8_t flags;
  uint16_t pred[4];
  uint16_t dst;      // finish slot (start slot for OP_START, acc for OP_ACC)
  uint16_t x0;
  uint16_t x1;
  uint16_t x2;
};
static_assert(sizeof(Op) == 32, "Op must stay 32 bytes");

// Coverage of a kernel k on a stream watched by a sync with stream set X:
//   cov_X(k) = min(start(k), cov_X(p) for kernel preds p on X-streams with
//                  finish(p) == start(k))
// so [cov_X(k), finish(k)) is covered without a gap by kernels running on
// X-streams.  One OpCov record carries up to two sets per kernel.
constexpr int kCovSets = 2;
struct alignas(16) OpCov {
  uint16_t src[kCovSets][4];  // per pred index: that pred's cov slot, or none
  uint16_t dst[kCovSets];     // this kernel's cov slot per set, or none
  uint16_t n_sets;
  uint16_t pad[5];
};
static_assert(sizeof(OpCov) == 32, "OpCov must stay 32 bytes");

// Certificate entries of one Stream/DeviceSync: per watched stream w,
//   fin  = slot holding finish(k*_w) (last kernel bound before the sync), or none
//   bs   = slot holding cov_X(k*_w) for the sync's watched set X
//   next = slot holding start(n_w) for the chain successor of k*_w when it is
//          not a descendant of the sync, else none.
struct alignas(16) OpExt {
  uint16_t fin[kCertPerExt];
  uint16_t bs[kCertPerExt];
  uint16_t next[kCertPerExt];
  uint16_t n;        // entries used in this record
  uint16_t pad[3];
};
static_assert(sizeof(OpExt) == 32, "OpExt must stay 32 bytes");

// Split breakdown accounting (breakdown_by_rank, metrics.cpp:43-103).  A
// component that is exactly one rank whose GPU streams are at most one
// compute-only stream A and at most three communication-only streams is
// "fused": its breakdown follows from |A|, |U| (U = union of the comm
// intervals) and |A n U|
//   exposed_compute = |A| - |A n U|, exposed_comm = |U| - |A n U|,
//   overlapped = |A n U|, other = window - |A| - |U| + |A n U|.
// The walk sums |A| in a register over the F_BUSY kernels (no extra memory
// traffic).  Intervals of two tasks ordered in the DAG are disjoint (finish <=
// start along every edge), so a compute kernel that is comparable with every
// comm kernel of its rank cannot meet U: the reduction reads the comm
// intervals and only the compute kernels DAG-incomparable with some comm
// kernel (the rank's "candidates", a few percent of A), instead of all of A.
constexpr int kFusedMaxComm = 3;  // comm streams a fused rank may have
struct FusedDesc {
  int32_t row;       // breakdown row (rank index), -1: not fused
  int32_t stream_a;  // stream slot of A, -1 none
};

struct ProgramDesc {
  int64_t op_offset;  // index into the op array (in 32-byte records)
  int32_t n_ops;      // records, including OpExt records
  int32_t n_slots;
};

struct ComponentDesc {
  int32_t program;
  int32_t node_base;  // global task id = node_base + op.node
  int32_t n_tasks;
  int32_t pad;
};

}  // namespace lumos
