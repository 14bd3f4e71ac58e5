// POD structures shared by the host planner (runtime.cpp) and the sm_100a interpreter
// (interp.cu). One launch executes every IR thread block of every rank hosted on one device;
// each IR thread block is replicated over `lanes` CUDA blocks that own disjoint tiles.
//
// Correspondence with the paper's interpreter (Fig. 4):
//   Instruction{step, opCode, srcOff, dstOff, count, srcPtr, dstPtr, depBid[D], depStep[D], hasDep}
//     -> DevOp (+ DevDep list; the buffer "pointers" are buffer ids resolved per rank per call)
//   semaphore[bid]          -> sems[(tb.sem + lane)]  (64-bit, epoch-tagged, .gpu scope)
//   remote buffer slots     -> DevChan.fifo (receiver memory, `slots` x slot_bytes)
#pragma once

#include <cstdint>

namespace gc3 {

constexpr int kMaxLocalRanks = 16;
#ifndef GC3_THREADS
#define GC3_THREADS 512
#endif
constexpr int kThreads = GC3_THREADS;  // CUDA threads per interpreter block

enum : uint8_t { kOpSend = 0, kOpRecv, kOpCopy, kOpReduce, kOpRrc, kOpRcs, kOpRrcs, kOpRrs, kOpNop };
enum : uint8_t { kInDirect = 1, kOutDirect = 2, kInPull = 4, kOutPull = 8,
                 kMsgDep = 16,      // the receive waits its sender's semaphore (last `nmsg` deps), not the head
                 kNoCtrIn = 32,     // the receive connection carries no FIFO message: no head/tail counters
                 kPubSem = 64,      // publish this op's semaphore (a receive waits on it)
                 kNoCtrOut = 128 }; // the send connection carries no FIFO message
enum : uint8_t { kSrcFromSource = 1, kDstFromSource = 2 };
constexpr int kBufs = 5;      // per rank: input, output, scratch, source, result (see LaunchArgs::bufs)
constexpr int kSource = 3;
constexpr int kResult = 4;

struct DevOp {  // 32 bytes
  uint8_t opcode;
  uint8_t src_buf;
  uint8_t dst_buf;
  uint8_t has_dep;
  int16_t ndeps;
  uint8_t direct;  // kInDirect: the incoming message is already in place;
                   // kOutDirect: write the outgoing message into the receiver's buffer;
                   // kInPull: read the incoming message from the sender's span (in_buf, in_off);
                   // kOutPull: the outgoing message stays in this rank's span (publish only)
  uint8_t in_buf;  // kInPull: sender's buffer id
  int32_t src_off;
  int32_t dst_off;
  int32_t count;
  int32_t dep_begin;
  int32_t in_off;   // kInPull: sender's chunk offset
  uint8_t src_rbuf;  // buffer the src span is read from (kSource: the caller's const send buffer)
  uint8_t dst_rbuf;  // buffer reduce's dst span is read from
  uint8_t nmsg;      // trailing deps that are message deps (kMsgDep; skipped in LL launches)
  uint8_t hot;       // 1: the data this op writes is read again soon (its message's receiver reads
                     // it): stores keep it in L2 (evict_last)
};

struct DevDep {
  int32_t sem;   // semaphore base index of the depended-on thread block (lane is added)
  int32_t step;  // depended-on step
  int32_t nops;  // op count of the depended-on thread block (progress encoding)
  int32_t mult;  // lane multiplier of the depended-on thread block (it has lanes x mult lanes)
  int32_t tbi;   // launch index of the depended-on thread block (work-queue progress table)
};

struct DevTb {
  int32_t rank_slot;  // index of the owning rank within LaunchArgs::bufs
  int32_t op_begin;
  int32_t nops;
  int32_t sem;        // semaphore base index (x lanes)
  int32_t chan_in;    // receive-side channel base index (x lanes), -1 if none
  int32_t chan_out;   // send-side channel base index (x lanes), -1 if none
  int32_t peer_slot;  // rank slot of the send peer when it runs in the same launch, else -1
  int32_t mult;       // lane multiplier: this thread block runs lanes x mult lanes (work balance)
  int32_t unit_base;  // sum of the multipliers of the launch's earlier thread blocks
  int32_t recv_slot;  // rank slot of the receive peer when it runs in the same launch, else -1
                      // (slots past the launch's own ranks hold other launches' ranks whose
                      // registered buffers this launch addresses: remote direct / pulled messages)
  int32_t sys;        // 1: a connection of this thread block reaches another GPU (.sys scope)
};

// Dataflow execution (interp_df_kernel): one node per op of every thread block of the launch; a work
// item is (node, tile) and becomes ready when all of the node's predecessors in the happens-before
// graph (the previous op of its thread block, its declared deps, the sender of its message) are
// done for that tile. Messages that are neither direct nor pulled travel through a per-launch
// mailbox (one span per message, written by the sender, read by the receiver).
struct alignas(64) DfNode {  // 64 bytes: everything an item needs in one line
  DevOp op;          // the op (launch order; DevOp::direct carries the in-launch transports)
  int32_t succ;      // first successor in LaunchArgs::df_succ
  int16_t nsucc;
  int16_t indeg;     // predecessors (distinct)
  int32_t in_mail;   // >= 0: the incoming message is read from mail + in_mail chunks
  int32_t out_mail;  // >= 0: the outgoing message is written to mail + out_mail chunks
  int8_t rank_slot;  // the thread block's rank slot (LaunchArgs::bufs), its send and receive peers'
  int8_t peer_slot;
  int8_t recv_slot;
  int8_t pad_;
  int32_t tbi;       // launch thread block
  int32_t pad2_[2];
};
struct DfSucc {  // successor node and its predecessor count
  int32_t node;
  int32_t indeg;
};

// One side of one connection for one lane.  The FIFOs and `head` live in the receiver's memory,
// `tail` in the sender's memory (NVLink buffers on the receiving GPU). Every
// protocol has its own slots (NCCL keeps per-protocol buffers for the same reason): a line protocol
// validates a slot by flags embedded in the data, so it must never see another protocol's payload.
enum : int { kProtoSimple = 0, kProtoLL = 1, kProtoLL128 = 2, kNumProtos = 3 };
struct DevChan {
  char* fifo[kNumProtos];            // per protocol: slots x slot_bytes[p]
  uint64_t* head;                    // messages posted (written by the sender; Simple only)
  uint64_t* tail;                    // messages consumed (written by the receiver)
  uint64_t* mine;                    // this side's persistent message counter
  int64_t slot_bytes[kNumProtos];    // bytes of one slot: tile unit x the connection's largest count
};

struct LaunchArgs {
  const DevTb* tbs;
  const DevOp* ops;
  const DevDep* deps;
  const DevChan* chans;
  uint64_t* sems;
  int32_t ntbs;
  int32_t weight;       // sum of the thread blocks' lane multipliers: units = lanes x weight
  int32_t lanes;
  int32_t slots;
  int32_t sys_scope;    // 1: peers on other GPUs (NVLink, .sys fences); 0: same-device loopback
  int64_t chunk_elems;  // elements per chunk
  int64_t tile_elems;   // elements per (big) tile
  int64_t ntiles;
  int64_t small_elems;  // tapered tiles: n_head small tiles, n_big big ones, then small ones to the end
  int64_t n_head;
  int64_t n_big;
  uint64_t epoch;       // launch counter of this device (semaphore tag); used when epoch_ptr is null
  uint64_t* epoch_ptr;  // device-side launch counter: read by every block at start, advanced by the last
                        // block to read it (so CUDA-graph replays of a captured launch get fresh epochs)
  int32_t* epoch_ctr;   // blocks of the current launch that have read *epoch_ptr (reset by the last one)
  uint64_t timeout_ns;  // spin-wait watchdog; 0 disables
  int32_t* abort_flag;  // device word: any block that times out raises it
  uint64_t* err_info;   // host-mapped: {code, rank, tb, step, tile, what, 0, 0}
  uint64_t* trace;      // optional %globaltimer event log: [block][op seq][4] (see interp.cuh)
  int32_t trace_ops;    // ops recorded per unit
  int32_t unit_warps;   // warps interpreting one (thread block, lane); kThreads/32 divisible by it
  int32_t group;        // tiles per op-major group inside a lane (1 = tile-major)
  int32_t tma_stages;   // shared-memory stages per unit for bulk copies (0: register path only)
  int32_t stage_bytes;  // bytes per stage
  int32_t discard;      // drop consumed FIFO lines from L2 (discard.global.L2)
  int32_t transports;   // mask applied to DevOp::direct (0: every message through the FIFO)
  int32_t tma_sys_ops;  // mask applied to tma_ops on thread blocks with a cross-GPU connection (DevTb::sys)
  int64_t clip_elems;   // > 0: ragged AllReduce on the caller's buffer, tiles cut at this many elements
                        // of the rank block (every op moves one chunk, src_off == dst_off)
  int32_t tma_ops;      // bit 0: bulk copies for pure-copy ops, bit 1: staged reductions
  int64_t tma_min;      // bytes below which an op takes the register path
  int32_t l2hint;       // bit 0: evict_last stores of hot data (DevOp::hot), bit 1: evict_first bulk loads
  int32_t pad4_;
  int32_t uniform;      // 1: every thread block runs `lanes` lanes (LL launches: FIFOs need matched lanes)
  int32_t wq;           // 1: work-queue mode (see interp.cuh interp_wq)
  int32_t* wq_next;     // work-queue claim counter (zeroed before the launch)
  const int32_t* wq_order;  // claim position -> item (tile * ntbs + thread block); null: identity
  uint64_t* prog;       // work-queue progress: [thread block][tile] = (epoch << 32) | steps done
  // dataflow mode (interp_df_kernel)
  const DfNode* df_nodes;
  const DfSucc* df_succ;     // successors
  const int32_t* df_roots;   // nodes without predecessors
  int32_t* df_cnt;           // [tile][node] predecessors done (self-resetting: zero between launches)
  int32_t* df_q;             // ready queue of items + 1 (self-resetting)
  int32_t* df_ctr;           // {pop, push} counters (zeroed before the launch)
  char* mail;                // mailbox of the launch's non-direct, non-pulled messages
  int32_t df_n;              // nodes
  int32_t df_nroots;
  int32_t df_policy;         // bit 0: continuations (a unit runs the successor it made ready next)
  int32_t df_window;         // tiles whose roots may run ahead of the finished items (0: unbounded)
  char* bufs[kMaxLocalRanks][kBufs];  // per local rank: input, output, scratch, source, result (the
                                     // caller's recvbuff shifted so that an owned ReduceScatter chunk
                                     // keeps its input offset; see result_writes), source (the caller's
                                     // const data the in-place IR's first reads see; = input when
                                     // the working buffer was pre-copied)
};

}  // namespace gc3
