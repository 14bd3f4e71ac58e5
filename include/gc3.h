/*
 * gc3.h — C ABI of the B200 GC3-IR runtime (libgc3.so).
 *
 * Drop-in boundary. The reference defines the compiler→runtime boundary as the
 * *.ir.json file (schema SPEC.md:425; reader ir.hpp:226-310; validate ir.hpp:341-439) and its paper
 * runtime as "API-compatible with NCCL". The reference ships no runtime, so each
 * entry point below cites the interface it replaces:
 *   - the nccl.h subset (NCCL 2.27.3 /usr/include/nccl.h line numbers; ncclAlltoAll from the
 *     torch-bundled NCCL 2.28.9 nccl.h:460) that the paper's MSCCL runtime exposes;
 *   - gc3Ir* : the reference IR library (ir.hpp deserialize/serialize/validate,
 *     scheduler.hpp check_slots, program.hpp parallelize) as host-only C calls;
 *   - gc3RegisterIR / gc3SetProtocolOverride / gc3QueryPlan / gc3SetConfig: the paper runtime's
 *     "IRs parsed and stored in GPU memory at setup" + "size-range selection" (PAPER.md:387,
 *     439-440) and the chunk/instance/protocol parameters.
 * All calls return ncclResult_t; no C++ exception crosses the ABI. Plain pointers and sizes only.
 */
#ifndef GC3_H_
#define GC3_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* cudaStream_t without pulling in the CUDA headers */
typedef struct CUstream_st* cudaStream_t;

#define GC3_VERSION_CODE 22809 /* reported by ncclGetVersion: NCCL 2.28.9-compatible subset */

/* nccl.h:41-49 */
typedef enum {
  ncclSuccess = 0,
  ncclUnhandledCudaError = 1,
  ncclSystemError = 2,
  ncclInternalError = 3,
  ncclInvalidArgument = 4,
  ncclInvalidUsage = 5,
  ncclRemoteError = 6,
  ncclInProgress = 7,
  ncclNumResults = 8
} ncclResult_t;

/* nccl.h:37-38 */
#define NCCL_UNIQUE_ID_BYTES 128
typedef struct {
  char internal[NCCL_UNIQUE_ID_BYTES];
} ncclUniqueId;

typedef struct gc3Comm* ncclComm_t;

/* nccl.h:260-268 (ncclAvg is rejected: the IR fixes a pure reduction, PAPER.md has no averaging) */
typedef enum { ncclSum = 0, ncclProd = 1, ncclMax = 2, ncclMin = 3, ncclAvg = 4, ncclNumOps = 5 } ncclRedOp_t;

/* nccl.h:278-290 */
typedef enum {
  ncclInt8 = 0, ncclChar = 0, ncclUint8 = 1, ncclInt32 = 2, ncclInt = 2, ncclUint32 = 3,
  ncclInt64 = 4, ncclUint64 = 5, ncclFloat16 = 6, ncclHalf = 6, ncclFloat32 = 7, ncclFloat = 7,
  ncclFloat64 = 8, ncclDouble = 8, ncclBfloat16 = 9, ncclFloat8e4m3 = 10, ncclFloat8e5m2 = 11,
  ncclNumTypes = 12
} ncclDataType_t;

/* ---- communicator lifecycle (nccl.h:140-239) ------------------------------------------------ */
ncclResult_t ncclGetVersion(int* version);                                               /* nccl.h:140 */
ncclResult_t ncclGetUniqueId(ncclUniqueId* uniqueId);                                    /* nccl.h:146 */
ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId commId, int rank); /* nccl.h:160 */
/* nccl.h:169. Extension: devlist may repeat a device; the ranks sharing a device then run as
 * "loopback" ranks inside one launch per device (single-GPU testing and measurement). */
ncclResult_t ncclCommInitAll(ncclComm_t* comm, int ndev, const int* devlist);
ncclResult_t ncclCommDestroy(ncclComm_t comm);                                           /* nccl.h:181 */
ncclResult_t ncclCommAbort(ncclComm_t comm);                                             /* nccl.h:186 */
const char* ncclGetErrorString(ncclResult_t result);                                    /* nccl.h:215 */
const char* ncclGetLastError(ncclComm_t comm);                                          /* nccl.h:219 */
ncclResult_t ncclCommGetAsyncError(ncclComm_t comm, ncclResult_t* asyncError);           /* nccl.h:227 */
ncclResult_t ncclCommCount(const ncclComm_t comm, int* count);                           /* nccl.h:231 */
ncclResult_t ncclCommCuDevice(const ncclComm_t comm, int* device);                       /* nccl.h:235 */
ncclResult_t ncclCommUserRank(const ncclComm_t comm, int* rank);                         /* nccl.h:239 */

/* ---- collectives: each runs the registered GC3-IR selected by collective + size_range ------ */
/* nccl.h:392-393 */
ncclResult_t ncclAllReduce(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t datatype,
                           ncclRedOp_t op, ncclComm_t comm, cudaStream_t stream);
/* nccl.h:408-410 */
ncclResult_t ncclReduceScatter(const void* sendbuff, void* recvbuff, size_t recvcount, ncclDataType_t datatype,
                               ncclRedOp_t op, ncclComm_t comm, cudaStream_t stream);
/* nccl.h:425-426 */
ncclResult_t ncclAllGather(const void* sendbuff, void* recvbuff, size_t sendcount, ncclDataType_t datatype,
                           ncclComm_t comm, cudaStream_t stream);
/* torch NCCL 2.28.9 nccl.h:460-461 */
ncclResult_t ncclAlltoAll(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t datatype,
                          ncclComm_t comm, cudaStream_t stream);
/* MSCCL spelling used by the north star */
ncclResult_t ncclAllToAll(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t datatype,
                          ncclComm_t comm, cudaStream_t stream);

/* nccl.h:493 / 503 */
ncclResult_t ncclGroupStart(void);
ncclResult_t ncclGroupEnd(void);

/* ---- GC3 extensions ------------------------------------------------------------------------ */
/* Registers a GC3-IR program (file path, or the text itself: GC3-IR JSON if it starts with '{', an
 * MSCCL algorithm XML if it starts with '<'; a file is XML if its content starts with '<') on this
 * rank; every rank must register the same programs in the same order (collective, like comm init).
 * instances > 1 applies the runtime parallelization rewrite (program.hpp:366-419; SURVEY.md
 * Finding 5). The IR is loaded with the reference schema rules, validated (ir.hpp:341-439) against
 * a 1 x nranks topology with the B200 budget (148 thread blocks), staged in device memory, and its
 * FIFOs are exchanged with the peers. *ir_id receives the registration index. */
ncclResult_t gc3RegisterIR(ncclComm_t comm, const char* path_or_json, int instances, int* ir_id);
/* proto: -1 = as tagged in the IR, 0 = simple, 1 = ll (16-byte lines, 8 payload bytes), 2 = ll128 (128-byte lines, 120 payload bytes) */
ncclResult_t gc3SetProtocolOverride(ncclComm_t comm, int ir_id, int proto);

typedef struct {
  int ir_id;          /* selected IR, -1 if none matches */
  int protocol;       /* effective protocol: 0 simple, 1 ll, 2 ll128 */
  int lanes;          /* CUDA blocks per IR thread block */
  int grid;           /* CUDA blocks in the launch on this rank's device */
  int local_ranks;    /* ranks executed by that launch */
  int slots;          /* FIFO slots per connection */
  int64_t chunk_elems;
  int64_t tile_elems;
  int64_t ntiles;
  int64_t slot_bytes;
  int64_t wire_bytes; /* max over ranks of bytes sent or received by send/recv-family ops */
  int64_t hbm_bytes;  /* algorithmic local bytes (reads + writes of user/scratch buffers) of the launch */
  char name[64];      /* IR name */
  int unit_warps;     /* warps interpreting one (thread block, lane) */
  int group;          /* tiles per op-major group inside a lane */
  int mode;           /* 0: static lanes, 1: work queue, 2: dataflow (ready (op, tile) items) */
  int mail_messages;  /* dataflow: messages carried through the launch's mailbox */
  int remote_messages; /* direct / pulled receives whose sender runs in another launch (registered user buffers) */
  int sys_scope;      /* 1: some thread block has a connection to another GPU (.sys fences there) */
  int tma_stages;     /* bulk-copy stages per unit (0: register path only) */
} gc3PlanInfo;
/* collective: 0 allreduce, 1 allgather, 2 reducescatter, 3 alltoall; count as in the NCCL call. */
ncclResult_t gc3QueryPlan(ncclComm_t comm, int collective, size_t count, ncclDataType_t datatype, gc3PlanInfo* info);

/* Runtime knobs; defaults from the GC3_<KEY> environment variables (upper case). Registration-time
 * keys (apply to IRs registered afterwards): "slots", "slot_bytes", "max_lanes", "direct" (bit 0
 * direct messages, bit 1 pulled messages), "source" (const-source reads and result writes),
 * "balance" (lane multipliers; 2 = rounded up), "mult_cap", "l2hint" (bit 0 evict_last stores, bit 1
 * evict_first loads). Launch-time keys: "lanes", "tile_bytes", "timeout_ms", "unit_warps", "group"
 * (0 = automatic), "tma" (bit 0 bulk copies, bit 1 staged reductions, bit 2 register-store copies),
 * "tma_min", "discard", "wq" (work-queue mode; 2 = also for chain programs), "wq_items", "taper",
 * "ll_max_bytes" / "ll128_max_bytes" (Simple IRs with >= "ll_wide_tbs" thread blocks per rank run
 * LL / LL128 up to these many bytes per rank; narrower IRs with >= 8 ops per thread block run LL up
 * to "ll_narrow_max_bytes"), "trace"; dataflow executor:
 * "df" (0 off, 1 reducing chain programs, 2 every Simple program), "df_items", "df_min_tile",
 * "df_max_tile", "df_big_bytes", "df_big_tile", "df_waves" (1: tile count rounded to whole waves
 * of units; 2: also one wave per level for reducing chain programs whose static plan has fewer than
 * "df_wave_max_lanes" lanes, tiles down to "df_wave_min_tile"), "df_policy" (bit 0 continuations,
 * bit 1 fence + atomic + fence successor counters), "df_window". */
ncclResult_t gc3SetConfig(ncclComm_t comm, const char* key, int64_t value);

/* In-kernel event log of the last launch on comm's device when config "trace" (GC3_TRACE) is set
 * (SURVEY.md §5 tracing): for CUDA block b and its q-th op, out[(b*ops_per_block + q)*4 + k] holds
 * %globaltimer ns at k = 0 start, 1 preconditions met, 2 warp 0's data done, 3 published (0 if not
 * reached). Block b executes IR thread block b / lanes (ranks of the device in rank order, thread
 * blocks in IR order), lane b % lanes. With out == NULL only the shape is returned. Synchronizes. */
ncclResult_t gc3GetTrace(ncclComm_t comm, uint64_t* out, size_t max_words, int* grid, int* ops_per_block, int* lanes);

/* ---- IR library, host only (no CUDA needed) ---------------------------------------------- */
typedef struct gc3Ir* gc3Ir_t;
/* ir.hpp:226-310. On a schema error returns ncclInvalidArgument and, if err is non-NULL, sets
 * *err to a malloc'd "path\tmessage" string (free with gc3Free). */
ncclResult_t gc3IrParse(const char* text, gc3Ir_t* ir, char** err);
/* MSCCL algorithm XML (the paper runtime's format) into the
 * same program: one dependency per step, `nop` steps carry extra dependencies and (fold_nops != 0)
 * are folded back into the following op. Errors: ncclInvalidArgument, *err = "xml: path: message". */
ncclResult_t gc3IrParseXml(const char* text, int fold_nops, gc3Ir_t* ir, char** err);
/* The program as MSCCL XML (multi-dependency ops expanded into nop chains); malloc'd. */
ncclResult_t gc3IrToXml(gc3Ir_t ir, char** text);
/* ir.hpp:145-186: canonical JSON (malloc'd, free with gc3Free) */
ncclResult_t gc3IrSerialize(gc3Ir_t ir, char** text);
/* ir.hpp:341-439: newline-separated issues ("" if valid) against an nodes x gpus_per_node
 * topology with the given budgets (<= 0 keeps the reference defaults 80 / 32). */
ncclResult_t gc3IrValidate(gc3Ir_t ir, int nodes, int gpus_per_node, int max_threadblocks, int max_channels, char** issues);
/* scheduler.hpp:633-734: newline-separated violations */
ncclResult_t gc3IrCheckSlots(gc3Ir_t ir, int slots, char** violations);
/* program.hpp:366-419 parallelize(k) as an IR rewrite; returns a new handle */
ncclResult_t gc3IrReplicate(gc3Ir_t ir, int instances, gc3Ir_t* out);
/* Host-side plan introspection (used by tests; no CUDA needed):
 * arena layout of `rank` (FIFO offsets, counter offsets) as JSON — every process computes every
 * peer's layout from the program text, so this must agree across processes; */
ncclResult_t gc3IrArenaLayout(gc3Ir_t ir, int rank, int lanes, int slots, int64_t slot_unit, char** json);
/* [rank][tb][step] flags of the happens-before analysis (1: receive written in place by its sender,
 * 2: send written into the receiver's span); */
ncclResult_t gc3IrDirectMessages(gc3Ir_t ir, char** json);
/* whether the lane order "groups of `group` tiles, op-major" is deadlock-free at FIFO depth `slots`. */
ncclResult_t gc3IrOrderCheck(gc3Ir_t ir, int64_t tiles, int group, int slots, int* deadlock_free);
/* Single-node bootstrap all-gather of fixed-size records through /dev/shm keyed by the unique id
 * (what ncclCommInitRank / gc3RegisterIR use to exchange device info and CUDA IPC handles):
 * out receives nranks * bytes, rank-major. */
ncclResult_t gc3BootstrapExchange(const ncclUniqueId* id, int rank, int nranks, const void* payload, size_t bytes, void* out,
                                  int timeout_ms);
/* [rank][tb][step] flags of the const-source analysis (1: the op's src read sees the caller's send
 * buffer, 2: reduce's dst read does); *complete = 1 when every first read of `input` is covered, so
 * in-place IRs need no pre-copy of sendbuff (SURVEY.md §7 hard part 6). */
ncclResult_t gc3IrSourceReads(gc3Ir_t ir, int* complete, char** json);
/* [rank][tb][step] flags (1: the op's final write of the rank's owned ReduceScatter block goes
 * straight to recvbuff); *complete = 1 when they cover every owned block (no copy-out). */
ncclResult_t gc3IrResultWrites(gc3Ir_t ir, int* complete, char** json);
/* per [rank][thread block] lane multipliers of the work balance (JSON); with balance on, thread block
 * i of a launch runs lanes x mult lanes (units in launch order). */
ncclResult_t gc3IrLaneMultipliers(gc3Ir_t ir, char** json);
/* The built-in program the runtime uses for `collective` ("allreduce", "allgather", "reducescatter",
 * "alltoall") on nranks ranks when no registered IR matches a call (see gc3RegisterIR). */
ncclResult_t gc3IrBuiltin(const char* collective, int nranks, gc3Ir_t* ir);
/* The built-in program a call of `bytes` (per-rank buffer bytes, the size_range measure) runs when no
 * registered IR matches: AllReduce per size tier (multi-channel ring with LL lines / with LL128 lines /
 * single ring / multi-channel ring, each with its size_range; config gen, gen_small, gen_ll128,
 * gen_large), the other collectives as gc3IrBuiltin. */
ncclResult_t gc3IrBuiltinSized(const char* collective, int nranks, uint64_t bytes, gc3Ir_t* ir);
/* Comm-time program generation (compiler in the loop): algo "ring" (allreduce on
 * `channels` rings, chunk k on channel k % channels; allgather / reducescatter on one), "allpairs"
 * (allreduce) or "direct" (alltoall), replicated into `instances` instances -- the reference
 * compiler's parallelize(k) (program.hpp:366-419). ncclInvalidArgument for other combinations. */
ncclResult_t gc3IrGenerate(const char* algo, const char* collective, int nranks, int channels, int instances, gc3Ir_t* ir);
/* Timed model (SPEC.md:464-481 run_timed, as an alpha-beta model over the happens-before graph,
 * calibrated on a B200 in loopback): predicted microseconds of one launch of the program with chunks
 * of chunk_bytes, protocol (0 simple, 1 ll) and `lanes` lanes per thread block. */
ncclResult_t gc3IrPredict(gc3Ir_t ir, int64_t chunk_bytes, int protocol, int lanes, double* us);
/* Timed simulator (SPEC.md:464-481 run_timed / sweep): discrete-event alpha-beta model with chunk
 * tiling; a message on an ordered GPU pair costs alpha + bytes / bandwidth of its link class (0 same
 * GPU, 1 same node, 2 other node), concurrent messages on one pair share its bandwidth (processor
 * sharing); local reductions cost bytes / gamma. gc3SimDefaults fills the B200 calibration. */
typedef struct {
  int nranks_gpu;          /* entries of rank_gpu (0: rank r on GPU r) */
  const int* rank_gpu;     /* GPU of each rank (e.g. all 0: loopback on one GPU) */
  int gpus_per_node;
  double alpha_us[3];      /* per message, per link class */
  double gbps[3];          /* bandwidth of one ordered GPU pair, per link class */
  double gamma_gbps;       /* local reduction rate */
  double copy_gbps;        /* local copy rate */
  int protocol;            /* 0 simple, 1 ll, 2 ll128 (alpha x 1 / 0.25 / 0.5, beta x 1 / 2 / 1.07) */
  int slots;               /* FIFO slots per connection (0: the protocol's, 2 / 8 / 4) */
  int64_t chunk_bytes;
  int64_t tile_bytes;      /* 0: one tile per chunk */
  double launch_us;        /* added to the makespan */
  double hbm_gbps;         /* 0: off (SPEC); else local reads/writes and same-GPU messages share one
                              processor-shared device-memory resource per GPU of this rate */
  int lanes;               /* units per thread block, lane l taking tiles l, l + lanes, ... (0 or 1: one) */
  int group;               /* tiles per op-major group inside a lane (0 or 1: tile-major, Fig. 4) */
  double op_us;            /* device-memory mode: fixed cost of every op per tile */
  int msg_read_passes;     /* device-memory mode: extra passes of a reducing receive reading its message */
  int workers;             /* > 0: dataflow execution (the runtime's dataflow executor) with this many units */
} gc3SimConfig;
typedef struct {
  int completed;           /* 0: deadlock (see `deadlock`) */
  double makespan_us;
  double util[3];          /* mean busy fraction of the ordered GPU pairs used, per link class */
  int64_t messages;
  int64_t tiles;
  char deadlock[256];
} gc3SimReport;
ncclResult_t gc3SimDefaults(gc3SimConfig* cfg);
ncclResult_t gc3IrSimulate(gc3Ir_t ir, const gc3SimConfig* cfg, gc3SimReport* report);
/* one run per size (bytes of a rank's input buffer); *csv = "size_bytes,makespan_us,util_intra,util_inter"
 * rows (free with gc3Free) */
ncclResult_t gc3IrSweep(gc3Ir_t ir, const gc3SimConfig* cfg, const int64_t* sizes, int nsizes, int64_t tile_bytes, char** csv);
ncclResult_t gc3IrFree(gc3Ir_t ir);
void gc3Free(void* p);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* GC3_H_ */
