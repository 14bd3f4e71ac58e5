/*
 * gc3_oracle.h — CPU restatement of the GC3-IR interpreter.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library, and only as the checker or as the timed CPU baseline.  The product path
 * (paper_2201_11840_b200/csrc, libgc3.so) never links or calls it.
 *
 * The reference ships no interpreter: its functional simulator is spec-only and symbolic
 * (SPEC.md:436-502).  This is a NUMERIC restatement of those semantics:
 *   - thread blocks step sequentially through their ops (Fig. 4);
 *   - cross-thread-block deps wait until semaphore[tb] >= step (
 *     scheduler.hpp:519-559);
 *   - the k-th send on a connection (src, dst, channel) is matched with the k-th receive
 *     (scheduler.hpp:251-273, 655-683), FIFO capacity s;
 *   - opcode dataflow per lowering.hpp:68-77 / 96-119;
 *   - chunk tiling loop outermost.
 * Numeric extensions defined by this build (the reference is symbolic): reduction = ncclRedOp_t
 * on ncclDataType_t; f16/bf16 via f32 with round-to-nearest-even; wrapping integers.
 *
 * Parity status: the symbolic level (which input chunks land/are combined where) is PINNED
 * against the reference's own chunk algebra and postconditions (oracle/_ref/libref.so, golden
 * files tests/golden/symbolic/).  Numeric values are a restatement (the reference has no
 * numeric semantics); interleaving- and fusion-invariance are tested.
 */
#ifndef GC3_ORACLE_H
#define GC3_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GC3O_MAX_DEPS 8

/* opcodes, in lowering.hpp:20-30 order */
enum { GC3O_SEND = 0, GC3O_RECV, GC3O_COPY, GC3O_REDUCE, GC3O_RRC, GC3O_RCS, GC3O_RRCS, GC3O_RRS, GC3O_NOP };
/* buffers, core.hpp:167 order */
enum { GC3O_INPUT = 0, GC3O_OUTPUT = 1, GC3O_SCRATCH = 2 };
/* modes */
enum { GC3O_DETERMINISTIC = 0, GC3O_RANDOM = 1, GC3O_THREADED = 2 };
/* return codes */
enum { GC3O_OK = 0, GC3O_DEADLOCK = 1, GC3O_ERROR = 2 };

typedef struct {
  int32_t opcode, src_buf, src_off, dst_buf, dst_off, count, has_dep, ndeps;
  int32_t dep_tb[GC3O_MAX_DEPS];   /* index of the tb within its rank's threadblock list */
  int32_t dep_step[GC3O_MAX_DEPS];
} gc3o_op;

typedef struct {
  int32_t rank, send_peer, recv_peer, channel, first_op, nops;
} gc3o_tb;

typedef struct {
  int32_t nranks, ntbs;
  const gc3o_tb* tbs;   /* grouped by rank, in IR order */
  const gc3o_op* ops;
  int32_t nchunks[3];
  int32_t inplace;
} gc3o_program;

/*
 * Executes the program.  bufs[r*3 + b] is rank r's buffer b (output may equal input for
 * in-place programs).  Every chunk holds chunk_elems elements of `dtype` (ncclDataType_t
 * numbering); chunk i of a buffer occupies elements [i*chunk_elems, (i+1)*chunk_elems).
 * mode: DETERMINISTIC (round-robin, unbounded FIFOs, untiled — the parity reference),
 *       RANDOM (seeded interleaving, FIFO capacity `slots`, tiles of tile_elems, fused ops
 *               atomic: they need a full incoming slot and a free outgoing slot at once),
 *       THREADED (one pthread per IR thread block, blocking FIFOs of capacity `slots`,
 *                 tiles of tile_elems — the timed CPU baseline; `nthreads_cap` unused > 0 caps
 *                 nothing, every tb needs its own thread to be deadlock-free).
 * Returns GC3O_OK, GC3O_DEADLOCK (err names the blocked thread blocks) or GC3O_ERROR.
 */
int gc3o_run(const gc3o_program* p, void* const* bufs, size_t chunk_elems, int dtype, int redop,
             int mode, uint64_t seed, int slots, size_t tile_elems, char* err, size_t errlen);

/* Element-wise reduction a[i] = a[i] (op) b[i] for n elements: the arithmetic every reducing
 * opcode uses, exported so tests can check the device arithmetic table against it. */
int gc3o_reduce(void* a, const void* b, size_t n, int dtype, int redop);

size_t gc3o_dtype_size(int dtype);

/* One conflicting pair of accesses to chunk slot (rank, buf, index): accesses (tb_a, step_a) and
 * (tb_b, step_b) of that rank, unordered by happens-before.  kind: 0 write/write, 1 write then
 * read, 2 read then write. */
typedef struct {
  int32_t rank, buf, index, kind, tb_a, step_a, tb_b, step_b;
} gc3o_race;

/* Vector-clock race detection over block steps, message edges (k-th send
 * -> k-th receive) and dep (semaphore) edges.  Fills up to `max` pairs into `out`; returns the
 * number of conflicting pairs found, or -1 (err set) for a malformed or deadlocking program. */
int gc3o_races(const gc3o_program* p, gc3o_race* out, int max, char* err, size_t errlen);

#ifdef __cplusplus
}
#endif
#endif
