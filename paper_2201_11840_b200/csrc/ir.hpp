// GC3-IR host library: data model, strict loader, canonical writer, structural validation,
// static slot check and the runtime `instances` rewrite.
//
// Drop-in for the reference compiler→runtime boundary:
//   data model      ir.hpp:68-140        → Program / ThreadBlock / Op / Dep
//   deserialize     ir.hpp:188-310       → parse_program (same required/unknown-key rules and the
//                                          same schema-error JSON paths, core.hpp:74-83, 478-491)
//   serialize       ir.hpp:145-186       → serialize (byte-identical canonical JSON)
//   validate        ir.hpp:341-439       → validate (same rules, same messages, same order)
//   check_slots     scheduler.hpp:633-734→ check_slots
//   parallelize(k)  program.hpp:366-419  → replicate_instances (SURVEY.md Finding 5)
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace gc3 {

// lowering.hpp:20-30 order; JSON names lowering.hpp:32-45
enum class Opcode : int8_t { send = 0, recv, copy, reduce, rrc, rcs, rrcs, rrs, nop };
// core.hpp:167 order
enum class Buf : int8_t { input = 0, output = 1, scratch = 2 };
// ir.hpp:21
enum class Proto : int8_t { simple = 0, ll = 1, ll128 = 2 };

const char* opcode_name(Opcode op);
const char* buf_name(Buf b);
const char* proto_name(Proto p);

// lowering.hpp:55-66
inline bool op_receives(Opcode op) {
  return op == Opcode::recv || op == Opcode::rrc || op == Opcode::rcs || op == Opcode::rrcs || op == Opcode::rrs;
}
inline bool op_sends(Opcode op) { return op == Opcode::send || op == Opcode::rcs || op == Opcode::rrcs || op == Opcode::rrs; }
inline bool op_reduces(Opcode op) { return op == Opcode::reduce || op == Opcode::rrc || op == Opcode::rrcs || op == Opcode::rrs; }

struct Dep {
  int tb = 0;
  int step = 0;
};

struct Op {
  int step = 0;
  Opcode op = Opcode::nop;
  Buf src_buf = Buf::input;
  int src_off = 0;
  Buf dst_buf = Buf::input;
  int dst_off = 0;
  int count = 1;
  std::vector<Dep> deps;
  bool has_dep = false;
};

struct ThreadBlock {
  int id = 0;
  int send_peer = -1;
  int recv_peer = -1;
  int channel = 0;
  std::vector<Op> ops;
};

struct Gpu {
  int rank = 0;
  std::vector<ThreadBlock> tbs;
};

struct Program {
  std::string name;
  std::string collective;
  Proto proto = Proto::simple;
  bool inplace = false;
  int nchunks[3] = {0, 0, 0};  // input, output, scratch
  uint64_t min_bytes = 0;
  uint64_t max_bytes = 1ull << 40;
  std::vector<Gpu> gpus;

  int ranks() const { return static_cast<int>(gpus.size()); }
  const ThreadBlock* find_tb(int rank, int id) const;
};

// collective names accepted by the reference (core.hpp:217-237)
bool known_collective(const std::string& name);

struct SchemaError {
  std::string path;     // e.g. "gpus[0].threadblocks[1].channel" ("" for the document)
  std::string message;  // e.g. "missing required key"
  // reference schema_error::what(): "schema: " + path + ": " + message (core.hpp:65, 78)
  std::string what() const { return "schema: " + path + ": " + message; }
};

bool parse_program(const std::string& text, Program& out, SchemaError& err);
std::string serialize(const Program& p);

// Machine budgets used by validate (core.hpp:444-474). B200 default budget: 148 SMs.
struct Topology {
  int nodes = 1;
  int gpus_per_node = 1;
  int slots = 8;
  int max_channels = 32;
  int max_threadblocks = 80;
  int ranks() const { return nodes * gpus_per_node; }
};

std::vector<std::string> validate(const Program& p, const Topology& topo);

struct SlotViolation {
  int src_gpu = 0, dst_gpu = 0, channel = 0, send_tb = -1, send_step = -1;
  std::string what;
};
std::vector<SlotViolation> check_slots(const Program& p, int slots);

// Replicates the program into k instances on disjoint channels and sub-chunks: instance j maps
// off -> off*k + j*count, channel -> channel + j*nch, tb id -> id + j*ntb, dep tb likewise, and
// multiplies nchunks by k. Equals the reference's compile-time parallelize(k) for programs whose
// ops all share one count (SURVEY.md Finding 5).
// Ops of several counts have no consistent blocking (a count-4 span's block j and a count-1 op on one
// of its chunks land on different sub-chunks), so callers must check uniform_counts first.
Program replicate_instances(const Program& p, int k);
bool uniform_counts(const Program& p);

// Built-in programs the runtime uses when no registered IR matches a call (drop-in NCCL use without
// gc3RegisterIR): ring AllReduce / AllGather / ReduceScatter on one channel and the direct AlltoAll,
// for any rank count >= 2. They are the reference compiler's programs for these algorithms
// (ring_allreduce / ring allgather / ring reducescatter / alltoall with one node):
// op for op identical to its output (tests/test_builtin_irs.py). collective: "allreduce",
// "allgather", "reducescatter" or "alltoall"; returns false for anything else.
bool builtin_program(const std::string& collective, int nranks, Program& out, int channels = 1);
// Comm-time program generation (compiler in the loop): algo "ring" (allreduce with
// `channels` rings: chunk k on channel k % channels; allgather / reducescatter: one ring), "direct"
// (alltoall), "allpairs" (allreduce), "hier" (allreduce over nranks / channels nodes of `channels`
// GPUs), each replicated into `instances` instances (the reference's
// parallelize(k), program.hpp:366-419). False for an unsupported combination.
bool generate_program(const std::string& algo, const std::string& collective, int nranks, int channels, int instances, Program& out);

}  // namespace gc3
