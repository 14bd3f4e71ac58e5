// Host runtime of the B200 GC3-IR interpreter: communicators, bootstrap, IR registration,
// FIFO arenas + CUDA IPC exchange, device plans, NCCL-style groups and kernel launch.
//
// Paper runtime, re-designed for one NVSwitch box of B200s:
//   * "all GC3-IR programs ... are parsed and stored in the GPU memory" ->
//     gc3RegisterIR stages each program as a device plan (DevTb/DevOp/DevDep, devplan.hpp);
//   * remote buffers on the receiving GPU with s FIFO slots -> one arena per
//     (rank, IR) holding the receive FIFOs, counters and credits, exported with cudaIpc handles;
//   * "selects the right algorithm ... based on user configurable size ranges" ->
//     select_ir() over the registered programs' size_range (ir.hpp:112-116); no NCCL fallback
//     exists on this path: an unmatched call returns ncclInvalidUsage;
//   * cooperative launch of all thread blocks -> one launch per device covering
//     every rank hosted there (several "loopback" ranks can share one GPU).
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <sys/types.h>
#include <dlfcn.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <cmath>
#include <map>
#include <numeric>
#include <memory>
#include <mutex>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing without an attached tool

#include "../../include/gc3.h"
#include "devplan.hpp"
#include "ir.hpp"
#include "msccl_xml.hpp"
#include "timed.hpp"

namespace gc3 {

using KernelFn = void (*)(LaunchArgs);
KernelFn interp_kernel(int dtype, int redop, int proto);
KernelFn interp_kernel_wq(int redop);  // work-queue kernel (copy-only programs), nullptr otherwise
KernelFn interp_kernel_df(int dtype, int redop);  // dataflow kernel (Simple, every rank in the launch)
cudaError_t interp_launch(KernelFn fn, const LaunchArgs& args, int grid, size_t smem, cudaStream_t stream);
int interp_blocks_per_sm(KernelFn fn, size_t smem);
constexpr int kStageBytesHost = 16 << 10;  // interp.cuh kStageBytes
constexpr int kMaxStagesHost = 8;          // interp.cuh kMaxStages
constexpr int kSmemBudget = 192 << 10;
constexpr size_t kDfQueueSlack = 4096;     // dataflow queue positions beyond the items (>= co-resident units)

namespace {

// ------------------------------------------------------------------------------- errors
thread_local std::string g_last_error;
std::recursive_mutex g_mu;  // communicators are not thread-safe (NCCL semantics); this guards globals

ncclResult_t set_error(ncclResult_t rc, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  if (getenv("GC3_DEBUG")) fprintf(stderr, "[gc3] %s\n", buf);
  return rc;
}

#define CUDA_TRY(call)                                                                              \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess)                                                                          \
      return set_error(ncclUnhandledCudaError, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                       __FILE__, __LINE__);                                                         \
  } while (0)

#define NCCL_TRY(call)                      \
  do {                                      \
    ncclResult_t r_ = (call);               \
    if (r_ != ncclSuccess) return r_;       \
  } while (0)

int64_t env_int(const char* name, int64_t def) {
  const char* v = getenv(name);
  return v && *v ? std::strtoll(v, nullptr, 10) : def;
}

// ------------------------------------------------------------------------------- config
struct Config {
  int slots = 2;                     // FIFO slots per connection; fused ops need >= 2 (SURVEY Finding 1)
  int64_t slot_bytes = 256 << 10;    // FIFO slot unit: max bytes of one tile (a slot holds count tiles)
  int max_lanes = 64;                // cap on lanes provisioned per connection in the arenas
  int lanes = 0;                     // 0: automatic
  int64_t tile_bytes = 0;            // 0: automatic
  int64_t timeout_ms = 20000;        // device spin-wait watchdog
  int trace = 0;                     // record the in-kernel %globaltimer event log
  int direct = 3;                    // bit 0: direct messages, bit 1: pulled messages (direct_messages)
  int source = 1;                    // in-place IRs read the caller's const buffer (source_reads)
  int unit_warps = 0;                // warps per (thread block, lane) unit; 0 = automatic
  int tma = 11;                      // bulk (TMA) engine on same-device peers: bit 0 copies, bit 1 staged
                                     // reductions, bit 3 in-place sums reduced by the L2
  int balance = 1;                   // per-component lane multipliers (lane_multipliers; 2: rounded up)
  int mult_cap = 4;                  // largest lane multiplier
  int taper = 0;                     // quarter tiles in the first and last round of every lane (measured: no gain)
  int l2hint = 3;                    // bit 0: evict_last stores for data the receiver reads soon; bit 1:
                                     // evict_first bulk loads (every span is read once)
  int wq = 1;                        // work-queue mode where possible (interp_wq)
  int64_t tma_min = 32 << 10;        // ops moving fewer bytes take the register path
  int64_t ll_max_bytes = 512 << 10;  // Simple IRs run LL up to this many bytes per rank (0: never;
                                     // measured: LL ~2x faster than Simple below ~1 MiB, BASELINE §5.2)
  int64_t ll128_max_bytes = 2 << 20;  // ... and LL128 above ll_max_bytes up to this many (0: never)
  int ll_wide_tbs = 8;               // both thresholds apply to IRs with this many thread blocks per rank
                                     // (many short chains); narrower IRs run LL only up to
  int64_t ll_narrow_max_bytes = 16 << 10;  // this many bytes (measured, profiles/r02bw_*: Simple
                                     // faster from 16-32 KiB on every narrow BASELINE program)
  int builtin = 1;                   // calls no registered IR matches run the built-in programs
  int clip = 1;                      // ragged AllReduce on the caller's buffer with clipped tiles (clip_ok IRs)
  int gen = 1;                       // built-in AllReduce per size tier (builtin_for); 0: one ring
  int64_t gen_small = 512 << 10;     // ... multi-channel ring with LL lines up to this many bytes
  int64_t gen_ll128 = 2 << 20;       // ... with LL128 lines up to this many
  int64_t gen_large = 8 << 20;       // ... single ring up to this many, multi-channel ring above
  int64_t smem_kb = 192;             // shared memory for bulk-engine stages per block (<= 220)
  int select = 0;                    // among matching IRs pick the lowest timed-model prediction
  int64_t stage_kb = 0;              // bytes per stage (0: automatic, 3+ stages per unit)
  int wq_items = 6;                  // work items per unit targeted by the work-queue tile size (measured,
                                     // C2: 4 -> 0.903, 5 -> 0.911, 6 -> 0.915, 7 -> 0.912, 8 -> 0.900 of the roofline)
  int wq_lag = 0;                    // claim deeper thread blocks' items this many tiles later (0: off)
  int discard = 1;                   // discard consumed FIFO lines from L2
  int group = 0;                     // tiles per op-major group in a lane; 0 = largest deadlock-free
  int df = 1;                        // dataflow execution (interp_df_kernel) when every rank is in the
                                     // launch: 1 = reducing programs with receive-and-forward chains,
                                     // >= 2 items per unit and >= 16 tiles per chunk, 2 = every Simple
                                     // program, 0 = off
  int df_items = 4;                  // dataflow: ready items per unit targeted by the tile size
  int64_t df_max_tile = 256 << 10;   // dataflow: largest tile
  int64_t df_min_tile = 128 << 10;   // dataflow: smallest tile (unless the chunk is smaller; measured
                                     // best on C3 / C4 / C5-RS: 64-128 KiB, per-item costs ~3 us)
  int df_policy = 1;                 // dataflow scheduling: bit 0 continuations (depth first); bit 1
                                     // successor counters with fence + atomic + fence (default: one acq_rel atomic)
  int df_window = 0;                 // dataflow: tiles in flight ahead of the finished items (0: unbounded)
  int64_t df_big_bytes = 1ll << 30;  // dataflow: programs with at least this many bytes of buffers ...
  int64_t df_big_tile = 64 << 10;    // ... use tiles of at most this many bytes
  int df_waves = 2;                  // dataflow: 1 tile count rounded to whole waves of units; 2 also
                                     // one-wave tiles for reducing chain programs (plan_launch)
  int64_t df_wave_min_tile = 4 << 10;  // ... down to this tile size
  int df_wave_max_lanes = 16;          // ... for programs whose static-lane plan has fewer lanes
  int remote = 1;                    // direct / pulled messages to ranks of other launches through
                                     // registered user buffers (exchange_buffers); 0: FIFO only
  int tma_remote = 0;                // bulk copies on thread blocks with a cross-GPU connection
  int force_sys = 0;                 // testing: treat other launches' ranks as other GPUs (DevTb::sys)
};

Config config_from_env() {
  Config c;
  c.slots = static_cast<int>(env_int("GC3_SLOTS", c.slots));
  c.slot_bytes = env_int("GC3_SLOT_BYTES", c.slot_bytes);
  c.max_lanes = static_cast<int>(env_int("GC3_MAX_LANES", c.max_lanes));
  c.lanes = static_cast<int>(env_int("GC3_LANES", c.lanes));
  c.tile_bytes = env_int("GC3_TILE_BYTES", c.tile_bytes);
  c.timeout_ms = env_int("GC3_TIMEOUT_MS", c.timeout_ms);
  c.trace = static_cast<int>(env_int("GC3_TRACE", 0));
  c.direct = static_cast<int>(env_int("GC3_DIRECT", c.direct));
  c.source = static_cast<int>(env_int("GC3_SOURCE", c.source));
  c.unit_warps = static_cast<int>(env_int("GC3_UNIT_WARPS", c.unit_warps));
  c.group = static_cast<int>(env_int("GC3_GROUP", c.group));
  c.tma = static_cast<int>(env_int("GC3_TMA", c.tma));
  c.balance = static_cast<int>(env_int("GC3_BALANCE", c.balance));
  c.mult_cap = static_cast<int>(env_int("GC3_MULT_CAP", c.mult_cap));
  c.taper = static_cast<int>(env_int("GC3_TAPER", c.taper));
  c.l2hint = static_cast<int>(env_int("GC3_L2HINT", c.l2hint));
  c.wq = static_cast<int>(env_int("GC3_WQ", c.wq));
  c.tma_min = env_int("GC3_TMA_MIN", c.tma_min);
  c.ll_max_bytes = env_int("GC3_LL_MAX_BYTES", c.ll_max_bytes);
  c.ll128_max_bytes = env_int("GC3_LL128_MAX_BYTES", c.ll128_max_bytes);
  c.ll_wide_tbs = static_cast<int>(env_int("GC3_LL_WIDE_TBS", c.ll_wide_tbs));
  c.ll_narrow_max_bytes = env_int("GC3_LL_NARROW_MAX_BYTES", c.ll_narrow_max_bytes);
  c.builtin = static_cast<int>(env_int("GC3_BUILTIN", c.builtin));
  c.clip = static_cast<int>(env_int("GC3_CLIP", c.clip));
  c.gen = static_cast<int>(env_int("GC3_GEN", c.gen));
  c.gen_small = env_int("GC3_GEN_SMALL", c.gen_small);
  c.gen_large = env_int("GC3_GEN_LARGE", c.gen_large);
  c.gen_ll128 = env_int("GC3_GEN_LL128", c.gen_ll128);
  c.smem_kb = env_int("GC3_SMEM_KB", c.smem_kb);
  c.select = static_cast<int>(env_int("GC3_SELECT", c.select));
  c.stage_kb = env_int("GC3_STAGE_KB", c.stage_kb);
  c.wq_items = static_cast<int>(env_int("GC3_WQ_ITEMS", c.wq_items));
  c.wq_lag = static_cast<int>(env_int("GC3_WQ_LAG", c.wq_lag));
  c.discard = static_cast<int>(env_int("GC3_DISCARD", c.discard));
  c.df = static_cast<int>(env_int("GC3_DF", c.df));
  c.df_items = static_cast<int>(env_int("GC3_DF_ITEMS", c.df_items));
  c.df_max_tile = env_int("GC3_DF_MAX_TILE", c.df_max_tile);
  c.df_min_tile = env_int("GC3_DF_MIN_TILE", c.df_min_tile);
  c.df_waves = static_cast<int>(env_int("GC3_DF_WAVES", c.df_waves));
  c.df_wave_min_tile = env_int("GC3_DF_WAVE_MIN_TILE", c.df_wave_min_tile);
  c.df_wave_max_lanes = static_cast<int>(env_int("GC3_DF_WAVE_MAX_LANES", c.df_wave_max_lanes));
  c.remote = static_cast<int>(env_int("GC3_REMOTE", c.remote));
  c.df_policy = static_cast<int>(env_int("GC3_DF_POLICY", c.df_policy));
  c.df_window = static_cast<int>(env_int("GC3_DF_WINDOW", c.df_window));
  c.df_big_bytes = env_int("GC3_DF_BIG_BYTES", c.df_big_bytes);
  c.df_big_tile = env_int("GC3_DF_BIG_TILE", c.df_big_tile);
  c.tma_remote = static_cast<int>(env_int("GC3_TMA_REMOTE", c.tma_remote));
  c.force_sys = static_cast<int>(env_int("GC3_FORCE_SYS", c.force_sys));
  return c;
}

size_t dtype_size(int dt) {
  switch (dt) {
    case ncclInt8: case ncclUint8: case ncclFloat8e4m3: case ncclFloat8e5m2: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
    default: return 0;
  }
}

// ------------------------------------------------------------------------------- bootstrap
// Single-node rendezvous through /dev/shm: the unique id names a directory; every rank posts
// small records (atomic write + rename) and polls for its peers' records.
std::string uid_key(const ncclUniqueId& id) {
  static const char* hex = "0123456789abcdef";
  std::string s;
  for (int i = 4; i < 20; ++i) {
    const unsigned char c = static_cast<unsigned char>(id.internal[i]);
    s += hex[c >> 4];
    s += hex[c & 15];
  }
  return s;
}

std::string shm_dir(const std::string& key) { return "/dev/shm/gc3-" + key; }

bool post_record(const std::string& dir, const std::string& name, const std::string& data) {
  mkdir(dir.c_str(), 0700);
  const std::string tmp = dir + "/." + name + ".tmp" + std::to_string(getpid());
  {
    std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
    if (!f) return false;
    f.write(data.data(), static_cast<std::streamsize>(data.size()));
  }
  return std::rename(tmp.c_str(), (dir + "/" + name).c_str()) == 0;
}

bool read_record(const std::string& dir, const std::string& name, std::string& out, int64_t timeout_ms) {
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms);
  for (;;) {
    std::ifstream f(dir + "/" + name, std::ios::binary);
    if (f) {
      std::ostringstream ss;
      ss << f.rdbuf();
      out = ss.str();
      return true;
    }
    if (std::chrono::steady_clock::now() > deadline) return false;
    std::this_thread::sleep_for(std::chrono::milliseconds(1));
  }
}

// ------------------------------------------------------------------------------- structures
using Comm = ::gc3Comm;  // the opaque ncclComm_t of gc3.h

// Arena layout of one rank for one program. Every rank can compute any peer's layout from the
// shared program text, so a sender addresses the receiver's FIFO without extra exchange.
constexpr size_t kCounterStride = 64;
size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct ArenaLayout {
  std::vector<int> in_index, out_index;  // per tb: index among receiving / sending tbs, or -1
  std::vector<size_t> fifo_off[kNumProtos];      // per protocol, per receiving tb: offset of its FIFOs (lanes x slots)
  std::vector<int64_t> slot_stride[kNumProtos];  // per protocol, per receiving tb: bytes of one slot = unit x max count
  std::vector<int> in_lane_base;         // per receiving tb: index of its first lane's head / counter
  std::vector<int> out_lane_base;        // per sending tb: index of its first lane's tail / counter
  int n_in = 0, n_out = 0;
  size_t off_head = 0, off_tail = 0, off_mine_in = 0, off_mine_out = 0, bytes = 0;
};

// Slot unit (bytes of one tile's message) per protocol for a Simple unit of `unit` bytes: Simple
// and LL128 slots hold `unit` bytes (LL128: unit / 128 lines of 120 payload bytes), LL slots hold
// unit / 2 bytes of 16-byte lines (unit / 4 payload bytes: LL is for small messages).
int64_t proto_unit(int proto, int64_t unit) { return proto == kProtoLL ? std::max<int64_t>(unit / 2 / 256 * 256, 256) : unit; }

// FIFO slots are sized per connection: one slot holds a message of `count` tiles, each at most
// `unit` bytes, so the tile size does not shrink with the aggregation count.
// Every protocol has its own slots (a line protocol must never read another protocol's payload as
// flags). Thread block t of `rank` runs lanes x mult[rank][t] lanes (work balance, see
// lane_multipliers); `lane_base` gives each receiving / sending thread block's first lane in the
// counter arrays.
ArenaLayout make_layout(const Program& p, int rank, int lanes, int slots, int64_t unit, const std::vector<std::vector<int>>& mult) {
  ArenaLayout a;
  const Gpu& g = p.gpus[rank];
  a.in_index.assign(g.tbs.size(), -1);
  a.out_index.assign(g.tbs.size(), -1);
  size_t off = 0;
  int in_lanes = 0, out_lanes = 0;
  for (size_t t = 0; t < g.tbs.size(); ++t) {
    const int lt = lanes * (mult.empty() ? 1 : mult[rank][t]);
    if (g.tbs[t].recv_peer >= 0) {
      a.in_index[t] = a.n_in++;
      int maxc = 1;
      for (const Op& op : g.tbs[t].ops)
        if (op_receives(op.op)) maxc = std::max(maxc, op.count);
      for (int pr = 0; pr < kNumProtos; ++pr) {
        const int64_t u = proto_unit(pr, unit);
        a.fifo_off[pr].push_back(off);
        a.slot_stride[pr].push_back(u * maxc);
        off += static_cast<size_t>(lt) * slots * u * maxc;
      }
      a.in_lane_base.push_back(in_lanes);
      in_lanes += lt;
    }
    if (g.tbs[t].send_peer >= 0) {
      a.out_index[t] = a.n_out++;
      a.out_lane_base.push_back(out_lanes);
      out_lanes += lt;
    }
  }
  off = align_up(off, 256);
  a.off_head = off;
  off += static_cast<size_t>(in_lanes) * kCounterStride;
  a.off_tail = off;
  off += static_cast<size_t>(out_lanes) * kCounterStride;
  a.off_mine_in = off;
  off += static_cast<size_t>(in_lanes) * 8;
  a.off_mine_out = off;
  off += static_cast<size_t>(out_lanes) * 8;
  a.bytes = align_up(std::max<size_t>(off, 256), 256);
  return a;
}

// One registered program on one rank: the (possibly replicated) IR plus its arena.
struct RankIR {
  Program prog;
  int proto_override = -1;
  int slots = 2;
  int64_t slot_bytes = 0;
  int lanes = 1;  // lanes provisioned in the arena
  bool has_reduce = false;
  bool has_chain = false;  // an op both receives and sends (rcs / rrcs / rrs): multi-hop chains
  bool clip_ok = false;    // AllReduce whose ops each move one chunk in place and whose messages land
                           // in the chunk they left: ragged calls run on the caller's buffer
                           // (LaunchArgs::clip_elems) instead of padded work buffers
  uint8_t lane_mask = 0;   // transports assumed by the lane multipliers (transport_mask)
  bool builtin = false;    // registered by the runtime (builtin_program), selected after user IRs
  std::map<int64_t, double> predicted;  // timed-model microseconds per chunk size (config "select")
  int max_count = 1;
  std::vector<std::vector<int>> mult;  // lane multiplier per (rank, tb) (lane_multipliers)
  ArenaLayout lay;
  std::vector<std::vector<std::vector<uint8_t>>> eff_direct;     // direct flags of this device's launch
  std::map<std::tuple<int64_t, int, int, int, bool>, bool> order_ok;  // (tiles, lanes, group, slots, ll) -> deadlock-free
  char* arena = nullptr;
  cudaIpcMemHandle_t handle{};
};

// Per-device execution state shared by the ranks a clique hosts on that device.
struct DevicePlan {  // one registered IR on one device
  bool built = false;
  bool wq_ok = false;  // work-queue mode possible (no FIFO message, one launch)
  std::vector<int> wq_level;  // per launch thread block: 1 + max level of the thread blocks its deps name
  std::map<std::pair<int64_t, int>, int32_t*> wq_order;  // (ntiles, lag) -> device claim-order table
  bool source_complete = false;  // every first read of `input` reads the source buffer (source_reads)
  bool result_complete = false;  // ReduceScatter owned blocks are written straight to recvbuff (result_writes)
  std::vector<int> ranks;  // local ranks in launch order (rank_slot -> rank)
  int ntbs = 0;
  int weight = 0;          // sum of lane multipliers: units = lanes x weight
  DevTb* d_tbs = nullptr;
  DevOp* d_ops = nullptr;
  DevDep* d_deps = nullptr;
  DevChan* d_chans = nullptr;
  uint64_t* d_sems = nullptr;
  bool sys_scope = false;     // some thread block has a connection to another GPU (DevTb::sys)
  std::vector<int> remote_ranks;  // ranks of other launches with buffer slots (remote transports)
  int remote_msgs = 0;            // direct / pulled receives of this launch whose sender is remote
  // dataflow graph (every rank of the program in this launch): nodes in launch op order
  bool df_ok = false;
  int df_n = 0, df_nroots = 0, df_mail_msgs = 0, df_depth = 1;
  int64_t df_mail_chunks = 0;  // mailbox size in chunks
  DfNode* d_df_nodes = nullptr;
  DfSucc* d_df_succ = nullptr;
  int32_t* d_df_roots = nullptr;
};

struct DeviceState {
  int device = -1;
  uint64_t epoch = 0;
  uint64_t* d_epoch = nullptr;     // device-side launch counter (LaunchArgs::epoch_ptr)
  int32_t* d_epoch_ctr = nullptr;  // blocks that have read it in the current launch
  int32_t* d_abort = nullptr;
  uint64_t* h_err = nullptr;  // host-mapped err_info[8]
  uint64_t* d_err = nullptr;
  std::vector<DevicePlan> plans;  // by ir id
  int num_sms = 0;
  std::map<std::pair<KernelFn, size_t>, int> occupancy;  // (kernel, dynamic smem) -> blocks per SM
  uint64_t* d_trace = nullptr;  // event log of the last traced launch
  size_t trace_bytes = 0;
  int32_t* d_df_cnt = nullptr;   // dataflow predecessor counters [tile][node] (self-resetting)
  int32_t* d_df_q = nullptr;     // dataflow ready queue (self-resetting)
  size_t df_items_cap = 0;       // entries of d_df_cnt / d_df_q
  char* d_mail = nullptr;        // dataflow mailbox
  size_t mail_bytes = 0;
  int32_t* d_wq_next = nullptr;  // work-queue claim counter
  uint64_t* d_prog = nullptr;    // work-queue progress table
  size_t prog_bytes = 0;
  int trace_grid = 0, trace_ops = 0, trace_lanes = 0;
  // every launch of this device waits for the previous one: launches share FIFO counters, scratch,
  // work buffers and the work-queue tables, so collectives issued on different streams must not
  // overlap (NCCL orders a communicator's kernels the same way)
  cudaEvent_t last_done = nullptr;
  cudaEvent_t launch_done = nullptr;                    // joins the other participating streams after a launch
  std::map<cudaStream_t, cudaEvent_t> stream_events;    // per participating stream, created once
  cudaStream_t last_stream = nullptr;
  bool has_last = false;
};

struct Clique {
  std::string key;
  int nranks = 0;
  std::vector<Comm*> local;   // by rank, nullptr when the rank lives in another process
  std::vector<int> rank_dev;  // device of every rank (exchanged at init)
  std::vector<int> rank_pid;
  std::map<int, DeviceState> devs;
  int refs = 0;
  std::vector<std::string> rank_uuid;  // GPU of every rank (UUID; read from the bootstrap records on demand)
  char* calls = nullptr;               // shared-memory call-descriptor table (remote transports)
  size_t calls_bytes = 0;
};

}  // namespace
}  // namespace gc3

struct gc3Comm {
  gc3::Clique* clique = nullptr;
  int rank = 0;
  int nranks = 0;
  int device = 0;
  gc3::Config cfg;
  std::vector<std::unique_ptr<gc3::RankIR>> irs;
  // peer arena base pointers per ir: [ir][rank]
  std::vector<std::vector<char*>> peer_arena;
  char* scratch = nullptr;
  size_t scratch_bytes = 0;
  char* work = nullptr;  // ReduceScatter working buffer; padded input block(s) of ragged calls
  size_t work_bytes = 0;
  char* work2 = nullptr;  // padded output blocks of ragged AllGather / AlltoAll calls
  size_t work2_bytes = 0;
  ncclResult_t async_error = ncclSuccess;
  std::string last_error;
  bool destroyed = false;
  std::vector<void*> opened_ipc;  // peer arenas opened via IPC (to close)
  // user-buffer registration (remote direct / pulled messages): allocations this rank exported
  // (driver buffer id -> registration), peers' registrations opened here ((rank, id) -> base)
  struct Reg {
    uint64_t buffer_id;
    uintptr_t base;
    size_t size;
  };
  std::vector<Reg> regs;
  std::map<std::pair<int, int>, char*> peer_regs;
  uint64_t xcall_seq = 0;  // calls whose buffers were exchanged with other launches
};

namespace gc3 {
namespace {

std::map<std::string, std::unique_ptr<Clique>> g_cliques;

// ------------------------------------------------------------------------------- groups
enum Coll { kAllReduce = 0, kAllGather = 1, kReduceScatter = 2, kAllToAll = 3 };
const char* coll_name(int c) {
  static const char* n[] = {"allreduce", "allgather", "reducescatter", "alltoall"};
  return n[c];
}

struct Pending {
  Comm* comm;
  int coll;
  const void* send;
  void* recv;
  size_t count;
  int dtype;
  int redop;
  cudaStream_t stream;
};

thread_local int g_group_depth = 0;
thread_local std::vector<Pending> g_pending;

// ------------------------------------------------------------------------------- helpers
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

ncclResult_t device_state(Clique* cl, int dev, DeviceState*& out) {
  auto it = cl->devs.find(dev);
  if (it != cl->devs.end()) {
    out = &it->second;
    return ncclSuccess;
  }
  DeviceState& ds = cl->devs[dev];
  ds.device = dev;
  DeviceGuard g(dev);
  CUDA_TRY(cudaMalloc(&ds.d_abort, sizeof(int32_t)));
  CUDA_TRY(cudaMemset(ds.d_abort, 0, sizeof(int32_t)));
  {
    CUDA_TRY(cudaMalloc(&ds.d_epoch, 256));
    const uint64_t one = 1;
    CUDA_TRY(cudaMemset(ds.d_epoch, 0, 256));
    CUDA_TRY(cudaMemcpy(ds.d_epoch, &one, sizeof(one), cudaMemcpyHostToDevice));
    ds.d_epoch_ctr = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ds.d_epoch) + 128);
  }
  CUDA_TRY(cudaHostAlloc(&ds.h_err, 8 * sizeof(uint64_t), cudaHostAllocMapped));
  std::memset(ds.h_err, 0, 8 * sizeof(uint64_t));
  CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ds.d_err), ds.h_err, 0));
  CUDA_TRY(cudaDeviceGetAttribute(&ds.num_sms, cudaDevAttrMultiProcessorCount, dev));
  out = &ds;
  return ncclSuccess;
}

// Reads a file or treats the argument as JSON text.
bool read_ir_text(const char* arg, std::string& text) {
  const char* p = arg;
  while (*p == ' ' || *p == '\n' || *p == '\t' || *p == '\r') ++p;
  if (*p == '{' || *p == '<') {  // GC3-IR JSON or MSCCL XML text
    text = arg;
    return true;
  }
  std::ifstream f(arg, std::ios::binary);
  if (!f) return false;
  std::ostringstream ss;
  ss << f.rdbuf();
  text = ss.str();
  return true;
}

// Receiver of connection (src -> dst, ch) as a tb index on dst (last match, as validate()).
int find_receiver(const Program& p, int src, int dst, int ch) {
  int found = -1;
  const auto& tbs = p.gpus[dst].tbs;
  for (size_t t = 0; t < tbs.size(); ++t)
    if (tbs[t].recv_peer == src && tbs[t].channel == ch) found = static_cast<int>(t);
  return found;
}
int find_sender(const Program& p, int src, int dst, int ch) {
  int found = -1;
  const auto& tbs = p.gpus[src].tbs;
  for (size_t t = 0; t < tbs.size(); ++t)
    if (tbs[t].send_peer == dst && tbs[t].channel == ch) found = static_cast<int>(t);
  return found;
}

int tb_index(const Program& p, int rank, int id) {
  const auto& tbs = p.gpus[rank].tbs;
  for (size_t t = 0; t < tbs.size(); ++t)
    if (tbs[t].id == id) return static_cast<int>(t);
  return -1;
}

// Resolves (and caches) the base pointer of rank `r`'s arena for ir `id` as seen from `c`.
ncclResult_t peer_arena(Comm* c, int id, int r, char*& out) {
  if (c->peer_arena.size() <= static_cast<size_t>(id)) c->peer_arena.resize(id + 1);
  auto& v = c->peer_arena[id];
  if (v.size() != static_cast<size_t>(c->nranks)) v.assign(c->nranks, nullptr);
  if (v[r]) {
    out = v[r];
    return ncclSuccess;
  }
  Clique* cl = c->clique;
  if (cl->local[r]) {  // same process: direct pointer (peer access enabled at init when needed)
    Comm* pc = cl->local[r];
    if (pc->irs.size() <= static_cast<size_t>(id))
      return set_error(ncclInvalidUsage, "rank %d has not registered IR %d yet (register on all local ranks before launching)", r, id);
    v[r] = pc->irs[id]->arena;
  } else {
    std::string rec;
    const std::string name = "ir" + std::to_string(id) + ".rank" + std::to_string(r);
    if (!read_record(shm_dir(cl->key), name, rec, c->cfg.timeout_ms + 60000))
      return set_error(ncclSystemError, "timed out waiting for rank %d's IR %d arena handle", r, id);
    if (rec.size() < sizeof(cudaIpcMemHandle_t)) return set_error(ncclSystemError, "bad arena record from rank %d", r);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, rec.data(), sizeof(h));
    DeviceGuard g(c->device);
    void* p = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->opened_ipc.push_back(p);
    v[r] = static_cast<char*>(p);
  }
  out = v[r];
  return ncclSuccess;
}

// ------------------------------------------------------------------------------- GPU identity
std::string device_bus_id(int dev) {
  char buf[64] = {0};
  if (cudaDeviceGetPCIBusId(buf, sizeof(buf), dev) != cudaSuccess) return "dev" + std::to_string(dev);
  return buf;
}

// PCI bus id of rank r's GPU (device ordinals differ across processes with CUDA_VISIBLE_DEVICES)
ncclResult_t rank_gpu(Comm* c, int r, std::string& out) {
  Clique* cl = c->clique;
  if (cl->rank_uuid.size() != static_cast<size_t>(cl->nranks)) cl->rank_uuid.assign(cl->nranks, "");
  if (cl->rank_uuid[r].empty()) {
    if (cl->local[r]) {
      cl->rank_uuid[r] = device_bus_id(cl->local[r]->device);
    } else {
      std::string rec;
      if (!read_record(shm_dir(cl->key), "rank" + std::to_string(r), rec, c->cfg.timeout_ms + 60000))
        return set_error(ncclSystemError, "timed out waiting for rank %d's bootstrap record", r);
      std::istringstream in(rec);
      long pid = 0;
      int dev = -1;
      std::string bus;
      in >> pid >> dev >> bus;
      cl->rank_uuid[r] = bus.empty() ? "pid" + std::to_string(pid) + "dev" + std::to_string(dev) : bus;
    }
  }
  out = cl->rank_uuid[r];
  return ncclSuccess;
}

// Process id of rank r (from its bootstrap record when it lives in another process).
ncclResult_t rank_pid(Comm* c, int r, long& out) {
  Clique* cl = c->clique;
  if (cl->local[r]) {
    out = static_cast<long>(getpid());
    return ncclSuccess;
  }
  std::string rec;
  if (!read_record(shm_dir(cl->key), "rank" + std::to_string(r), rec, c->cfg.timeout_ms + 60000))
    return set_error(ncclSystemError, "timed out waiting for rank %d's bootstrap record", r);
  std::istringstream in(rec);
  in >> out;
  return ncclSuccess;
}

// ------------------------------------------------------------------------------- user buffers
// Direct and pulled messages between ranks of different launches (other processes or GPUs) address
// the peer's user buffers. As with NCCL user-buffer registration, every allocation a collective
// touches is exported once (cudaIpcGetMemHandle of the allocation's base, keyed by the driver's
// process-wide unique buffer id, so a freed and re-allocated range is never taken for the old one)
// and opened once by each peer process that addresses it; per call, the ranks exchange
// (registration, offset) descriptors through a shared-memory table (exchange_buffers).
using CuPointerGetAttributeFn = int (*)(void*, int, unsigned long long);
CuPointerGetAttributeFn cu_pointer_get_attribute() {
  static CuPointerGetAttributeFn fn = [] {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libcuda.so.1", RTLD_NOW);
    return h ? reinterpret_cast<CuPointerGetAttributeFn>(dlsym(h, "cuPointerGetAttribute")) : nullptr;
  }();
  return fn;
}

// Registration id and offset of device pointer p (exports its allocation on first use).
ncclResult_t export_buffer(Comm* c, const void* p, int32_t& id, int64_t& off) {
  id = -1;
  off = 0;
  if (!p) return ncclSuccess;
  CuPointerGetAttributeFn fn = cu_pointer_get_attribute();
  if (!fn) return set_error(ncclSystemError, "cuPointerGetAttribute unavailable (libcuda.so.1)");
  const auto ptr = static_cast<unsigned long long>(reinterpret_cast<uintptr_t>(p));
  unsigned long long bid = 0, base = 0;
  size_t size = 0;
  if (fn(&bid, 7 /* CU_POINTER_ATTRIBUTE_BUFFER_ID */, ptr) || fn(&base, 11 /* RANGE_START_ADDR */, ptr) ||
      fn(&size, 12 /* RANGE_SIZE */, ptr))
    return set_error(ncclInvalidArgument, "buffer %p is not device memory the driver knows", p);
  for (size_t i = 0; i < c->regs.size(); ++i)
    if (c->regs[i].buffer_id == bid) {
      id = static_cast<int32_t>(i);
      off = static_cast<int64_t>(ptr - c->regs[i].base);
      return ncclSuccess;
    }
  cudaIpcMemHandle_t h{};
  {
    DeviceGuard g(c->device);
    CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(static_cast<uintptr_t>(base))));
  }
  id = static_cast<int32_t>(c->regs.size());
  std::string rec(reinterpret_cast<const char*>(&h), sizeof(h));
  rec.append(reinterpret_cast<const char*>(&base), sizeof(base));
  rec.append(reinterpret_cast<const char*>(&size), sizeof(size));
  if (!post_record(shm_dir(c->clique->key), "buf" + std::to_string(c->rank) + "." + std::to_string(id), rec))
    return set_error(ncclSystemError, "cannot post the buffer registration record");
  c->regs.push_back({bid, static_cast<uintptr_t>(base), size});
  off = static_cast<int64_t>(ptr - base);
  return ncclSuccess;
}

// Base address, in this process, of rank r's registration `id` (opened on first use).
ncclResult_t peer_buffer(Comm* c, int r, int32_t id, char*& out) {
  out = nullptr;
  if (id < 0) return ncclSuccess;
  Clique* cl = c->clique;
  if (cl->local[r]) {  // same process: the exporter's own pointer (unified addressing)
    if (static_cast<size_t>(id) >= cl->local[r]->regs.size()) return set_error(ncclInternalError, "unknown registration");
    out = reinterpret_cast<char*>(cl->local[r]->regs[id].base);
    return ncclSuccess;
  }
  auto f = c->peer_regs.find({r, id});
  if (f != c->peer_regs.end()) {
    out = f->second;
    return ncclSuccess;
  }
  std::string rec;
  if (!read_record(shm_dir(cl->key), "buf" + std::to_string(r) + "." + std::to_string(id), rec, c->cfg.timeout_ms + 60000) ||
      rec.size() < sizeof(cudaIpcMemHandle_t))
    return set_error(ncclSystemError, "rank %d's buffer registration %d is missing", r, id);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, rec.data(), sizeof(h));
  void* p = nullptr;
  DeviceGuard g(c->device);
  CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  c->opened_ipc.push_back(p);
  out = static_cast<char*>(p);
  c->peer_regs[{r, id}] = out;
  return ncclSuccess;
}

// Call-descriptor table: one ring of kCallRing records per rank in a shared-memory file of the
// clique. Record (rank, seq % kCallRing) holds the registration and offset of each of the rank's
// launch buffers for its seq-th exchanged call; `done` is the last seq for which the rank has read
// every peer record it needs (a writer never laps a reader: it waits for done >= seq - kCallRing).
constexpr int kCallRing = 64;
struct CallRec {
  std::atomic<uint64_t> seq;
  int32_t reg[kBufs];
  int32_t pad;
  int64_t off[kBufs];
};
struct CallRank {
  std::atomic<uint64_t> done;
  char pad[56];
  CallRec rec[kCallRing];
};

ncclResult_t call_table(Comm* c, CallRank*& out) {
  Clique* cl = c->clique;
  if (!cl->calls) {
    const std::string dir = shm_dir(cl->key);
    mkdir(dir.c_str(), 0700);
    const std::string path = dir + "/calls";
    const size_t bytes = sizeof(CallRank) * static_cast<size_t>(cl->nranks);
    const int fd = open(path.c_str(), O_RDWR | O_CREAT, 0600);
    if (fd < 0) return set_error(ncclSystemError, "cannot open %s", path.c_str());
    if (ftruncate(fd, static_cast<off_t>(bytes)) != 0) {
      close(fd);
      return set_error(ncclSystemError, "cannot size %s", path.c_str());
    }
    void* m = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) return set_error(ncclSystemError, "cannot map %s", path.c_str());
    cl->calls = static_cast<char*>(m);
    cl->calls_bytes = bytes;
  }
  out = reinterpret_cast<CallRank*>(cl->calls);
  return ncclSuccess;
}

bool spin_until(const std::function<bool()>& ok, int64_t timeout_ms) {
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms);
  for (int i = 0; !ok(); ++i) {
    if (i > 64) std::this_thread::yield();
    if ((i & 1023) == 1023 && std::chrono::steady_clock::now() > deadline) return false;
  }
  return true;
}

// Message transports, decided statically from the happens-before relation of the program:
// sequential execution, declared deps and the k-th send -> k-th receive matching (the graph of
// scheduler.hpp:652-717). An edge a -> b means a's data movement is finished before b's starts.
//
// Direct (kInDirect / kOutDirect). A receive that only stores the message (recv, rcs) may have it
// written by the sender straight into the receive's local span x when every other access of x on
// the receiving rank is ordered with that write: before the send, or after the receive. The sender
// addresses x through its own op's dst fields (lowering.hpp:71), which must name it exactly.
//
// Pull (kInPull / kOutPull). A message whose content is a span Y the sender stores (send reads Y;
// rcs and rrcs write the message to Y) may stay there: the receive reads Y from the sender's
// buffers once the sender has published it, provided every write to Y on the sending rank is
// ordered with that window: before the send, or after the receive. This removes the FIFO round trip
// of reducing receives (rrc, rrcs, rrs), which can never be direct.
//
// A receive op u that writes a span (recv, rcs) may have its data written at its sender's op x(u)
// (if that message is direct), so "after the receive" is checked at both u and x(u).
// Returns flags[rank][tb index][step]; pull_src (optional) gets the sender span (buf, off) of
// every kInPull receive.
struct PullSrc {  // the sending op of a pulled message and the span it stores the message in
  int buf = -1, off = -1, rank = -1, tb = -1, step = -1;
};

// Happens-before graph over every op of every rank: sequential order, declared deps and the k-th
// send -> k-th receive message edges (the graph of scheduler.hpp:652-717), with its transitive
// closure. ok == false when connections are unbalanced or the graph has a cycle.
struct HbGraph {
  struct Ref {
    int rank, tb, step;
  };
  bool ok = false;
  int n = 0;
  std::vector<std::vector<int>> base;  // node index of (rank, tb, 0)
  std::vector<int> sender_of;          // receive node -> matched send node
  std::map<std::tuple<int, int, int>, std::pair<std::vector<Ref>, std::vector<Ref>>> conns;  // (src, dst, ch)
  size_t words = 0;
  std::vector<uint64_t> reach;
  bool reaches(int a, int b) const { return (reach[static_cast<size_t>(a) * words + b / 64] >> (b % 64)) & 1; }
  int node(int r, int t, int s) const { return base[r][t] + s; }

  explicit HbGraph(const Program& p) {
    const int R = p.ranks();
    base.resize(R);
    for (int r = 0; r < R; ++r)
      for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) {
        base[r].push_back(n);
        n += static_cast<int>(p.gpus[r].tbs[t].ops.size());
      }
    if (n == 0 || n > 65536) return;
    std::vector<std::vector<int>> succ(n);
    for (int r = 0; r < R; ++r)
      for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) {
        const ThreadBlock& tb = p.gpus[r].tbs[t];
        for (size_t s = 0; s < tb.ops.size(); ++s) {
          const int u = base[r][t] + static_cast<int>(s);
          if (s + 1 < tb.ops.size()) succ[u].push_back(u + 1);
          for (const Dep& d : tb.ops[s].deps) {
            const int ti = tb_index(p, r, d.tb);
            if (ti >= 0 && d.step >= 0 && d.step < static_cast<int>(p.gpus[r].tbs[ti].ops.size())) succ[base[r][ti] + d.step].push_back(u);
          }
          if (op_sends(tb.ops[s].op) && tb.send_peer >= 0) conns[{r, tb.send_peer, tb.channel}].first.push_back({r, static_cast<int>(t), static_cast<int>(s)});
          if (op_receives(tb.ops[s].op) && tb.recv_peer >= 0) conns[{tb.recv_peer, r, tb.channel}].second.push_back({r, static_cast<int>(t), static_cast<int>(s)});
        }
      }
    sender_of.assign(n, -1);
    for (auto& [key, c] : conns) {
      if (c.first.size() != c.second.size()) return;  // unbalanced
      for (size_t k = 0; k < c.first.size(); ++k) {
        const int su = base[c.first[k].rank][c.first[k].tb] + c.first[k].step;
        const int ru = base[c.second[k].rank][c.second[k].tb] + c.second[k].step;
        succ[su].push_back(ru);
        sender_of[ru] = su;
      }
    }
    std::vector<int> indeg(n, 0), order;
    for (int u = 0; u < n; ++u)
      for (int v : succ[u]) ++indeg[v];
    for (int u = 0; u < n; ++u)
      if (!indeg[u]) order.push_back(u);
    for (size_t i = 0; i < order.size(); ++i)
      for (int v : succ[order[i]])
        if (--indeg[v] == 0) order.push_back(v);
    if (static_cast<int>(order.size()) != n) return;  // cycle: no static order
    words = (n + 63) / 64;
    reach.assign(static_cast<size_t>(n) * words, 0);
    for (auto it = order.rbegin(); it != order.rend(); ++it) {
      uint64_t* ru = &reach[static_cast<size_t>(*it) * words];
      ru[*it / 64] |= 1ull << (*it % 64);
      for (int v : succ[*it])
        for (size_t w = 0; w < words; ++w) ru[w] |= reach[static_cast<size_t>(v) * words + w];
    }
    ok = true;
  }
};

// The sending op of every receive (k-th send -> k-th receive per connection, scheduler.hpp:251-273);
// rank -1 where unmatched.
std::vector<std::vector<std::vector<HbGraph::Ref>>> matched_senders(const Program& p) {
  std::vector<std::vector<std::vector<HbGraph::Ref>>> out(p.ranks());
  std::map<std::tuple<int, int, int>, std::pair<std::vector<HbGraph::Ref>, std::vector<HbGraph::Ref>>> conns;
  for (int r = 0; r < p.ranks(); ++r) {
    out[r].resize(p.gpus[r].tbs.size());
    for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) {
      const ThreadBlock& tb = p.gpus[r].tbs[t];
      out[r][t].assign(tb.ops.size(), HbGraph::Ref{-1, -1, -1});
      for (size_t s = 0; s < tb.ops.size(); ++s) {
        if (op_sends(tb.ops[s].op) && tb.send_peer >= 0) conns[{r, tb.send_peer, tb.channel}].first.push_back({r, static_cast<int>(t), static_cast<int>(s)});
        if (op_receives(tb.ops[s].op) && tb.recv_peer >= 0) conns[{tb.recv_peer, r, tb.channel}].second.push_back({r, static_cast<int>(t), static_cast<int>(s)});
      }
    }
  }
  for (auto& [key, c] : conns)
    for (size_t k = 0; k < c.second.size() && k < c.first.size(); ++k) out[c.second[k].rank][c.second[k].tb][c.second[k].step] = c.first[k];
  return out;
}

// Receive-side transport mask a launch applies when every rank of the program runs in it (all
// loopback ranks on one device): direct (config bit 0) and pulled (bit 1) messages.
uint8_t transport_mask(int direct_cfg) {
  uint8_t m = 0;
  if (direct_cfg & 1) m |= kInDirect | kOutDirect;
  if (direct_cfg & 2) m |= kInPull | kOutPull;
  return m;
}

std::vector<std::vector<std::vector<uint8_t>>> direct_messages(
    const Program& p, bool pull, std::vector<std::vector<std::vector<PullSrc>>>* pull_src) {
  const int R = p.ranks();
  std::vector<std::vector<std::vector<uint8_t>>> flags(R);
  for (int r = 0; r < R; ++r) {
    flags[r].resize(p.gpus[r].tbs.size());
    for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) flags[r][t].assign(p.gpus[r].tbs[t].ops.size(), 0);
  }
  if (pull_src) {
    pull_src->assign(R, {});
    for (int r = 0; r < R; ++r)
      for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) (*pull_src)[r].emplace_back(p.gpus[r].tbs[t].ops.size(), PullSrc{});
  }
  const HbGraph g(p);
  if (!g.ok) return flags;
  using Ref = HbGraph::Ref;
  const auto& base = g.base;
  const auto& sender_of = g.sender_of;
  auto reaches = [&](int a, int b) { return g.reaches(a, b); };
  auto storage = [&](Buf b) { return p.inplace && b == Buf::output ? Buf::input : b; };
  struct Span {
    Buf b;
    int off, count;
  };
  auto overlaps = [&](const Span& x, const Span& y) {
    return storage(x.b) == storage(y.b) && x.off < y.off + y.count && y.off < x.off + x.count;
  };
  // local reads + writes (lowering.hpp:96-119); writes only with `writes_only`
  auto accesses = [&](const Op& op, bool writes_only, std::vector<Span>& out) {
    out.clear();
    switch (op.op) {
      case Opcode::send: case Opcode::rrs:
        if (!writes_only) out.push_back({op.src_buf, op.src_off, op.count});
        break;
      case Opcode::recv: out.push_back({op.dst_buf, op.dst_off, op.count}); break;
      case Opcode::rcs: case Opcode::rrcs: out.push_back({op.src_buf, op.src_off, op.count}); break;
      case Opcode::copy: case Opcode::reduce: case Opcode::rrc:
        if (!writes_only) out.push_back({op.src_buf, op.src_off, op.count});
        out.push_back({op.dst_buf, op.dst_off, op.count});
        break;
      default: break;
    }
  };
  // is every access u (on `rank`) of span x ordered with the window [send su, receive ru]?
  std::vector<Span> acc;
  auto window_clear = [&](int rank, int self, const Span& x, int su, int ru, bool writes_only) {
    for (size_t t = 0; t < p.gpus[rank].tbs.size(); ++t)
      for (size_t s = 0; s < p.gpus[rank].tbs[t].ops.size(); ++s) {
        const int u = base[rank][t] + static_cast<int>(s);
        if (u == self) continue;
        const Op& op = p.gpus[rank].tbs[t].ops[s];
        accesses(op, writes_only, acc);
        for (const Span& y : acc) {
          if (!overlaps(x, y)) continue;
          if (!reaches(ru, u) && !reaches(u, su)) return false;
          const bool msg_write = (op.op == Opcode::recv || op.op == Opcode::rcs) && sender_of[u] >= 0;
          if (msg_write && !reaches(sender_of[u], su) && !reaches(ru, sender_of[u])) return false;
        }
      }
    return true;
  };
  for (auto& [key, c] : g.conns) {
    for (size_t k = 0; k < c.second.size(); ++k) {
      const Ref rx = c.second[k], tx = c.first[k];
      const Op& rop = p.gpus[rx.rank].tbs[rx.tb].ops[rx.step];
      const Op& sop = p.gpus[tx.rank].tbs[tx.tb].ops[tx.step];
      if (rop.op != Opcode::recv && rop.op != Opcode::rcs) continue;
      const Span x = rop.op == Opcode::recv ? Span{rop.dst_buf, rop.dst_off, rop.count} : Span{rop.src_buf, rop.src_off, rop.count};
      if (storage(sop.dst_buf) != storage(x.b) || sop.dst_off != x.off || sop.count != x.count) continue;
      const int ru = base[rx.rank][rx.tb] + rx.step, su = base[tx.rank][tx.tb] + tx.step;
      if (window_clear(rx.rank, ru, x, su, ru, false)) {
        flags[rx.rank][rx.tb][rx.step] |= kInDirect;
        flags[tx.rank][tx.tb][tx.step] |= kOutDirect;
      }
    }
  }
  if (!pull) return flags;
  for (auto& [key, c] : g.conns) {
    for (size_t k = 0; k < c.second.size(); ++k) {
      const Ref rx = c.second[k], tx = c.first[k];
      if (flags[rx.rank][rx.tb][rx.step] & kInDirect) continue;
      const Op& rop = p.gpus[rx.rank].tbs[rx.tb].ops[rx.step];
      const Op& sop = p.gpus[tx.rank].tbs[tx.tb].ops[tx.step];
      if (sop.op != Opcode::send && sop.op != Opcode::rcs && sop.op != Opcode::rrcs) continue;  // rrs stores nothing
      if (sop.count != rop.count) continue;
      const Span y{sop.src_buf, sop.src_off, sop.count};
      const int ru = base[rx.rank][rx.tb] + rx.step, su = base[tx.rank][tx.tb] + tx.step;
      if (window_clear(tx.rank, su, y, su, ru, true)) {
        flags[rx.rank][rx.tb][rx.step] |= kInPull;
        flags[tx.rank][tx.tb][tx.step] |= kOutPull;
        if (pull_src) (*pull_src)[rx.rank][rx.tb][rx.step] = {static_cast<int>(sop.src_buf), sop.src_off, tx.rank, tx.tb, tx.step};
      }
    }
  }
  return flags;
}

// Reads of the caller's const send buffer (SURVEY.md §7 hard part 6). AllReduce and ReduceScatter
// IRs run in place on `input` (core.hpp:305-327, 351-375), but NCCL's sendbuff is const and usually
// differs from recvbuff. A read of an input span that no write on its rank happens before sees the
// caller's data, so it can read sendbuff itself and the working buffer needs no pre-copy. Returns
// flags[rank][tb][step] (kSrcFromSource: the op's src read; kDstFromSource: reduce's dst read), and
// `complete` = every input read is either remapped or preceded by a write (otherwise the runtime
// keeps the pre-copy).
std::vector<std::vector<std::vector<uint8_t>>> source_reads(const Program& p, bool& complete) {
  const int R = p.ranks();
  std::vector<std::vector<std::vector<uint8_t>>> flags(R);
  for (int r = 0; r < R; ++r) {
    flags[r].resize(p.gpus[r].tbs.size());
    for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) flags[r][t].assign(p.gpus[r].tbs[t].ops.size(), 0);
  }
  complete = false;
  if (!p.inplace || R < 2) return flags;
  const HbGraph g(p);
  if (!g.ok) return flags;
  auto is_input = [&](Buf b) { return b == Buf::input || b == Buf::output; };
  auto writes = [&](const Op& op, int& off, int& cnt) {  // the op's local write span, if any
    switch (op.op) {
      case Opcode::recv: case Opcode::copy: case Opcode::reduce: case Opcode::rrc:
        if (!is_input(op.dst_buf)) return false;
        off = op.dst_off, cnt = op.count;
        return true;
      case Opcode::rcs: case Opcode::rrcs:
        if (!is_input(op.src_buf)) return false;
        off = op.src_off, cnt = op.count;
        return true;
      default: return false;
    }
  };
  // 0: remappable, 1: a write happens before (reads the working buffer), 2: unordered write
  auto classify = [&](int r, int u, int off, int cnt) {
    int verdict = 0;
    for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t)
      for (size_t s = 0; s < p.gpus[r].tbs[t].ops.size(); ++s) {
        const int w = g.node(r, static_cast<int>(t), static_cast<int>(s));
        if (w == u) continue;
        int wo, wc;
        if (!writes(p.gpus[r].tbs[t].ops[s], wo, wc) || !(wo < off + cnt && off < wo + wc)) continue;
        if (g.reaches(w, u)) verdict = std::max(verdict, 1);
        else if (!g.reaches(u, w)) verdict = 2;
      }
    return verdict;
  };
  complete = true;
  for (int r = 0; r < R; ++r)
    for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t)
      for (size_t s = 0; s < p.gpus[r].tbs[t].ops.size(); ++s) {
        const Op& op = p.gpus[r].tbs[t].ops[s];
        const int u = g.node(r, static_cast<int>(t), static_cast<int>(s));
        bool reads_src = false, reads_dst = false;
        switch (op.op) {
          case Opcode::send: case Opcode::copy: case Opcode::rrc: case Opcode::rrcs: case Opcode::rrs: reads_src = true; break;
          case Opcode::reduce: reads_src = reads_dst = true; break;
          default: break;  // recv writes only; rcs reads its span only after writing it (or after a direct write)
        }
        if (reads_src && is_input(op.src_buf)) {
          const int v = classify(r, u, op.src_off, op.count);
          if (v == 0) flags[r][t][s] |= kSrcFromSource;
          if (v == 2) complete = false;
        }
        if (reads_dst && is_input(op.dst_buf)) {
          const int v = classify(r, u, op.dst_off, op.count);
          if (v == 0) flags[r][t][s] |= kDstFromSource;
          if (v == 2) complete = false;
        }
      }
  return flags;
}

// Final writes of a ReduceScatter's owned block straight into recvbuff. The IR is in place over
// R x c chunks and rank r owns [r*c, (r+1)*c) (core.hpp:351-375); the runtime used to copy the owned
// block out of its working buffer after the kernel. A local op (recv / copy / reduce / rrc) that
// writes part of the owned block may write it into the result buffer instead when every other
// write of that span happens before it and every read of it happens before it too (no one reads
// the final value from the working buffer). Returns flags[rank][tb][step] (1 = write to the result
// buffer); `complete` = on every rank such writes cover the whole owned block (the copy is dropped).
std::vector<std::vector<std::vector<uint8_t>>> result_writes(const Program& p, bool& complete) {
  const int R = p.ranks();
  std::vector<std::vector<std::vector<uint8_t>>> flags(R);
  for (int r = 0; r < R; ++r) {
    flags[r].resize(p.gpus[r].tbs.size());
    for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) flags[r][t].assign(p.gpus[r].tbs[t].ops.size(), 0);
  }
  complete = false;
  if (!p.inplace || R < 2 || p.collective != "reducescatter" || p.nchunks[0] % R) return flags;
  const int c = p.nchunks[0] / R;
  const HbGraph g(p);
  if (!g.ok) return flags;
  auto is_input = [&](Buf b) { return b == Buf::input || b == Buf::output; };
  struct Acc {
    int node, off, cnt;
    bool write;
  };
  complete = true;
  for (int r = 0; r < R; ++r) {
    std::vector<Acc> acc;  // every local access of `input` on this rank
    for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t)
      for (size_t s = 0; s < p.gpus[r].tbs[t].ops.size(); ++s) {
        const Op& op = p.gpus[r].tbs[t].ops[s];
        const int u = g.node(r, static_cast<int>(t), static_cast<int>(s));
        switch (op.op) {
          case Opcode::send: case Opcode::rrs:
            if (is_input(op.src_buf)) acc.push_back({u, op.src_off, op.count, false});
            break;
          case Opcode::recv:
            if (is_input(op.dst_buf)) acc.push_back({u, op.dst_off, op.count, true});
            break;
          case Opcode::copy: case Opcode::reduce: case Opcode::rrc:
            if (is_input(op.src_buf)) acc.push_back({u, op.src_off, op.count, false});
            if (is_input(op.dst_buf)) acc.push_back({u, op.dst_off, op.count, true});
            if (op.op == Opcode::reduce && is_input(op.dst_buf)) acc.push_back({u, op.dst_off, op.count, false});
            break;
          case Opcode::rcs: case Opcode::rrcs:
            if (is_input(op.src_buf)) {
              acc.push_back({u, op.src_off, op.count, true});
              acc.push_back({u, op.src_off, op.count, false});  // forwards (or is pulled from) its span
            }
            break;
          default: break;
        }
      }
    std::vector<bool> covered(c, false);
    for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t)
      for (size_t s = 0; s < p.gpus[r].tbs[t].ops.size(); ++s) {
        const Op& op = p.gpus[r].tbs[t].ops[s];
        const bool local_writer = op.op == Opcode::recv || op.op == Opcode::copy || op.op == Opcode::reduce || op.op == Opcode::rrc;
        if (!local_writer || !is_input(op.dst_buf)) continue;
        if (op.dst_off < r * c || op.dst_off + op.count > (r + 1) * c) continue;  // not inside the owned block
        const int u = g.node(r, static_cast<int>(t), static_cast<int>(s));
        bool final_write = true;
        for (const Acc& a : acc) {
          if (a.node == u || !(a.off < op.dst_off + op.count && op.dst_off < a.off + a.cnt)) continue;
          if (!g.reaches(a.node, u)) final_write = false;  // another access is not before this write
        }
        if (final_write) {
          flags[r][t][s] = 1;
          for (int k = op.dst_off; k < op.dst_off + op.count; ++k) covered[k - r * c] = true;
        }
      }
    for (bool b : covered) complete = complete && b;
  }
  return flags;
}

// Work balance. Thread blocks joined by FIFO connections must run the same number of lanes (lane
// l of a sender talks to lane l of its receiver), but separate components need not: a component
// whose thread blocks move more bytes per tile (e.g. the coalesced count-G exchange of the two-step
// AllToAll) gets proportionally more lanes. Weight of a thread block = chunk
// passes its units make per tile (a direct receive moves nothing; its sender does the writing).
std::vector<std::vector<int>> lane_multipliers(const Program& p, int mode, int cap, uint8_t mask) {
  const int R = p.ranks();
  auto direct = direct_messages(p, true, nullptr);
  for (auto& g : direct)
    for (auto& tb : g)
      for (auto& f : tb) f &= mask;
  // connections that carry a FIFO message (under `mask`) need the same lanes at both ends
  std::set<std::tuple<int, int, int>> fifo_conn;
  for (int r = 0; r < R; ++r)
    for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) {
      const ThreadBlock& tb = p.gpus[r].tbs[t];
      for (size_t s = 0; s < tb.ops.size(); ++s)
        if (op_receives(tb.ops[s].op) && tb.recv_peer >= 0 && !(direct[r][t][s] & (kInDirect | kInPull)))
          fifo_conn.insert({tb.recv_peer, r, tb.channel});
    }
  std::vector<int> base(R + 1, 0);
  for (int r = 0; r < R; ++r) base[r + 1] = base[r] + static_cast<int>(p.gpus[r].tbs.size());
  std::vector<int> parent(base[R]);
  for (int i = 0; i < base[R]; ++i) parent[i] = i;
  std::function<int(int)> find = [&](int x) { return parent[x] == x ? x : parent[x] = find(parent[x]); };
  std::vector<int> weight(base[R], 0);
  for (int r = 0; r < R; ++r)
    for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) {
      const ThreadBlock& tb = p.gpus[r].tbs[t];
      if (tb.send_peer >= 0 && tb.send_peer < R && fifo_conn.count({r, tb.send_peer, tb.channel})) {
        const int rt = find_receiver(p, r, tb.send_peer, tb.channel);
        if (rt >= 0) parent[find(base[r] + static_cast<int>(t))] = find(base[tb.send_peer] + rt);
      }
      int w = 0;
      for (size_t s = 0; s < tb.ops.size(); ++s) {
        const Op& op = tb.ops[s];
        const uint8_t f = direct.empty() ? 0 : direct[r][t][s];
        const bool in_d = f & kInDirect, out_p = f & kOutPull;
        // reads + writes of the unit (the message: read unless direct-in, written unless pulled)
        int passes = 0;
        switch (op.op) {
          case Opcode::send: passes = out_p ? 0 : 2; break;
          case Opcode::copy: passes = 2; break;
          case Opcode::recv: passes = in_d ? 0 : 2; break;
          case Opcode::reduce: passes = 3; break;
          case Opcode::rrc: case Opcode::rrs: passes = 3; break;
          case Opcode::rcs: passes = (in_d ? 1 : 2) + (out_p ? 0 : 1); break;
          case Opcode::rrcs: passes = 3 + (out_p ? 0 : 1); break;
          default: break;
        }
        w += passes * op.count;
      }
      weight[base[r] + static_cast<int>(t)] = w;
    }
  std::map<int, int> comp_w;
  for (int i = 0; i < base[R]; ++i) comp_w[find(i)] = std::max(comp_w[find(i)], weight[i]);
  int wmin = 0;
  for (const auto& [root, w] : comp_w)
    if (w > 0 && (wmin == 0 || w < wmin)) wmin = w;
  std::vector<std::vector<int>> mult(R);
  for (int r = 0; r < R; ++r)
    for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) {
      const int w = comp_w[find(base[r] + static_cast<int>(t))];
      // mode 1: nearest multiple of the lightest component, mode 2: rounded up
      const int k = wmin > 0 ? (mode >= 2 ? (w + wmin - 1) / wmin : (w + wmin / 2) / wmin) : 1;
      mult[r].push_back(std::max(1, std::min(cap, k)));
    }
  return mult;
}

ncclResult_t build_plan(Clique* cl, DeviceState& ds, int id) {
  if (ds.plans.size() <= static_cast<size_t>(id)) ds.plans.resize(id + 1);
  DevicePlan& plan = ds.plans[id];
  if (plan.built) return ncclSuccess;
  plan.ranks.clear();
  for (int r = 0; r < cl->nranks; ++r)
    if (cl->local[r] && cl->local[r]->device == ds.device) plan.ranks.push_back(r);
  if (plan.ranks.empty()) return set_error(ncclInternalError, "no local ranks on device %d", ds.device);
  if (static_cast<int>(plan.ranks.size()) > kMaxLocalRanks)
    return set_error(ncclInvalidUsage, "%zu ranks on one device exceeds %d", plan.ranks.size(), kMaxLocalRanks);
  Comm* c0 = cl->local[plan.ranks[0]];
  for (int r : plan.ranks)
    if (cl->local[r]->irs.size() <= static_cast<size_t>(id))
      return set_error(ncclInvalidUsage, "rank %d has not registered IR %d", r, id);
  const RankIR& ir0 = *c0->irs[id];
  const Program& p = ir0.prog;
  const int L = ir0.lanes;

  std::vector<DevTb> tbs;
  std::vector<DevOp> ops;
  std::vector<DevDep> deps;
  std::vector<DevChan> chans;
  plan.sys_scope = false;
  // direct messages only between ranks of this launch: the sender needs the receiver's buffers
  std::vector<std::vector<std::vector<PullSrc>>> pull_src;
  bool source_complete = false;
  const auto source = c0->cfg.source ? source_reads(p, source_complete) : std::vector<std::vector<std::vector<uint8_t>>>();
  plan.source_complete = c0->cfg.source && source_complete;
  bool result_complete = false;
  const auto result = c0->cfg.source ? result_writes(p, result_complete) : std::vector<std::vector<std::vector<uint8_t>>>();
  plan.result_complete = c0->cfg.source && result_complete;
  auto direct = c0->cfg.direct ? direct_messages(p, (c0->cfg.direct & 2) != 0, &pull_src)
                               : std::vector<std::vector<std::vector<uint8_t>>>();
  if (!(c0->cfg.direct & 1))  // pulls only: drop the direct flags
    for (auto& g : direct)
      for (auto& tb : g)
        for (auto& f : tb) f &= static_cast<uint8_t>(~(kInDirect | kOutDirect));
  auto slot_of = [&](int rank) {
    for (size_t i = 0; i < plan.ranks.size(); ++i)
      if (plan.ranks[i] == rank) return static_cast<int>(i);
    return -1;
  };
  // GPU of every rank: scope per thread block (.sys only where a connection reaches another GPU)
  std::vector<std::string> gpu_of(p.ranks());
  for (int r = 0; r < p.ranks(); ++r) NCCL_TRY(rank_gpu(c0, r, gpu_of[r]));
  const std::string& my_gpu = gpu_of[plan.ranks[0]];
  // remote transports: direct and pulled messages to and from ranks of other launches address their
  // registered user buffers (exchanged per call, exchange_buffers); those ranks get buffer slots
  // after the launch's own. Every rank of the program decides the same way (same program, config
  // and placement), so both ends of a connection agree on its transport.
  plan.remote_ranks.clear();
  bool remote_ok = c0->cfg.remote && static_cast<int>(plan.ranks.size()) < p.ranks() && !direct.empty();
  // every launch of a process exchanges with the other processes' launches in call order, so every
  // process must drive exactly one launch per call (one device). Decided from the bootstrap records
  // (pid and GPU of every rank), identically in every process: if any process hosts ranks on
  // several devices, every cross-launch message keeps the FIFOs
  if (remote_ok) {
    std::map<long, std::string> gpu_of_pid;
    for (int r = 0; r < p.ranks() && remote_ok; ++r) {
      long pid = 0;
      NCCL_TRY(rank_pid(c0, r, pid));
      auto [it, fresh] = gpu_of_pid.emplace(pid, gpu_of[r]);
      if (!fresh && it->second != gpu_of[r]) remote_ok = false;
    }
  }
  if (remote_ok) {
    for (int r = 0; r < p.ranks(); ++r)
      if (slot_of(r) < 0) plan.remote_ranks.push_back(r);
    if (plan.ranks.size() + plan.remote_ranks.size() > static_cast<size_t>(kMaxLocalRanks)) {
      remote_ok = false;
      plan.remote_ranks.clear();
    }
  }
  auto vslot_of = [&](int rank) {
    const int s0 = slot_of(rank);
    if (s0 >= 0) return s0;
    for (size_t i = 0; i < plan.remote_ranks.size(); ++i)
      if (plan.remote_ranks[i] == rank) return static_cast<int>(plan.ranks.size() + i);
    return -1;
  };
  // the transports this launch applies (both ends in it, or reachable through registered buffers);
  // with per-connection lanes (lane_mask) exactly the ones the lane multipliers assumed
  std::vector<std::vector<std::vector<uint8_t>>> eff(p.ranks());
  plan.remote_msgs = 0;
  for (int r = 0; r < p.ranks(); ++r) {
    eff[r].resize(p.gpus[r].tbs.size());
    for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) {
      const ThreadBlock& tb = p.gpus[r].tbs[t];
      eff[r][t].assign(tb.ops.size(), 0);
      if (direct.empty() || vslot_of(r) < 0) continue;
      for (size_t s = 0; s < tb.ops.size(); ++s) {
        uint8_t f = direct[r][t][s];
        if (ir0.lane_mask) f &= ir0.lane_mask;
        if ((f & (kInDirect | kInPull)) && tb.recv_peer >= 0 && vslot_of(tb.recv_peer) >= 0) {
          eff[r][t][s] |= f & (kInDirect | kInPull);
          if (slot_of(r) >= 0 && slot_of(tb.recv_peer) < 0) plan.remote_msgs++;
        }
        if ((f & (kOutDirect | kOutPull)) && tb.send_peer >= 0 && vslot_of(tb.send_peer) >= 0)
          eff[r][t][s] |= f & (kOutDirect | kOutPull);
      }
    }
  }
  for (int r : plan.ranks) {
    cl->local[r]->irs[id]->eff_direct = eff;
    cl->local[r]->irs[id]->order_ok.clear();  // verdicts computed without the direct flags
  }
  // direct / pulled receives wait on their sender's semaphore (message deps), which works across
  // thread blocks of different lane counts; connections without FIFO messages then need no
  // head / tail counters at all (only when lanes may differ across connections, lane_mask)
  const auto senders = matched_senders(p);
  std::map<std::tuple<int, int, int>, std::tuple<int, int, int>> receiver_of;  // send op -> receive op
  for (int r = 0; r < p.ranks(); ++r)
    for (size_t t = 0; t < senders[r].size(); ++t)
      for (size_t s = 0; s < senders[r][t].size(); ++s)
        if (senders[r][t][s].rank >= 0)
          receiver_of[{senders[r][t][s].rank, senders[r][t][s].tb, senders[r][t][s].step}] = {r, static_cast<int>(t), static_cast<int>(s)};
  // spans each rank reads (for the L2 hints): (buffer, first chunk, end chunk)
  std::vector<std::vector<std::tuple<Buf, int, int>>> reads(p.ranks());
  auto storage = [&](Buf b) { return p.inplace && b == Buf::output ? Buf::input : b; };
  for (int r = 0; r < p.ranks(); ++r)
    for (const auto& tb : p.gpus[r].tbs)
      for (const auto& op : tb.ops) {
        if (op.op == Opcode::recv || op.op == Opcode::nop) continue;
        reads[r].emplace_back(op.src_buf, op.src_off, op.src_off + op.count);
        if (op.op == Opcode::reduce) reads[r].emplace_back(op.dst_buf, op.dst_off, op.dst_off + op.count);
      }
  std::set<std::tuple<int, int, int>> fifo_conn;
  std::set<std::tuple<int, int, int>> pub_sem;
  for (int r = 0; r < p.ranks(); ++r)
    for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) {
      const ThreadBlock& tb = p.gpus[r].tbs[t];
      for (size_t s = 0; s < tb.ops.size(); ++s) {
        if (!op_receives(tb.ops[s].op) || tb.recv_peer < 0) continue;
        if (eff[r][t][s] & (kInDirect | kInPull)) {
          const auto& sd = senders[r][t][s];
          if (sd.rank >= 0) pub_sem.insert({sd.rank, sd.tb, sd.step});
        } else {
          fifo_conn.insert({tb.recv_peer, r, tb.channel});
        }
      }
    }
  // semaphores: lanes x mult per thread block, in launch order
  const auto& mult = ir0.mult;
  std::map<std::pair<int, int>, int> sem_base;  // (rank, tb index) -> first semaphore
  std::map<std::pair<int, int>, int> launch_index;  // (rank, tb index) -> thread block index in the launch
  int sem_next = 0, weight = 0;
  for (size_t slot = 0; slot < plan.ranks.size(); ++slot) {
    const int r = plan.ranks[slot];
    for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) {
      sem_base[{r, static_cast<int>(t)}] = sem_next;
      launch_index[{r, static_cast<int>(t)}] = static_cast<int>(launch_index.size());
      sem_next += L * mult[r][t];
    }
  }
  // work-queue mode needs every message direct or pulled (no FIFO) and every rank in this launch
  plan.wq_ok = ir0.lane_mask != 0 && fifo_conn.empty();
  plan.wq_level.assign(launch_index.size(), 0);
  for (int pass = 0; pass < static_cast<int>(launch_index.size()); ++pass)  // longest dep chain, by relaxation
    for (size_t slot = 0; slot < plan.ranks.size(); ++slot) {
      const int r = plan.ranks[slot];
      for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) {
        int& lv = plan.wq_level[launch_index[{r, static_cast<int>(t)}]];
        for (const Op& op : p.gpus[r].tbs[t].ops)
          for (const Dep& d : op.deps) {
            const int ti = tb_index(p, r, d.tb);
            if (ti >= 0 && ti != static_cast<int>(t)) lv = std::max(lv, 1 + plan.wq_level[launch_index[{r, ti}]]);
          }
        lv = std::min(lv, 64);
      }
    }
  for (size_t slot = 0; slot < plan.ranks.size(); ++slot) {
    const int r = plan.ranks[slot];
    Comm* c = cl->local[r];
    const RankIR& ir = *c->irs[id];
    const Gpu& g = p.gpus[r];
    for (size_t t = 0; t < g.tbs.size(); ++t) {
      const ThreadBlock& tb = g.tbs[t];
      const int Lt = L * mult[r][t];
      DevTb d{};
      d.rank_slot = static_cast<int>(slot);
      d.op_begin = static_cast<int>(ops.size());
      d.nops = static_cast<int>(tb.ops.size());
      d.sem = sem_base[{r, static_cast<int>(t)}];
      d.mult = mult[r][t];
      d.unit_base = weight;
      weight += mult[r][t];
      d.chan_in = d.chan_out = -1;
      d.peer_slot = tb.send_peer >= 0 ? vslot_of(tb.send_peer) : -1;
      d.recv_slot = tb.recv_peer >= 0 ? vslot_of(tb.recv_peer) : -1;
      d.sys = ((tb.send_peer >= 0 && gpu_of[tb.send_peer] != my_gpu) || (tb.recv_peer >= 0 && gpu_of[tb.recv_peer] != my_gpu)) ? 1 : 0;
      // config force_sys (testing): connections to ranks of other launches behave as if those ranks
      // were on another GPU (.sys scope, no bulk copies) -- the N-GPU code path, on one GPU
      if (c0->cfg.force_sys && ((tb.send_peer >= 0 && slot_of(tb.send_peer) < 0) || (tb.recv_peer >= 0 && slot_of(tb.recv_peer) < 0)))
        d.sys = 1;
      if (d.sys) plan.sys_scope = true;
      const bool in_local = d.recv_slot >= 0;
      for (size_t s = 0; s < tb.ops.size(); ++s) {
        const Op& op = tb.ops[s];
        DevOp o{};
        (void)in_local;
        o.direct = eff[r][t][s];
        if (o.direct & kInPull) {
          const PullSrc& ps = pull_src[r][t][s];
          o.in_buf = static_cast<uint8_t>(ps.buf);
          o.in_off = ps.off;
          // a send whose read of the span comes from the caller's buffer is pulled from there too
          if (plan.source_complete && p.gpus[ps.rank].tbs[ps.tb].ops[ps.step].op == Opcode::send &&
              (source[ps.rank][ps.tb][ps.step] & kSrcFromSource))
            o.in_buf = kSource;
        }
        if (pub_sem.count({r, static_cast<int>(t), static_cast<int>(s)})) o.direct |= kPubSem;
        if ((c0->cfg.l2hint & 1) && op_sends(op.op)) {  // its receiver reads what it writes: keep it in L2
          const auto rcv = receiver_of.find({r, static_cast<int>(t), static_cast<int>(s)});
          if (!(o.direct & kOutDirect)) {
            o.hot = 1;  // FIFO slot or pulled span: read by the receive
          } else if (rcv != receiver_of.end()) {  // a span of the receiving rank some op reads again
            const int rr = std::get<0>(rcv->second);
            for (const auto& [b, lo, hi] : reads[rr])
              if (storage(b) == storage(op.dst_buf) && lo < op.dst_off + op.count && op.dst_off < hi) o.hot = 1;
          }
        }
        if (ir0.lane_mask) {
          if (op_sends(op.op) && tb.send_peer >= 0 && !fifo_conn.count({r, tb.send_peer, tb.channel})) o.direct |= kNoCtrOut;
          if (op_receives(op.op) && tb.recv_peer >= 0 && !fifo_conn.count({tb.recv_peer, r, tb.channel})) o.direct |= kNoCtrIn;
        }
        o.opcode = static_cast<uint8_t>(op.op);
        o.src_buf = static_cast<uint8_t>(op.src_buf);
        o.dst_buf = static_cast<uint8_t>(op.dst_buf);
        o.src_rbuf = plan.source_complete && (source[r][t][s] & kSrcFromSource) ? kSource : o.src_buf;
        o.dst_rbuf = plan.source_complete && (source[r][t][s] & kDstFromSource) ? kSource : o.dst_buf;
        if (plan.result_complete && result[r][t][s]) o.dst_buf = kResult;  // final owned write -> recvbuff
        if (plan.result_complete && (o.direct & kOutDirect)) {
          // a direct message whose receive is a final owned write: the sender stores it straight into
          // the receiver's result buffer (the receive itself moves nothing)
          const auto rcv = receiver_of.find({r, static_cast<int>(t), static_cast<int>(s)});
          if (rcv != receiver_of.end()) {
            const auto [rr, rt, rs] = rcv->second;
            if (result[rr][rt][rs]) o.dst_buf = kResult;
          }
        }
        o.has_dep = op.has_dep ? 1 : 0;
        o.src_off = op.src_off;
        o.dst_off = op.dst_off;
        o.count = op.count;
        o.dep_begin = static_cast<int>(deps.size());
        o.ndeps = static_cast<int16_t>(op.deps.size());
        for (const Dep& dp : op.deps) {
          const int ti = tb_index(p, r, dp.tb);
          if (ti < 0) return set_error(ncclInvalidArgument, "IR dep on unknown tb %d", dp.tb);
          DevDep dd{};
          dd.sem = sem_base[{r, ti}];
          dd.step = dp.step;
          dd.nops = static_cast<int>(g.tbs[ti].ops.size());
          dd.mult = mult[r][ti];
          dd.tbi = launch_index[{r, ti}];
          deps.push_back(dd);
        }
        if (o.direct & (kInDirect | kInPull)) {  // message dep on the sending op
          const auto& sd = senders[r][t][s];
          if (sd.rank >= 0 && sem_base.count({sd.rank, sd.tb})) {
            DevDep dd{};
            dd.sem = sem_base[{sd.rank, sd.tb}];
            dd.step = sd.step;
            dd.nops = static_cast<int>(p.gpus[sd.rank].tbs[sd.tb].ops.size());
            dd.mult = mult[sd.rank][sd.tb];
            dd.tbi = launch_index[{sd.rank, sd.tb}];
            deps.push_back(dd);
            o.nmsg = 1;
            o.ndeps = static_cast<int16_t>(o.ndeps + 1);
            o.direct |= kMsgDep;
          }
        }
        ops.push_back(o);
      }
      if (tb.recv_peer >= 0) {
        const int s = tb.recv_peer;
        const int st = find_sender(p, s, r, tb.channel);
        if (st < 0) return set_error(ncclInvalidArgument, "connection %d->%d ch %d has no sender", s, r, tb.channel);
        char* sender_arena = nullptr;
        NCCL_TRY(peer_arena(c, id, s, sender_arena));
        const int k = ir.lay.in_index[t];
        const ArenaLayout slay = make_layout(p, s, L, ir.slots, ir.slot_bytes, mult);
        const int m = slay.out_index[st];
        const size_t kb = ir.lay.in_lane_base[k], mb = slay.out_lane_base[m];
        d.chan_in = static_cast<int>(chans.size());
        for (int l = 0; l < Lt; ++l) {
          DevChan ch{};
          for (int pr = 0; pr < kNumProtos; ++pr) {
            ch.fifo[pr] = ir.arena + ir.lay.fifo_off[pr][k] + static_cast<size_t>(l) * ir.slots * ir.lay.slot_stride[pr][k];
            ch.slot_bytes[pr] = ir.lay.slot_stride[pr][k];
          }
          ch.head = reinterpret_cast<uint64_t*>(ir.arena + ir.lay.off_head + (kb + l) * kCounterStride);
          ch.tail = reinterpret_cast<uint64_t*>(sender_arena + slay.off_tail + (mb + l) * kCounterStride);
          ch.mine = reinterpret_cast<uint64_t*>(ir.arena + ir.lay.off_mine_in + (kb + l) * 8);
          chans.push_back(ch);
        }
      }
      if (tb.send_peer >= 0) {
        const int dst = tb.send_peer;
        const int rt = find_receiver(p, r, dst, tb.channel);
        if (rt < 0) return set_error(ncclInvalidArgument, "connection %d->%d ch %d has no receiver", r, dst, tb.channel);
        char* recv_arena = nullptr;
        NCCL_TRY(peer_arena(c, id, dst, recv_arena));
        const ArenaLayout rlay = make_layout(p, dst, L, ir.slots, ir.slot_bytes, mult);
        const int k = rlay.in_index[rt];
        const int m = ir.lay.out_index[t];
        const size_t kb = rlay.in_lane_base[k], mb = ir.lay.out_lane_base[m];
        d.chan_out = static_cast<int>(chans.size());
        for (int l = 0; l < Lt; ++l) {
          DevChan ch{};
          for (int pr = 0; pr < kNumProtos; ++pr) {
            ch.fifo[pr] = recv_arena + rlay.fifo_off[pr][k] + static_cast<size_t>(l) * ir.slots * rlay.slot_stride[pr][k];
            ch.slot_bytes[pr] = rlay.slot_stride[pr][k];
          }
          ch.head = reinterpret_cast<uint64_t*>(recv_arena + rlay.off_head + (kb + l) * kCounterStride);
          ch.tail = reinterpret_cast<uint64_t*>(ir.arena + ir.lay.off_tail + (mb + l) * kCounterStride);
          ch.mine = reinterpret_cast<uint64_t*>(ir.arena + ir.lay.off_mine_out + (mb + l) * 8);
          chans.push_back(ch);
        }
      }
      tbs.push_back(d);
    }
  }
  for (const DevOp& o : ops)
    if (o.ndeps > 400) return set_error(ncclInvalidArgument, "an op with %d deps exceeds the 400-dep limit", o.ndeps);
  // dataflow graph: possible when every rank of the program runs in this launch and the
  // happens-before graph is acyclic. Node = op (launch order); edges = previous op of the thread
  // block, declared deps, message sender -> receiver; messages neither direct nor pulled get a
  // mailbox span each.
  std::vector<DfNode> df_nodes;
  std::vector<DfSucc> df_succ;
  std::vector<int32_t> df_roots;
  plan.df_ok = false;
  plan.df_mail_chunks = 0;
  plan.df_mail_msgs = 0;
  if (static_cast<int>(plan.ranks.size()) == p.ranks() && HbGraph(p).ok) {
    std::vector<std::set<int>> succ(ops.size()), msg_succ(ops.size());
    std::vector<int> indeg(ops.size(), 0);
    auto node = [&](int r, int t, int s) { return tbs[launch_index[{r, t}]].op_begin + s; };
    df_nodes.assign(ops.size(), DfNode{});
    for (size_t v = 0; v < ops.size(); ++v) {
      df_nodes[v].op = ops[v];
      df_nodes[v].in_mail = df_nodes[v].out_mail = -1;
    }
    for (int r : plan.ranks)
      for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) {
        const ThreadBlock& tb = p.gpus[r].tbs[t];
        for (size_t s = 0; s < tb.ops.size(); ++s) {
          const int v = node(r, static_cast<int>(t), static_cast<int>(s));
          const DevTb& dtb = tbs[launch_index[{r, static_cast<int>(t)}]];
          df_nodes[v].tbi = launch_index[{r, static_cast<int>(t)}];
          df_nodes[v].rank_slot = static_cast<int8_t>(dtb.rank_slot);
          df_nodes[v].peer_slot = static_cast<int8_t>(dtb.peer_slot);
          df_nodes[v].recv_slot = static_cast<int8_t>(dtb.recv_slot);
          if (s > 0) succ[node(r, static_cast<int>(t), static_cast<int>(s) - 1)].insert(v);
          for (const Dep& dp : tb.ops[s].deps) succ[node(r, tb_index(p, r, dp.tb), dp.step)].insert(v);
          const auto& sd = senders[r][t][s];
          if (op_receives(tb.ops[s].op) && tb.recv_peer >= 0 && sd.rank >= 0) {
            const int x = node(sd.rank, sd.tb, sd.step);
            succ[x].insert(v);
            msg_succ[x].insert(v);
            if (!(eff[r][t][s] & (kInDirect | kInPull))) {  // a mailed message
              df_nodes[v].in_mail = static_cast<int32_t>(plan.df_mail_chunks);
              df_nodes[x].out_mail = static_cast<int32_t>(plan.df_mail_chunks);
              plan.df_mail_chunks += tb.ops[s].count;
              plan.df_mail_msgs++;
            }
          }
        }
      }
    bool fits = true;
    for (size_t u = 0; u < ops.size(); ++u) {
      df_nodes[u].nsucc = static_cast<int16_t>(succ[u].size());
      fits = fits && succ[u].size() < 32768;
      for (int v : succ[u]) indeg[v]++;
    }
    // successors in priority order for the continuation (interp_df_kernel): the receivers of the
    // node's message first (they read what it just produced), then the rest
    for (size_t u = 0; u < ops.size(); ++u) {
      df_nodes[u].succ = static_cast<int32_t>(df_succ.size());
      for (int pass = 0; pass < 2; ++pass)
        for (int v : succ[u])
          if (msg_succ[u].count(v) == (pass == 0 ? 1u : 0u)) df_succ.push_back(DfSucc{v, indeg[v]});
    }
    for (size_t u = 0; u < ops.size(); ++u) {
      df_nodes[u].indeg = static_cast<int16_t>(indeg[u]);
      fits = fits && indeg[u] < 32768;
      if (indeg[u] == 0) df_roots.push_back(static_cast<int32_t>(u));
    }
    // average width of the graph (nodes / longest path): the ready items of one tile at a time
    std::vector<int> level(ops.size(), 1);
    std::vector<int> order(df_roots.begin(), df_roots.end()), deg(indeg);
    for (size_t i = 0; i < order.size(); ++i)
      for (int v : succ[order[i]]) {
        level[v] = std::max(level[v], level[order[i]] + 1);
        if (--deg[v] == 0) order.push_back(v);
      }
    plan.df_depth = order.empty() ? 1 : *std::max_element(level.begin(), level.end());
    plan.df_ok = fits && !df_roots.empty() && order.size() == ops.size() && ops.size() < (1u << 20);
    plan.df_n = static_cast<int>(ops.size());
    plan.df_nroots = static_cast<int>(df_roots.size());
  }
  DeviceGuard g(ds.device);
  auto upload = [&](auto*& dptr, const auto& vec) -> ncclResult_t {
    using T = typename std::decay_t<decltype(vec)>::value_type;
    const size_t n = std::max<size_t>(vec.size(), 1) * sizeof(T);
    CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&dptr), n));
    if (!vec.empty()) CUDA_TRY(cudaMemcpy(dptr, vec.data(), vec.size() * sizeof(T), cudaMemcpyHostToDevice));
    return ncclSuccess;
  };
  NCCL_TRY(upload(plan.d_tbs, tbs));
  NCCL_TRY(upload(plan.d_ops, ops));
  NCCL_TRY(upload(plan.d_deps, deps));
  NCCL_TRY(upload(plan.d_chans, chans));
  if (plan.df_ok) {
    NCCL_TRY(upload(plan.d_df_nodes, df_nodes));
    NCCL_TRY(upload(plan.d_df_succ, df_succ));
    NCCL_TRY(upload(plan.d_df_roots, df_roots));
  }
  const size_t nsem = std::max(sem_next, 1);
  CUDA_TRY(cudaMalloc(&plan.d_sems, nsem * sizeof(uint64_t)));
  CUDA_TRY(cudaMemset(plan.d_sems, 0, nsem * sizeof(uint64_t)));
  plan.ntbs = static_cast<int>(tbs.size());
  plan.weight = weight;
  plan.built = true;
  return ncclSuccess;
}

// Algorithmic traffic of one rank's program for a given chunk size.
void traffic(const Program& p, int rank, int64_t chunk_bytes, int64_t& sent, int64_t& recvd, int64_t& hbm) {
  sent = recvd = hbm = 0;
  for (const auto& tb : p.gpus[rank].tbs)
    for (const auto& op : tb.ops) {
      const int64_t b = chunk_bytes * op.count;
      if (op_sends(op.op)) sent += b;
      if (op_receives(op.op)) recvd += b;
      switch (op.op) {
        case Opcode::send: hbm += b; break;
        case Opcode::recv: hbm += b; break;
        case Opcode::copy: hbm += 2 * b; break;
        case Opcode::reduce: hbm += 3 * b; break;
        case Opcode::rrc: hbm += 2 * b; break;
        case Opcode::rcs: hbm += b; break;
        case Opcode::rrcs: hbm += 2 * b; break;
        case Opcode::rrs: hbm += b; break;
        default: break;
      }
    }
}

// Timed model ("run_timed", restated as an alpha-beta model over the program's
// happens-before graph and calibrated on this B200 in loopback): every op of a tile
// costs alpha (synchronisation: poll, fences, barriers; lower for LL, which has no fences) plus its
// bytes over one unit's streaming rate beta_u. A tile's latency is the heaviest path through the
// per-tile op graph (sequential order, deps, messages); a lane then streams its k tiles at the pace
// of its heaviest thread block. The launch is bounded below by the algorithmic bytes over the
// aggregate bandwidth. Used to rank matching IRs (config "select") and reported by gc3IrPredict.
struct TimedModel {
  // least-squares fit (log error) on the C4 sweep of BASELINE.md §5.2 (r01f3): 8% / 9% rms
  double alpha_us[2] = {3.5, 1.5};        // per op: Simple, LL
  double beta_unit_gbs[2] = {60.0, 40.0};  // one unit's streaming rate
  double bw_gbs[2] = {4000.0, 600.0};      // aggregate rate of algorithmic bytes (loopback: HBM; LL lines)
  double bw_copy_gbs = 5600.0;             // Simple, programs without reductions (measured C2 / C2D)
  double launch_us = 8.0;
};

double predict_us(const Program& p, int64_t chunk_bytes, int proto, int lanes, const TimedModel& m = TimedModel()) {
  if (chunk_bytes <= 0) return m.launch_us;
  const int ll = proto == 1 ? 1 : 0;
  lanes = std::max(1, lanes);
  int64_t tile = std::min<int64_t>(256 << 10, std::max<int64_t>(4 << 10, (chunk_bytes + lanes - 1) / lanes));
  tile = std::min(tile, chunk_bytes);
  const double k = std::ceil(static_cast<double>(chunk_bytes) / (static_cast<double>(tile) * lanes));
  auto passes = [](Opcode o) {
    switch (o) {
      case Opcode::send: case Opcode::recv: case Opcode::rcs: return 2;
      case Opcode::copy: case Opcode::rrc: case Opcode::rrs: return 2;
      case Opcode::reduce: case Opcode::rrcs: return 3;
      default: return 0;
    }
  };
  auto op_us = [&](const Op& op) {
    return m.alpha_us[ll] + passes(op.op) * op.count * static_cast<double>(tile) / (m.beta_unit_gbs[ll] * 1e3);
  };
  const HbGraph g(p);
  double path = 0.0, tb_max = 0.0;
  if (g.ok) {  // heaviest path: longest-path DP over the nodes in index order repeated to a fixpoint
    std::vector<double> w(g.n, 0.0), best(g.n, 0.0);
    for (int r = 0; r < p.ranks(); ++r)
      for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) {
        double tbsum = 0.0;
        for (size_t s = 0; s < p.gpus[r].tbs[t].ops.size(); ++s) {
          const double c = op_us(p.gpus[r].tbs[t].ops[s]);
          w[g.node(r, static_cast<int>(t), static_cast<int>(s))] = c;
          tbsum += c;
        }
        tb_max = std::max(tb_max, tbsum);
      }
    // best[v] = w[v] + max over predecessors u (reaches(u, v), u != v) of best[u]; nodes sorted by
    // the number of their ancestors give a topological order
    std::vector<int> order(g.n), anc(g.n, 0);
    for (int v = 0; v < g.n; ++v) {
      order[v] = v;
      for (int u = 0; u < g.n; ++u) anc[v] += (u != v && g.reaches(u, v)) ? 1 : 0;
    }
    std::sort(order.begin(), order.end(), [&](int a, int b) { return anc[a] < anc[b]; });
    for (int v : order) {
      double pre = 0.0;
      for (int u = 0; u < g.n; ++u)
        if (u != v && g.reaches(u, v)) pre = std::max(pre, best[u]);
      best[v] = pre + w[v];
      path = std::max(path, best[v]);
    }
  }
  const double pipe = path + (k - 1.0) * tb_max;
  double bytes = 0.0;
  for (int r = 0; r < p.ranks(); ++r) {
    int64_t snt, rcv, h;
    traffic(p, r, chunk_bytes, snt, rcv, h);
    bytes += static_cast<double>(h);
  }
  bool reduces = false;
  for (const auto& gp : p.gpus)
    for (const auto& tb : gp.tbs)
      for (const auto& op : tb.ops) reduces = reduces || op_reduces(op.op);
  const double bw = bytes / ((!ll && !reduces ? m.bw_copy_gbs : m.bw_gbs[ll]) * 1e3);
  return m.launch_us + std::max(pipe, bw);
}

// IR chunk geometry of a collective call. The NCCL count of one rank's block (AllReduce: count;
// AllGather: sendcount; ReduceScatter: recvcount; AlltoAll: count per peer) is split into the IR's
// c chunks per block of ceil(count / c) elements; when c does not divide the count the last chunks
// are clipped ("ragged": element p of a block is element p % ce of chunk p / ce, the runtime pads
// each block to c x ce elements in work buffers). Returns elements per chunk, -1 if the IR's shape
// does not fit the collective.
int64_t chunk_elems_for(const Program& p, int coll, size_t count, int nranks, bool* ragged = nullptr) {
  const int cin = p.nchunks[0];
  if (cin <= 0) return -1;
  int c = cin;
  switch (coll) {
    case kAllReduce: break;
    case kAllGather:
      if (p.nchunks[1] != nranks * cin) return -1;
      break;
    case kReduceScatter:
      if (cin % nranks) return -1;
      c = cin / nranks;
      break;
    case kAllToAll:
      if (cin % nranks || p.nchunks[1] != cin) return -1;
      c = cin / nranks;
      break;
    default: return -1;
  }
  if (ragged) *ragged = count % c != 0;
  return static_cast<int64_t>((count + c - 1) / c);
}

// bytes used for size_range selection: the per-rank message buffer size
uint64_t selection_bytes(int coll, size_t count, size_t esize, int nranks) {
  switch (coll) {
    case kAllReduce: return count * esize;
    case kAllGather: return count * esize * nranks;
    case kReduceScatter: return count * esize * nranks;
    case kAllToAll: return count * esize * nranks;
  }
  return 0;
}

// The first registered IR whose collective and size_range match (ir.hpp:112-116);
// the runtime's built-in programs only when no user IR does.
// With config "select", the matching user IR with the lowest timed-model prediction instead of
// the first one (predictions cached per IR and chunk size).
int select_ir(Comm* c, int coll, size_t count, int dtype) {
  const uint64_t bytes = selection_bytes(coll, count, dtype_size(dtype), c->nranks);
  for (int pass = 0; pass < 2; ++pass) {
    int best = -1;
    double best_us = 0.0;
    for (size_t i = 0; i < c->irs.size(); ++i) {
      if (c->irs[i]->builtin != (pass == 1)) continue;
      RankIR& ir = *c->irs[i];
      const Program& p = ir.prog;
      if (p.collective != coll_name(coll)) continue;
      if (bytes < p.min_bytes || bytes > p.max_bytes) continue;
      const int64_t ce = chunk_elems_for(p, coll, count, c->nranks);
      if (ce < 0) continue;
      if (!c->cfg.select) return static_cast<int>(i);
      const int64_t cb = ce * static_cast<int64_t>(dtype_size(dtype));
      auto f = ir.predicted.find(cb);
      if (f == ir.predicted.end()) {
        const int proto = ir.proto_override >= 0 ? ir.proto_override : static_cast<int>(p.proto);
        f = ir.predicted.emplace(cb, predict_us(p, cb, proto, ir.lanes)).first;
      }
      if (best < 0 || f->second < best_us) {
        best = static_cast<int>(i);
        best_us = f->second;
      }
    }
    if (best >= 0) return best;
  }
  return -1;
}

// Deadlock check of the kernel's execution order: every thread block walks its lane's tiles in
// groups of G, op-major inside a group; a non-direct send needs a free slot (FIFO depth `slots`),
// a receive needs a posted message, a dep needs its (thread block, step, tile) done. Enabling is
// monotone (only the owner of a connection end consumes it), so one greedy maximal run decides
// whether the order can deadlock: it completes iff every fair execution does.
bool order_is_deadlock_free(const Program& p, const std::vector<std::vector<std::vector<uint8_t>>>& direct, int64_t ntiles,
                            int lanes, const std::vector<std::vector<int>>& mult, int G, int slots) {
  if (ntiles <= 0) return true;
  struct Unit {
    int r, t, lane, lt;
    int64_t ntl;      // tiles of this lane
    int64_t pos = 0;  // ops completed in the lane's order
  };
  std::vector<Unit> units;
  std::map<std::pair<int, int>, int> first;  // (rank, tb) -> its lane-0 unit
  for (int r = 0; r < p.ranks(); ++r)
    for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) {
      const int lt = lanes * (mult.empty() ? 1 : mult[r][t]);
      first[{r, static_cast<int>(t)}] = static_cast<int>(units.size());
      for (int l = 0; l < lt; ++l) units.push_back({r, static_cast<int>(t), l, lt, ntiles > l ? (ntiles - 1 - l) / lt + 1 : 0});
    }
  auto position = [&](int64_t i, int step, int nops, int64_t ntl) {
    const int64_t g0 = i / G * G;
    const int64_t gsize = std::min<int64_t>(G, ntl - g0);
    return g0 * nops + step * gsize + (i - g0);
  };
  std::map<std::tuple<int, int, int, int>, std::pair<int64_t, int64_t>> conn;  // (src, dst, ch, lane) -> (sent, consumed)
  const auto senders = matched_senders(p);
  for (bool progress = true; progress;) {
    progress = false;
    for (Unit& u : units) {
      const ThreadBlock& tb = p.gpus[u.r].tbs[u.t];
      const int nops = static_cast<int>(tb.ops.size());
      while (nops > 0 && u.pos < u.ntl * nops) {
        const int64_t g0 = u.pos / (static_cast<int64_t>(G) * nops) * G;
        const int64_t gsize = std::min<int64_t>(G, u.ntl - g0);
        const int64_t in_group = u.pos - g0 * nops;
        const int step = static_cast<int>(in_group / gsize);
        const int64_t tile = u.lane + (g0 + in_group % gsize) * u.lt;
        const Op& op = tb.ops[step];
        bool ok = true;
        for (const Dep& d : op.deps) {
          const int ti = tb_index(p, u.r, d.tb);
          const Unit& du = units[first[{u.r, ti}] + static_cast<int>(tile % units[first[{u.r, ti}]].lt)];
          const int dn = static_cast<int>(p.gpus[u.r].tbs[ti].ops.size());
          if (du.pos < position(tile / du.lt, d.step, dn, du.ntl) + 1) ok = false;
        }
        const bool direct_out = !direct.empty() && (direct[u.r][u.t][step] & (kOutDirect | kOutPull));
        const bool direct_in = !direct.empty() && (direct[u.r][u.t][step] & (kInDirect | kInPull));
        if (ok && op_receives(op.op) && direct_in) {  // message dep: the sending op done for this tile
          const auto& sd = senders[u.r][u.t][step];
          const Unit& su = units[first[{sd.rank, sd.tb}] + static_cast<int>(tile % units[first[{sd.rank, sd.tb}]].lt)];
          const int sn = static_cast<int>(p.gpus[sd.rank].tbs[sd.tb].ops.size());
          if (su.pos < position(tile / su.lt, sd.step, sn, su.ntl) + 1) ok = false;
        } else if (ok && op_receives(op.op)) {
          const auto& c = conn[{tb.recv_peer, u.r, tb.channel, u.lane}];
          if (c.first <= c.second) ok = false;
        }
        if (ok && op_sends(op.op) && !direct_out) {
          const auto& c = conn[{u.r, tb.send_peer, tb.channel, u.lane}];
          if (c.first - c.second >= slots) ok = false;
        }
        if (!ok) break;
        if (op_receives(op.op)) conn[{tb.recv_peer, u.r, tb.channel, u.lane}].second++;
        if (op_sends(op.op)) conn[{u.r, tb.send_peer, tb.channel, u.lane}].first++;
        u.pos++;
        progress = true;
      }
    }
  }
  for (const Unit& u : units)
    if (u.pos < u.ntl * static_cast<int64_t>(p.gpus[u.r].tbs[u.t].ops.size())) return false;
  return true;
}

struct CallPlan {
  int id = -1;
  bool ll = false;  // a line protocol (LL or LL128): every message through the FIFO lines
  int proto = kProtoSimple;
  int lanes = 1;
  int grid = 0;
  int unit_warps = 4;
  int group = 1;
  int tma_stages = 0;
  size_t smem = 0;
  int64_t chunk_elems = 0, tile_elems = 0, ntiles = 0;  // in kernel element units
  int kesize = 1;                                          // kernel element size
  KernelFn fn = nullptr;
  int redop = -1;
  bool uniform = false;  // every thread block on the base lanes (LL with per-connection lanes)
  int64_t small_elems = 0, n_head = 0, n_big = 0;  // tapered tiles (see plan_call)
  int stage_bytes = 16 << 10;
  bool wq = false;  // work-queue mode (interp_wq)
  bool df = false;  // dataflow mode (interp_df_kernel)
  int weight = 0;        // units per lane: sum of multipliers, or thread blocks when uniform
};

ncclResult_t plan_call(Comm* c, DeviceState& ds, int id, int coll, size_t count, int dtype, int redop, int weight, bool sys_scope,
                       CallPlan& cp) {
  const RankIR& ir = *c->irs[id];
  const Program& p = ir.prog;
  const size_t esize = dtype_size(dtype);
  int64_t ce = chunk_elems_for(p, coll, count, c->nranks);
  if (ce < 0) return set_error(ncclInvalidArgument, "count %zu does not divide into the IR's chunks", count);
  cp.id = id;
  cp.redop = ir.has_reduce ? redop : -1;
  if (ir.has_reduce && (redop < 0 || redop > 3)) return set_error(ncclInvalidArgument, "unsupported reduction op %d", redop);
  if (ir.has_reduce && (dtype == ncclFloat8e4m3 || dtype == ncclFloat8e5m2))
    return set_error(ncclInvalidArgument, "fp8 reductions are not supported");
  // copy-only programs run the byte kernel: element = 1 byte
  cp.kesize = ir.has_reduce ? static_cast<int>(esize) : 1;
  const int64_t chunk_bytes = ce * static_cast<int64_t>(esize);
  cp.chunk_elems = chunk_bytes / cp.kesize;
  // protocol: the override, else the IR's tag; a Simple IR with many thread blocks per rank (many
  // short chains, e.g. 8 channels x 4 instances) runs LL for messages up to ll_max_bytes per rank
  // and LL128 up to ll128_max_bytes (no fences on the data path: C4's program 1 MiB 52 -> 32 us,
  // 2 MiB 71 -> 44 us); narrower programs only up to ll_narrow_max_bytes (Simple measured faster
  // above 16-32 KiB for one ring, all-pairs, hierarchical, two-step, ring AG / RS)
  int proto = ir.proto_override >= 0 ? ir.proto_override : static_cast<int>(p.proto);
  if (ir.proto_override < 0 && proto == kProtoSimple) {
    const uint64_t sb = selection_bytes(coll, count, esize, c->nranks);
    size_t tbs_rank = 0, ops_tb = 0;
    for (const auto& g : p.gpus) {
      tbs_rank = std::max(tbs_rank, g.tbs.size());
      for (const auto& tb : g.tbs) ops_tb = std::max(ops_tb, tb.ops.size());
    }
    const bool wide = static_cast<int64_t>(tbs_rank) >= c->cfg.ll_wide_tbs;
    // (narrow programs with short op lists — all-pairs, hierarchical, two-step — measured faster on
    // Simple at every size tried; long sequential chains gain from LL's cheaper hops)
    const int64_t ll_max = wide ? c->cfg.ll_max_bytes
                                : ops_tb >= 8 ? std::min(c->cfg.ll_max_bytes, c->cfg.ll_narrow_max_bytes) : 0;
    const int64_t ll128_max = wide ? c->cfg.ll128_max_bytes : 0;
    if (ll_max > 0 && sb <= static_cast<uint64_t>(ll_max)) proto = kProtoLL;
    else if (ll128_max > 0 && sb <= static_cast<uint64_t>(ll128_max)) proto = kProtoLL128;
  }
  // line protocols move 8-byte words: chunks of other sizes run Simple
  cp.proto = proto != kProtoSimple && chunk_bytes % 8 == 0 ? proto : kProtoSimple;
  cp.ll = cp.proto != kProtoSimple;
  // an LL launch sends every message through lane-matched FIFOs: with per-connection lane counts
  // (lane_mask) it runs every thread block on the base lanes instead
  int ntbs_local = 0;
  for (int r = 0; r < c->nranks; ++r)
    if (c->clique->local[r] && c->clique->local[r]->device == ds.device) ntbs_local += static_cast<int>(p.gpus[r].tbs.size());
  cp.uniform = cp.ll && ir.lane_mask != 0;
  // payload bytes of one tile that fit the protocol's slot unit (slots scale with count)
  const int64_t unit = proto_unit(cp.proto, ir.slot_bytes);
  const int64_t cap_bytes = cp.proto == kProtoLL ? unit / 2 : cp.proto == kProtoLL128 ? unit / 128 * 120 : unit;
  int64_t tile_bytes_cap = cap_bytes / 16 * 16;
  if (tile_bytes_cap < 16) return set_error(ncclInvalidUsage, "FIFO slot unit too small");
  cp.fn = interp_kernel(cp.redop < 0 ? 0 : dtype, cp.redop, cp.proto);
  if (!cp.fn) return set_error(ncclInvalidArgument, "no kernel for dtype %d op %d", dtype, redop);
  auto occupancy = [&](size_t smem) {
    auto f = ds.occupancy.find({cp.fn, smem});
    if (f == ds.occupancy.end()) f = ds.occupancy.emplace(std::make_pair(cp.fn, smem), interp_blocks_per_sm(cp.fn, smem)).first;
    return f->second;
  };
  const int bps_plain = occupancy(0);
  if (!cp.uniform && weight > ntbs_local) {
    // balanced lanes only where they fit: if the multipliers leave much of the GPU idle (or do not
    // fit at all) at 4-warp units, every thread block runs the base lanes instead
    const int cap4 = bps_plain * ds.num_sms * (kThreads / 32 / 4);
    const int lb = std::min(cap4 / weight, ir.lanes), lu = std::min(cap4 / ntbs_local, ir.lanes);
    if (lb < 1 || 4LL * lb * weight < 3LL * lu * ntbs_local) cp.uniform = true;
  }
  if (cp.uniform) weight = ntbs_local;
  cp.weight = weight;
  // units: `unit_warps` warps interpret one (thread block, lane); all units must be co-resident
  int uw = c->cfg.unit_warps;
  if (uw <= 0) {  // automatic: reductions move two operands per element, give them wider units
    uw = 4;
    while (uw > 1 && bps_plain * ds.num_sms * (kThreads / 32 / uw) < weight) uw /= 2;
  }
  if (uw < 1 || uw > kThreads / 32 || (kThreads / 32) % uw) uw = kThreads / 32;
  const int units_per_block = kThreads / 32 / uw;
  // TMA staging for pure-copy ops (same-device peers; shared-memory stages per unit)
  cp.tma_stages = 0;
  // three or more stages per unit: 16 KiB stages for wide units, smaller ones (>= 4 KiB) when
  // many narrow units share the SM's shared memory
  // reductions stream two operands per piece: fewer, larger stages (2 x 24 KiB per 4-warp unit in
  // 216 KiB) measured 3-4% faster on C3/C4/C5-RS; copies keep 3 x 16 KiB in 192 KiB
  const bool wide = ir.has_reduce && c->cfg.smem_kb == 192 && c->cfg.stage_kb <= 0 && units_per_block == 4;
  const int budget = static_cast<int>(std::min<int64_t>(wide ? 216 : c->cfg.smem_kb, 220)) << 10;
  cp.stage_bytes = c->cfg.stage_kb > 0 ? static_cast<int>(c->cfg.stage_kb) << 10
                   : wide             ? 24 << 10
                                      : std::max(4 << 10, std::min(kStageBytesHost, budget / (units_per_block * 3) / 1024 * 1024));
  // (thread blocks with a cross-GPU connection use them only with config tma_remote: LaunchArgs::tma_sys_ops)
  if (c->cfg.tma) cp.tma_stages = std::min(kMaxStagesHost, budget / (units_per_block * cp.stage_bytes));
  cp.smem = static_cast<size_t>(units_per_block) * cp.tma_stages * cp.stage_bytes;
  int bps = occupancy(cp.smem);
  if (bps * ds.num_sms * units_per_block < weight && cp.smem) {  // staging would break co-residency
    cp.tma_stages = 0;
    cp.smem = 0;
    bps = bps_plain;
  }
  const int capacity = bps * ds.num_sms * units_per_block;
  if (capacity < weight)
    return set_error(ncclInvalidUsage, "%d thread-block lanes cannot be co-resident (capacity %d units)", weight, capacity);
  // aim for every resident warp busy: one unit per unit_warps resident warps
  const int target_units = bps * ds.num_sms * (kThreads / 32) / uw;
  int lanes = c->cfg.lanes > 0 ? c->cfg.lanes : std::max(1, target_units / std::max(1, weight));
  lanes = std::min({lanes, ir.lanes, capacity / weight});
  lanes = std::max(lanes, 1);
  int64_t tile_bytes;
  if (c->cfg.tile_bytes > 0) {
    tile_bytes = std::min<int64_t>(c->cfg.tile_bytes / 16 * 16, tile_bytes_cap);
  } else {  // one tile per lane when it fits a slot; larger chunks give each lane several tiles,
            // which pipeline through multi-hop chains in op-major groups. The tile count is a
            // multiple of every thread block's lane count (lanes x multiplier), so all lanes of a
            // thread block get the same number of tiles (no straggler lane).
    int lcm = 1;
    if (!cp.uniform)
      for (const auto& g : ir.mult)
        for (int m : g) lcm = std::lcm(lcm, std::max(m, 1));
    const int64_t lanes_all = static_cast<int64_t>(lanes) * lcm;
    int64_t k = std::max<int64_t>(1, (chunk_bytes + lanes_all * tile_bytes_cap - 1) / (lanes_all * tile_bytes_cap));
    // few lanes on multi-hop chains (e.g. 32 rings per rank in loopback): the chain fills per lane,
    // so give every lane a deep pipeline of >= 64 KiB tiles (measured: C4 0.55 -> 0.43 ms)
    if (ir.has_chain && lanes_all <= 4) k = std::max<int64_t>(k, std::min<int64_t>(16, chunk_bytes / (lanes_all * (64 << 10))));
    tile_bytes = (chunk_bytes + lanes_all * k - 1) / (lanes_all * k);
    tile_bytes = std::max<int64_t>(tile_bytes, 4 << 10);
    tile_bytes = align_up(static_cast<size_t>(std::max<int64_t>(tile_bytes, 16)), 16);
    tile_bytes = std::min<int64_t>(tile_bytes, tile_bytes_cap);
  }
  tile_bytes = std::max<int64_t>(tile_bytes, 16);
  if (chunk_bytes <= tile_bytes) tile_bytes = chunk_bytes;
  if (cp.ll && tile_bytes % 8) tile_bytes = tile_bytes / 8 * 8;
  cp.tile_elems = std::max<int64_t>(tile_bytes / cp.kesize, chunk_bytes > 0 ? 1 : 0);
  cp.ntiles = cp.tile_elems > 0 ? (cp.chunk_elems + cp.tile_elems - 1) / cp.tile_elems : 0;
  cp.small_elems = cp.tile_elems;
  cp.n_head = 0;
  cp.n_big = cp.ntiles;
  {  // tapered tiles: the first and the last round of every lane use quarter tiles, so pipelines
     // fill and drain in a quarter of the time (the drain is one unit moving its last tile alone)
    int lcm = 1;
    if (!cp.uniform)
      for (const auto& g : ir.mult)
        for (int m : g) lcm = std::lcm(lcm, std::max(m, 1));
    const int64_t lanes_all = static_cast<int64_t>(lanes) * lcm;
    const int64_t T = cp.tile_elems, C = cp.chunk_elems;
    const int64_t align = std::max<int64_t>(1, 16 / cp.kesize);
    const int64_t ts = (T / 4) / align * align;
    const int64_t round_small = 4 * lanes_all * ts;  // one round of quarter tiles
    if (c->cfg.taper && c->cfg.tile_bytes <= 0 && !cp.ll && ts * cp.kesize >= (4 << 10) && C >= 2 * round_small + 2 * lanes_all * T) {
      const int64_t nh = 4 * lanes_all;
      const int64_t nb = (C - 2 * round_small) / T;
      const int64_t rest = C - nh * ts - nb * T;
      const int64_t nt = (rest + ts - 1) / ts;
      cp.small_elems = ts;
      cp.n_head = nh;
      cp.n_big = nb;
      cp.ntiles = nh + nb + nt;
    }
  }
  if (cp.ntiles < lanes) lanes = static_cast<int>(std::max<int64_t>(cp.ntiles, 1));
  cp.lanes = lanes;
  cp.unit_warps = uw;
  cp.grid = (weight * lanes + units_per_block - 1) / units_per_block;
  // op-major tile groups: the largest G (<= tiles of a lane) whose order is deadlock-free here
  const int64_t max_tiles = cp.ntiles > 0 ? (cp.ntiles + lanes - 1) / lanes : 0;
  // (groups only pay off where tiles pipeline through multi-hop chains; single-hop programs such as
  // AllToAll / two-step run tile-major)
  int G = c->cfg.group > 0 ? c->cfg.group
                           : (ir.has_chain ? static_cast<int>(std::min<int64_t>(std::max<int64_t>(max_tiles, 1), 64)) : 1);
  RankIR& mir = *c->irs[id];
  for (; G > 1; G /= 2) {
    // LL launches move every message through the FIFO lines (no direct / pulled transports)
    const auto key = std::make_tuple(cp.ntiles, lanes, G, ir.slots, cp.ll);
    auto f = mir.order_ok.find(key);
    if (f == mir.order_ok.end())
      f = mir.order_ok
              .emplace(key, order_is_deadlock_free(p, cp.ll ? std::vector<std::vector<std::vector<uint8_t>>>() : mir.eff_direct,
                                                   cp.ntiles, lanes, cp.uniform ? std::vector<std::vector<int>>() : mir.mult,
                                                   G, ir.slots))
              .first;
    if (f->second) break;
  }
  cp.group = std::max(G, 1);
  // work-queue mode: every co-resident unit claims (thread block, tile) items until none is left
  cp.wq = false;
  const bool wq_ok = ds.plans.size() > static_cast<size_t>(id) && ds.plans[id].wq_ok;
  // (chains of receive-and-forward ops run better on static lanes: measured on ring AllGather /
  // ReduceScatter; phase-structured programs such as the two-step AllToAll gain: C2 0.31 -> 0.29 ms)
  KernelFn wq_fn = interp_kernel_wq(cp.redop);
  if (c->cfg.wq && wq_ok && wq_fn && (!ir.has_chain || c->cfg.wq > 1) && !cp.ll && !sys_scope && c->cfg.lanes <= 0 &&
      capacity >= ntbs_local && chunk_bytes > 0 && interp_blocks_per_sm(wq_fn, cp.smem) >= bps) {
    cp.wq = true;
    cp.fn = wq_fn;
    cp.uniform = true;
    const int units = capacity;
    int64_t tb_bytes = c->cfg.tile_bytes > 0 ? c->cfg.tile_bytes / 16 * 16
                                              : chunk_bytes * ntbs_local / (static_cast<int64_t>(std::max(1, c->cfg.wq_items)) * units);
    tb_bytes = std::min<int64_t>(std::max<int64_t>(tb_bytes, 32 << 10), 1 << 20);
    tb_bytes = align_up(static_cast<size_t>(tb_bytes), 16);
    if (chunk_bytes <= tb_bytes) tb_bytes = chunk_bytes;
    cp.tile_elems = std::max<int64_t>(tb_bytes / cp.kesize, 1);
    cp.ntiles = (cp.chunk_elems + cp.tile_elems - 1) / cp.tile_elems;
    cp.small_elems = cp.tile_elems;
    cp.n_head = 0;
    cp.n_big = cp.ntiles;
    cp.lanes = 1;
    cp.weight = units;
    cp.group = 1;
    cp.grid = (units + units_per_block - 1) / units_per_block;
  }
  // dataflow mode: every co-resident unit runs ready (op, tile) items (interp_df_kernel)
  cp.df = false;
  const bool df_ok = ds.plans.size() > static_cast<size_t>(id) && ds.plans[id].df_ok;
  KernelFn df_fn = df_ok ? interp_kernel_df(cp.redop < 0 ? 0 : dtype, cp.redop) : nullptr;
  // df 1 (default): reducing programs with receive-and-forward chains (measured on B200: C3 1.61 ->
  // 1.39 ms, C4 0.377 -> 0.335 ms, C5-RS 0.230 -> 0.228 ms; the copy-only ring AllGather runs faster
  // on static lanes) when the launch has at least two items per unit and 16 tiles per chunk (C4 at 16
  // / 32 MiB per rank, 4 / 8 tiles: 247 / 266 us dataflow vs 177 / 243 us static lanes); df 2: every
  // Simple program
  const int df_units = capacity;
  int64_t df_tile = 0;
  bool use_df = c->cfg.df && df_fn && !cp.ll && !sys_scope && c->cfg.lanes <= 0 && chunk_bytes > 0 &&
                interp_blocks_per_sm(df_fn, cp.smem) >= bps;
  if (use_df) {
    // enough tiles that the graph's average width (nodes / depth) x tiles gives every unit
    // df_items ready items at a time, within [df_min_tile, df_max_tile]
    const int64_t width = std::max<int64_t>(1, ds.plans[id].df_n / std::max(1, ds.plans[id].df_depth));
    df_tile = c->cfg.tile_bytes > 0 ? c->cfg.tile_bytes
                                    : chunk_bytes * width / (static_cast<int64_t>(std::max(1, c->cfg.df_items)) * df_units);
    df_tile = std::min<int64_t>(std::max<int64_t>(df_tile, c->cfg.df_min_tile), c->cfg.df_max_tile);
    // programs whose buffers far exceed the L2 keep fewer bytes per tile in flight, so a producer's
    // span is still in L2 when its consumer reads it (C3, 2 GiB of buffers: 128 KiB tiles 8.9 GB of
    // DRAM traffic per launch and 1.39 ms, 64 KiB tiles 7.3 GB and 1.25 ms)
    const int64_t footprint = static_cast<int64_t>(p.ranks()) * (p.nchunks[0] + (p.inplace ? 0 : p.nchunks[1]) + p.nchunks[2]) * chunk_bytes;
    if (c->cfg.tile_bytes <= 0 && footprint >= c->cfg.df_big_bytes) df_tile = std::min<int64_t>(df_tile, c->cfg.df_big_tile);
    df_tile = std::max<int64_t>(df_tile / 128 * 128, 128);  // whole L2 lines (mailbox discard, bulk alignment)
    // whole waves: a chain program's items run level by level (width items per tile per level), so
    // width x tiles just above a multiple of the units leaves a partial wave at every level (C4,
    // width 32 on 592 units: 20 tiles 0.425 ms, 16 tiles 0.314 ms, 18 tiles 0.303 ms). When about
    // one wave per level fits, round the tile count to units / width if that moves the tile by
    // <= 25 % (several waves per level overlap: C5-RS, 64 -> 74 tiles, measured 1 % slower).
    if (c->cfg.tile_bytes <= 0 && c->cfg.df_waves && footprint < c->cfg.df_big_bytes && chunk_bytes > df_tile) {
      const int64_t per_wave = df_units / width;  // tiles whose items fill one wave of units
      if (per_wave >= 1) {
        const int64_t tile1 = ((chunk_bytes + per_wave - 1) / per_wave + 127) / 128 * 128;
        const int64_t tiles0 = (chunk_bytes + df_tile - 1) / df_tile, tiles1 = (chunk_bytes + tile1 - 1) / tile1;
        // (never below the 16 tiles per chunk the dataflow choice below asks for)
        if (4 * tile1 >= 3 * df_tile && 4 * tile1 <= 5 * df_tile && tile1 <= c->cfg.df_max_tile && width * tiles1 <= df_units &&
            (tiles1 >= 16 || tiles1 >= tiles0))
          df_tile = tile1;
      }
    }
    if (chunk_bytes <= df_tile) df_tile = chunk_bytes;
    const int64_t items = static_cast<int64_t>(ds.plans[id].df_n) * ((chunk_bytes + df_tile - 1) / df_tile);
    const int64_t tiles = (chunk_bytes + df_tile - 1) / df_tile;
    if (c->cfg.df == 1) use_df = ir.has_chain && ir.has_reduce && items >= 2LL * df_units && tiles >= 16;
    // one wave per level (df_waves 2): a reducing chain program that runs dataflow anyway, or whose
    // static-lane plan has fewer than df_wave_max_lanes lanes (tiles that barely pipeline), runs on
    // the dataflow executor with exactly units ÷ width tiles when that tile is >= df_wave_min_tile
    // (measured, `profiles/r02bt_one_wave.jsonl`: C4's program 8 MiB 124 -> 88 us, 16 MiB 153 ->
    // 115 us, 32 MiB 213 -> 169 us, 96 MiB 530 -> 495 us; C3's 4 MiB 176 -> 78 us, 32 MiB 260 ->
    // 179 us; programs of few thread blocks keep their 64 static lanes: C1 / C5-RS at 4 MiB are
    // faster there)
    if (c->cfg.df == 1 && c->cfg.df_waves >= 2 && c->cfg.tile_bytes <= 0 && footprint < c->cfg.df_big_bytes && ir.has_chain &&
        ir.has_reduce && (use_df || cp.lanes < c->cfg.df_wave_max_lanes)) {
      const int64_t per_wave = df_units / width;
      const int64_t tile_w = per_wave >= 1 ? ((chunk_bytes + per_wave - 1) / per_wave + 127) / 128 * 128 : 0;
      if (per_wave >= 16 && tile_w >= c->cfg.df_wave_min_tile && tile_w <= c->cfg.df_max_tile && tile_w < chunk_bytes &&
          width * ((chunk_bytes + tile_w - 1) / tile_w) <= df_units) {
        df_tile = tile_w;
        use_df = true;
      }
    }
  }
  if (use_df) {
    cp.df = true;
    cp.wq = false;
    cp.fn = df_fn;
    cp.uniform = true;
    const int units = df_units;
    const int64_t tb_bytes = df_tile;
    cp.tile_elems = std::max<int64_t>(tb_bytes / cp.kesize, 1);
    cp.ntiles = (cp.chunk_elems + cp.tile_elems - 1) / cp.tile_elems;
    cp.small_elems = cp.tile_elems;
    cp.n_head = 0;
    cp.n_big = cp.ntiles;
    cp.lanes = 1;
    cp.weight = units;
    cp.group = 1;
    cp.grid = (units + units_per_block - 1) / units_per_block;
  }
  // every op below the bulk-engine threshold takes the register path: launch without staging memory
  // (measured: small LL calls 37 -> 33 us)
  if (cp.tile_elems * cp.kesize * ir.max_count < c->cfg.tma_min) {
    cp.tma_stages = 0;
    cp.smem = 0;
  }
  return ncclSuccess;
}

ncclResult_t ensure_buffer(Comm* c, char*& buf, size_t& have, size_t need) {
  if (need <= have) return ncclSuccess;
  DeviceGuard g(c->device);
  if (buf) CUDA_TRY(cudaFree(buf));
  buf = nullptr;
  have = 0;
  CUDA_TRY(cudaMalloc(&buf, need));
  have = need;
  return ncclSuccess;
}

// Launches one group's collectives that live on one device.
// The (cached) event a participating stream records before a launch on another stream waits on it.
ncclResult_t stream_event(DeviceState& ds, cudaStream_t s, cudaEvent_t& ev) {
  auto f = ds.stream_events.find(s);
  if (f == ds.stream_events.end()) {
    CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    ds.stream_events[s] = ev;
  } else {
    ev = f->second;
  }
  return ncclSuccess;
}

// Per-call exchange of the launch buffers with the ranks of other launches (remote direct and
// pulled messages, see export_buffer): every local rank posts (registration, offset) of its five
// launch buffers as its next call record, then each remote rank's record of the same call is read
// and its buffers are opened into the launch's remote slots. anchor[slot] (non-null): the result
// buffer is recvbuff `anchor` shifted (ReduceScatter result_writes).
ncclResult_t exchange_buffers(Clique* cl, const DevicePlan& plan, LaunchArgs& a, const std::vector<char*>& anchor) {
  Comm* c0 = cl->local[plan.ranks[0]];
  CallRank* tab = nullptr;
  NCCL_TRY(call_table(c0, tab));
  const int64_t tmo = c0->cfg.timeout_ms + 60000;
  uint64_t seq = 0;
  for (size_t slot = 0; slot < plan.ranks.size(); ++slot) {
    Comm* c = cl->local[plan.ranks[slot]];
    const uint64_t sq = ++c->xcall_seq;
    if (slot > 0 && sq != seq) return set_error(ncclInternalError, "ranks of one launch disagree on the call sequence");
    seq = sq;
    if (sq > static_cast<uint64_t>(kCallRing)) {  // never overwrite a record a peer has not read yet
      const uint64_t need = sq - kCallRing;
      const bool ok = spin_until([&] {
        for (int r = 0; r < cl->nranks; ++r)
          if (r != c->rank && tab[r].done.load(std::memory_order_acquire) < need) return false;
        return true;
      }, tmo);
      if (!ok) return set_error(ncclSystemError, "timed out waiting for peers to read call %llu's buffers", static_cast<unsigned long long>(need));
    }
    CallRec& rec = tab[c->rank].rec[sq % kCallRing];
    for (int b = 0; b < kBufs; ++b) {
      const char* p = a.bufs[slot][b];
      const char* anc = (b == kResult && anchor[slot]) ? anchor[slot] : p;
      int32_t reg = -1;
      int64_t off = 0;
      NCCL_TRY(export_buffer(c, anc, reg, off));
      rec.reg[b] = reg;
      rec.off[b] = off + (p - anc);
    }
    rec.seq.store(sq, std::memory_order_release);
  }
  for (size_t i = 0; i < plan.remote_ranks.size(); ++i) {
    const int r = plan.remote_ranks[i];
    CallRec& rec = tab[r].rec[seq % kCallRing];
    if (!spin_until([&] { return rec.seq.load(std::memory_order_acquire) == seq; }, tmo))
      return set_error(ncclSystemError, "timed out waiting for rank %d's buffers of call %llu (collectives issued in different orders?)", r,
                       static_cast<unsigned long long>(seq));
    const size_t vs = plan.ranks.size() + i;
    for (int b = 0; b < kBufs; ++b) {
      char* base = nullptr;
      NCCL_TRY(peer_buffer(c0, r, rec.reg[b], base));
      a.bufs[vs][b] = base ? base + rec.off[b] : nullptr;
    }
  }
  for (int r : plan.ranks) tab[r].done.store(seq, std::memory_order_release);
  return ncclSuccess;
}

struct NvtxRange {  // one range per collective launch (SURVEY.md §5 tracing)
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

ncclResult_t launch_device(Clique* cl, int dev, std::vector<Pending*>& ops) {
  char range_name[96];
  std::snprintf(range_name, sizeof(range_name), "gc3 %s count=%zu dev=%d ranks=%zu", coll_name(ops[0]->coll), ops[0]->count, dev,
                ops.size());
  NvtxRange range(range_name);
  DeviceState* ds = nullptr;
  NCCL_TRY(device_state(cl, dev, ds));
  Comm* c0 = ops[0]->comm;
  const Pending& p0 = *ops[0];
  for (Pending* q : ops) {
    if (q->coll != p0.coll || q->count != p0.count || q->dtype != p0.dtype || q->redop != p0.redop)
      return set_error(ncclInvalidUsage, "ranks on one device issued mismatched collectives in a group");
    if (q->comm->async_error != ncclSuccess) return set_error(q->comm->async_error, "communicator is in an error state");
  }
  if (p0.count == 0) return ncclSuccess;
  if (ds->h_err && reinterpret_cast<volatile uint64_t*>(ds->h_err)[0]) {
    // a previous launch on this device hit the watchdog: its abort flag is still raised, so a new
    // launch would exit early and leave recvbuff unwritten; fail the call instead
    for (Pending* q : ops) q->comm->async_error = ncclSystemError;
    return set_error(ncclSystemError, "a previous collective on device %d timed out (watchdog); abort the communicator", dev);
  }
  const int id = select_ir(c0, p0.coll, p0.count, p0.dtype);
  if (id < 0)
    return set_error(ncclInvalidUsage, "no registered %s IR matches %zu elements of type %d (no NCCL fallback on this path)",
                     coll_name(p0.coll), p0.count, p0.dtype);
  NCCL_TRY(build_plan(cl, *ds, id));
  DevicePlan& plan = ds->plans[id];
  if (plan.ranks.size() != ops.size())
    return set_error(ncclInvalidUsage, "all %zu ranks hosted on device %d must issue the collective in one group (got %zu)",
                     plan.ranks.size(), dev, ops.size());
  CallPlan cp;
  NCCL_TRY(plan_call(c0, *ds, id, p0.coll, p0.count, p0.dtype, p0.redop, plan.weight, plan.sys_scope, cp));
  const RankIR& ir0 = *c0->irs[id];
  const size_t esize = dtype_size(p0.dtype);
  const int64_t chunk_bytes = cp.chunk_elems * cp.kesize;
  bool ragged = false;
  const int64_t ce = chunk_elems_for(ir0.prog, p0.coll, p0.count, c0->nranks, &ragged);
  const int cblk = (p0.coll == kAllReduce || p0.coll == kAllGather) ? ir0.prog.nchunks[0] : ir0.prog.nchunks[0] / c0->nranks;
  // ragged AllReduce on the caller's buffer: tiles clipped at the block's end (16-byte multiples
  // keep the bulk, LL and LL128 paths valid) instead of staging through padded work buffers
  const bool clip = ragged && p0.coll == kAllReduce && c0->cfg.clip && ir0.clip_ok && !cp.wq &&
                    (p0.count * esize) % 16 == 0 && (static_cast<size_t>(ce) * esize) % 16 == 0;
  struct PostCopy {  // result copies after the launch (cudaMemcpy2DAsync arguments)
    char* dst;
    size_t dpitch;
    const char* src;
    size_t spitch, width, rows;
  };
  std::vector<PostCopy> post;
  std::vector<char*> anchor(plan.ranks.size(), nullptr);

  LaunchArgs a{};
  a.tbs = plan.d_tbs;
  a.ops = plan.d_ops;
  a.deps = plan.d_deps;
  a.clip_elems = clip ? static_cast<int64_t>(p0.count * esize / cp.kesize) : 0;
  a.chans = plan.d_chans;
  a.sems = plan.d_sems;
  a.ntbs = plan.ntbs;
  a.weight = cp.weight;
  a.uniform = cp.uniform ? 1 : 0;
  a.wq = cp.wq ? 1 : 0;
  a.lanes = cp.lanes;
  a.unit_warps = cp.unit_warps;
  a.group = cp.group;
  a.tma_stages = cp.tma_stages;
  a.stage_bytes = cp.stage_bytes;
  a.tma_ops = c0->cfg.tma;
  a.tma_sys_ops = c0->cfg.tma_remote ? 0xff : 0;
  a.tma_min = c0->cfg.tma_min;
  a.l2hint = c0->cfg.l2hint;
  a.discard = c0->cfg.discard;
  // LL: every message travels as flagged lines through the receiver's FIFO (lowest latency, no
  // fences); Simple: direct and pulled messages where the plan found them safe
  a.transports = cp.ll ? 0 : 0xff;
  a.slots = ir0.slots;
  a.sys_scope = plan.sys_scope ? 1 : 0;
  a.chunk_elems = cp.chunk_elems;
  a.tile_elems = cp.tile_elems;
  a.ntiles = cp.ntiles;
  a.small_elems = cp.small_elems;
  a.n_head = cp.n_head;
  a.n_big = cp.n_big;
  a.epoch = ++ds->epoch;
  a.epoch_ptr = ds->d_epoch;
  a.epoch_ctr = ds->d_epoch_ctr;
  a.timeout_ns = static_cast<uint64_t>(c0->cfg.timeout_ms) * 1000000ull;
  a.abort_flag = ds->d_abort;
  a.err_info = ds->d_err;
  if (c0->cfg.trace) {
    int max_nops = 0;
    for (int r : plan.ranks)
      for (const auto& tb : c0->irs[id]->prog.gpus[r].tbs) max_nops = std::max(max_nops, static_cast<int>(tb.ops.size()));
    int ops_per_block = static_cast<int>(std::min<int64_t>((cp.ntiles + cp.lanes - 1) / cp.lanes * max_nops, 1 << 20));
    int rows = cp.weight * cp.lanes;
    if (cp.df) {  // dataflow: one row per (node, tile) item: claim, ready, moved, published
      rows = static_cast<int>(plan.df_n * cp.ntiles);
      ops_per_block = 1;
    }
    const size_t need = static_cast<size_t>(rows) * ops_per_block * 4 * sizeof(uint64_t);
    DeviceGuard gt(dev);
    if (need > ds->trace_bytes) {
      if (ds->d_trace) cudaFree(ds->d_trace);
      ds->d_trace = nullptr;
      ds->trace_bytes = 0;
      CUDA_TRY(cudaMalloc(&ds->d_trace, need));
      ds->trace_bytes = need;
    }
    CUDA_TRY(cudaMemsetAsync(ds->d_trace, 0, need, p0.stream));
    a.trace = ds->d_trace;
    a.trace_ops = ops_per_block;
    ds->trace_grid = rows;
    ds->trace_ops = ops_per_block;
    ds->trace_lanes = cp.lanes;
  }
  // LaunchArgs::sems are indexed with the lane count used when the plan was built (ir.lanes); the
  // kernel adds its lane (< cp.lanes <= ir.lanes) to each tb's base.
  cudaStream_t stream = p0.stream;
  DeviceGuard g(dev);
  // order every participating stream before the launch stream
  std::vector<cudaStream_t> others;
  for (Pending* q : ops)
    if (q->stream != stream && std::find(others.begin(), others.end(), q->stream) == others.end()) others.push_back(q->stream);
  for (cudaStream_t s : others) {
    cudaEvent_t ev = nullptr;
    NCCL_TRY(stream_event(*ds, s, ev));
    CUDA_TRY(cudaEventRecord(ev, s));
    CUDA_TRY(cudaStreamWaitEvent(stream, ev, 0));
  }
  // serialise with the previous launch of this device when it went to another stream (same stream:
  // stream order suffices). Under stream capture the graph's own edges order the launches.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CUDA_TRY(cudaStreamIsCapturing(stream, &cap));
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  if (!capturing && ds->has_last && ds->last_stream != stream) CUDA_TRY(cudaStreamWaitEvent(stream, ds->last_done, 0));
  for (size_t slot = 0; slot < plan.ranks.size(); ++slot) {
    const int r = plan.ranks[slot];
    Pending* q = nullptr;
    for (Pending* x : ops)
      if (x->comm->rank == r) q = x;
    if (!q) return set_error(ncclInvalidUsage, "rank %d missing from the group", r);
    Comm* c = q->comm;
    const RankIR& ir = *c->irs[id];
    const size_t scratch_need = static_cast<size_t>(ir.prog.nchunks[2]) * chunk_bytes;
    NCCL_TRY(ensure_buffer(c, c->scratch, c->scratch_bytes, std::max<size_t>(scratch_need, 256)));
    char* in = nullptr;
    char* out = nullptr;
    // blk: one rank block of the user's buffers; pblk: the same block padded to c x ce elements
    // (equal unless the call is ragged, see chunk_elems_for)
    const size_t blk = p0.count * esize, pblk = static_cast<size_t>(cblk) * ce * esize;
    const int R = c->nranks;
    char* send = const_cast<char*>(static_cast<const char*>(q->send));
    char* recv = static_cast<char*>(q->recv);
    char* source = nullptr;  // what the in-place IR's first reads see (source_reads); null: `in`
    char* result = nullptr;  // ReduceScatter: recvbuff shifted to the owned block's offset (result_writes)
    switch (p0.coll) {
      case kAllReduce:  // in-place IR on `input` (core.hpp:305-327)
        if (ragged && !clip) {
          NCCL_TRY(ensure_buffer(c, c->work, c->work_bytes, pblk));
          CUDA_TRY(cudaMemcpyAsync(c->work, send, blk, cudaMemcpyDeviceToDevice, stream));
          in = out = c->work;
          post.push_back({recv, blk, c->work, pblk, blk, 1});
        } else {
          if (send != recv) {
            if (plan.source_complete) source = send;  // first reads come from sendbuff: no pre-copy
            else CUDA_TRY(cudaMemcpyAsync(recv, send, blk, cudaMemcpyDeviceToDevice, stream));
          }
          in = out = recv;
        }
        break;
      case kAllGather:
        if (ragged) {
          NCCL_TRY(ensure_buffer(c, c->work, c->work_bytes, pblk));
          NCCL_TRY(ensure_buffer(c, c->work2, c->work2_bytes, pblk * R));
          CUDA_TRY(cudaMemcpyAsync(c->work, send, blk, cudaMemcpyDeviceToDevice, stream));
          in = c->work;
          out = c->work2;
          post.push_back({recv, blk, c->work2, pblk, blk, static_cast<size_t>(R)});
        } else {
          in = send;
          out = recv;
        }
        break;
      case kReduceScatter:  // in-place IR over R*c chunks; rank r owns [r*c, (r+1)*c)
        NCCL_TRY(ensure_buffer(c, c->work, c->work_bytes, pblk * R));
        if (!ragged && plan.source_complete) source = send;  // first reads come from sendbuff
        else if (!ragged) CUDA_TRY(cudaMemcpyAsync(c->work, send, blk * R, cudaMemcpyDeviceToDevice, stream));
        else CUDA_TRY(cudaMemcpy2DAsync(c->work, pblk, send, blk, blk, R, cudaMemcpyDeviceToDevice, stream));
        in = out = c->work;
        // the owned block's final writes land in recvbuff: its chunk k sits at recvbuff + (k - r*c)*ce
        if (!ragged && plan.result_complete) result = recv - static_cast<ptrdiff_t>(c->rank) * static_cast<ptrdiff_t>(pblk);
        else post.push_back({recv, blk, c->work + static_cast<size_t>(c->rank) * pblk, pblk, blk, 1});
        break;
      case kAllToAll:
        if (q->send == q->recv) return set_error(ncclInvalidArgument, "in-place AllToAll is not supported");
        if (ragged) {
          NCCL_TRY(ensure_buffer(c, c->work, c->work_bytes, pblk * R));
          NCCL_TRY(ensure_buffer(c, c->work2, c->work2_bytes, pblk * R));
          CUDA_TRY(cudaMemcpy2DAsync(c->work, pblk, send, blk, blk, R, cudaMemcpyDeviceToDevice, stream));
          in = c->work;
          out = c->work2;
          post.push_back({recv, blk, c->work2, pblk, blk, static_cast<size_t>(R)});
        } else {
          in = send;
          out = recv;
        }
        break;
    }
    if (ir.prog.inplace) out = in;
    a.bufs[slot][0] = in;
    a.bufs[slot][1] = out;
    a.bufs[slot][2] = c->scratch;
    a.bufs[slot][kSource] = source ? source : in;
    a.bufs[slot][kResult] = result ? result : in;
    // the result base may lie outside recvbuff's allocation (shifted by the owned block's offset):
    // peers get it as recvbuff's registration plus that shift
    anchor[slot] = result ? recv : nullptr;
  }
  // (line-protocol launches move every message through the FIFO lines: nothing to exchange; every
  // rank decides this the same way, so the per-rank call sequences stay aligned)
  if (!plan.remote_ranks.empty() && !cp.ll) NCCL_TRY(exchange_buffers(cl, plan, a, anchor));
  if (cp.df) {  // ready-queue counters reset; self-resetting tables sized for this tile count; mailbox
    DeviceGuard gw(dev);
    const size_t items = static_cast<size_t>(plan.df_n) * static_cast<size_t>(cp.ntiles);
    if (items > ds->df_items_cap) {
      if (ds->d_df_cnt) CUDA_TRY(cudaFree(ds->d_df_cnt));
      if (ds->d_df_q) CUDA_TRY(cudaFree(ds->d_df_q));
      ds->d_df_cnt = ds->d_df_q = nullptr;
      ds->df_items_cap = 0;
      CUDA_TRY(cudaMalloc(&ds->d_df_cnt, items * sizeof(int32_t)));
      // queue positions: every pushed item plus one idle claim per unit at the end
      CUDA_TRY(cudaMalloc(&ds->d_df_q, (items + kDfQueueSlack) * sizeof(int32_t)));
      CUDA_TRY(cudaMemset(ds->d_df_cnt, 0, items * sizeof(int32_t)));
      CUDA_TRY(cudaMemset(ds->d_df_q, 0, (items + kDfQueueSlack) * sizeof(int32_t)));
      ds->df_items_cap = items;
    }
    const size_t mail_need = std::max<size_t>(static_cast<size_t>(plan.df_mail_chunks) * static_cast<size_t>(chunk_bytes), 256);
    if (mail_need > ds->mail_bytes) {
      if (ds->d_mail) CUDA_TRY(cudaFree(ds->d_mail));
      ds->d_mail = nullptr;
      ds->mail_bytes = 0;
      CUDA_TRY(cudaMalloc(&ds->d_mail, mail_need));
      ds->mail_bytes = mail_need;
    }
    if (!ds->d_wq_next) CUDA_TRY(cudaMalloc(&ds->d_wq_next, 1024));
    CUDA_TRY(cudaMemsetAsync(ds->d_wq_next, 0, 512, stream));  // four counters, one 128-byte line each
    a.df_nodes = plan.d_df_nodes;
    a.df_succ = plan.d_df_succ;
    a.df_roots = plan.d_df_roots;
    a.df_cnt = ds->d_df_cnt;
    a.df_q = ds->d_df_q;
    a.df_ctr = ds->d_wq_next;
    a.mail = ds->d_mail;
    a.df_n = plan.df_n;
    a.df_nroots = plan.df_nroots;
    a.df_policy = c0->cfg.df_policy;
    a.df_window = c0->cfg.df_window;
  }
  if (cp.wq) {  // claim counter reset + progress table (epoch-tagged, never reset)
    DeviceGuard gw(dev);
    const size_t need = static_cast<size_t>(plan.ntbs) * cp.ntiles * sizeof(uint64_t);
    if (!ds->d_wq_next) CUDA_TRY(cudaMalloc(&ds->d_wq_next, 1024));
    if (need > ds->prog_bytes) {
      if (ds->d_prog) CUDA_TRY(cudaFree(ds->d_prog));
      ds->d_prog = nullptr;
      ds->prog_bytes = 0;
      CUDA_TRY(cudaMalloc(&ds->d_prog, need));
      CUDA_TRY(cudaMemset(ds->d_prog, 0, need));
      ds->prog_bytes = need;
    }
    CUDA_TRY(cudaMemsetAsync(ds->d_wq_next, 0, sizeof(int32_t), stream));
    a.wq_next = ds->d_wq_next;
    a.prog = ds->d_prog;
    a.wq_order = nullptr;
    const int lag = c0->cfg.wq_lag;
    if (lag > 0) {  // items of a deeper thread block are claimed `lag` tiles later: fewer blocked units
      auto key = std::make_pair(cp.ntiles, lag);
      auto f = plan.wq_order.find(key);
      if (f == plan.wq_order.end()) {
        const int nt = plan.ntbs;
        std::vector<std::pair<int64_t, int32_t>> items;
        items.reserve(static_cast<size_t>(nt) * cp.ntiles);
        for (int64_t tile = 0; tile < cp.ntiles; ++tile)
          for (int tb = 0; tb < nt; ++tb)
            items.push_back({(tile + static_cast<int64_t>(plan.wq_level[tb]) * lag) * nt + tb, static_cast<int32_t>(tile * nt + tb)});
        std::stable_sort(items.begin(), items.end());
        std::vector<int32_t> order(items.size());
        for (size_t i = 0; i < items.size(); ++i) order[i] = items[i].second;
        int32_t* d = nullptr;
        CUDA_TRY(cudaMalloc(&d, std::max<size_t>(order.size(), 1) * sizeof(int32_t)));
        CUDA_TRY(cudaMemcpy(d, order.data(), order.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        f = plan.wq_order.emplace(key, d).first;
      }
      a.wq_order = f->second;
    }
  }
  CUDA_TRY(interp_launch(cp.fn, a, cp.grid, cp.smem, stream));
  for (const PostCopy& pc : post)
    CUDA_TRY(cudaMemcpy2DAsync(pc.dst, pc.dpitch, pc.src, pc.spitch, pc.width, pc.rows, cudaMemcpyDeviceToDevice, stream));
  if (!capturing) {
    if (!ds->last_done) CUDA_TRY(cudaEventCreateWithFlags(&ds->last_done, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(ds->last_done, stream));
    ds->last_stream = stream;
    ds->has_last = true;
  }
  for (cudaStream_t s : others) {  // the launch stream's event: recorded once, waited on by every other stream
    if (!ds->launch_done) CUDA_TRY(cudaEventCreateWithFlags(&ds->launch_done, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(ds->launch_done, stream));
    CUDA_TRY(cudaStreamWaitEvent(s, ds->launch_done, 0));
  }
  return ncclSuccess;
}

// Validates a program against the communicator, sizes and allocates its arena and publishes it to
// the other processes of the clique (the part of gc3RegisterIR after parsing).
ncclResult_t register_program(Comm* comm, std::unique_ptr<RankIR> ir, int* ir_id) {
  Topology topo;
  topo.nodes = 1;
  topo.gpus_per_node = comm->nranks;
  topo.max_threadblocks = 148;
  topo.max_channels = 1 << 20;
  const auto issues = validate(ir->prog, topo);
  if (!issues.empty()) return set_error(ncclInvalidUsage, "IR %s fails validation: %s", ir->prog.name.c_str(), issues[0].c_str());
  if (ir->prog.collective != "allreduce" && ir->prog.collective != "allgather" && ir->prog.collective != "reducescatter" &&
      ir->prog.collective != "alltoall")
    return set_error(ncclInvalidUsage, "collective %s has no NCCL entry point", ir->prog.collective.c_str());
  {  // buffer shapes the NCCL entry points map onto (core.hpp:305-397): AllReduce and
     // ReduceScatter run in place on `input`, AllGather / AlltoAll out of place
    const Program& p = ir->prog;
    const int R = comm->nranks, cin = p.nchunks[0], cout = p.nchunks[1];
    const std::string& coll = p.collective;
    const char* bad = nullptr;
    if (cin < 1) bad = "nchunks.input must be >= 1";
    else if ((coll == "allreduce" || coll == "reducescatter") && !p.inplace) bad = "must be in place";
    else if ((coll == "allreduce" || coll == "reducescatter") && cout != cin) bad = "needs nchunks.output == nchunks.input";
    else if (coll == "reducescatter" && cin % R) bad = "needs nchunks.input divisible by the rank count";
    else if ((coll == "allgather" || coll == "alltoall") && p.inplace) bad = "must be out of place";
    else if (coll == "allgather" && cout != R * cin) bad = "needs nchunks.output == ranks x nchunks.input";
    else if (coll == "alltoall" && (cout != cin || cin % R)) bad = "needs nchunks.output == nchunks.input, divisible by the rank count";
    if (bad) return set_error(ncclInvalidUsage, "%s IR %s %s", coll.c_str(), p.name.c_str(), bad);
  }
  ir->clip_ok = ir->prog.collective == "allreduce";
  for (const auto& g : ir->prog.gpus)
    for (const auto& tb : g.tbs)
      for (const auto& op : tb.ops) {
        if (op_reduces(op.op)) ir->has_reduce = true;
        if (op_receives(op.op) && op_sends(op.op)) ir->has_chain = true;
        if (op_sends(op.op) || op_receives(op.op)) ir->max_count = std::max(ir->max_count, op.count);
        if (op.op != Opcode::nop && (op.count != 1 || op.src_off != op.dst_off)) ir->clip_ok = false;
      }
  if (ir->clip_ok) {  // every message lands in the chunk it left (same clip length at both ends)
    const auto snd = matched_senders(ir->prog);
    for (int r = 0; r < ir->prog.ranks(); ++r)
      for (size_t t = 0; t < ir->prog.gpus[r].tbs.size(); ++t)
        for (size_t s2 = 0; s2 < ir->prog.gpus[r].tbs[t].ops.size(); ++s2) {
          const auto& x = snd[r][t][s2];
          if (x.rank >= 0 && ir->prog.gpus[x.rank].tbs[x.tb].ops[x.step].src_off != ir->prog.gpus[r].tbs[t].ops[s2].src_off)
            ir->clip_ok = false;
        }
  }
  ir->slots = std::max(1, comm->cfg.slots);
  ir->slot_bytes = std::max<int64_t>(comm->cfg.slot_bytes / 256 * 256, 256);
  {  // lanes provisioned: enough for ~2 CUDA blocks per SM when one rank owns a device
    int max_tbs = 1;
    for (const auto& g : ir->prog.gpus) max_tbs = std::max(max_tbs, static_cast<int>(g.tbs.size()));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, comm->device);
    ir->lanes = std::max(1, std::min(comm->cfg.max_lanes, (2 * sms + max_tbs - 1) / max_tbs));
  }
  {  // direct / pulled messages (and lanes that differ across their connections) only when every
     // rank runs in one launch: all ranks hosted here, on one device
    bool one_launch = true;
    for (int r = 0; r < comm->nranks; ++r)
      one_launch = one_launch && comm->clique->local[r] && comm->clique->local[r]->device == comm->device;
    ir->lane_mask = one_launch ? transport_mask(comm->cfg.direct) : 0;
  }
  ir->mult = comm->cfg.balance ? lane_multipliers(ir->prog, comm->cfg.balance, comm->cfg.mult_cap, ir->lane_mask)
                               : std::vector<std::vector<int>>();
  if (ir->mult.empty())
    for (const auto& g : ir->prog.gpus) ir->mult.emplace_back(g.tbs.size(), 1);
  ir->lay = make_layout(ir->prog, comm->rank, ir->lanes, ir->slots, ir->slot_bytes, ir->mult);
  {
    DeviceGuard g(comm->device);
    CUDA_TRY(cudaMalloc(&ir->arena, ir->lay.bytes));
    CUDA_TRY(cudaMemset(ir->arena, 0, ir->lay.bytes));
    CUDA_TRY(cudaDeviceSynchronize());
    // publish the arena to the other processes of the clique
    bool remote_peers = false;
    for (int r = 0; r < comm->nranks; ++r) remote_peers = remote_peers || !comm->clique->local[r];
    if (remote_peers) {
      CUDA_TRY(cudaIpcGetMemHandle(&ir->handle, ir->arena));
      const std::string rec(reinterpret_cast<const char*>(&ir->handle), sizeof(ir->handle));
      const int id = static_cast<int>(comm->irs.size());
      if (!post_record(shm_dir(comm->clique->key), "ir" + std::to_string(id) + ".rank" + std::to_string(comm->rank), rec))
        return set_error(ncclSystemError, "cannot publish arena handle");
    }
  }
  comm->irs.push_back(std::move(ir));
  if (ir_id) *ir_id = static_cast<int>(comm->irs.size()) - 1;
  return ncclSuccess;
}

// Built-in program for a call of `bytes` (selection bytes): comm-time generated, per size tier
// (the paper's mechanism: programs with disjoint size ranges, ir.hpp:112-116). With
// config gen (default) AllReduce uses four tiers, the measured best of the generated family on a
// B200 (8 ranks): up to gen_small bytes the ring on min(R, 8) channels x 4
// instances with LL lines (1 KiB: 28 us vs 65-80 us for one ring), up to gen_ll128 bytes the same
// program with LL128 lines (2 MiB: 58 us vs 86 us LL, 85 us one ring), up to gen_large bytes the
// single-channel ring (4 MiB: 87 us vs 100 us), above it the multi-channel ring again (Simple,
// dataflow mode: 64 MiB 0.33 ms vs 0.38 ms). Other collectives: the single-ring / direct programs.
bool builtin_for(const Config& cfg, const std::string& coll, int R, uint64_t bytes, Program& out) {
  if (!cfg.gen || coll != "allreduce") return builtin_program(coll, R, out);
  const int C = std::min(R, 8);
  const uint64_t small = static_cast<uint64_t>(cfg.gen_small), mid = std::max(small, static_cast<uint64_t>(cfg.gen_ll128)),
                 large = std::max(mid, static_cast<uint64_t>(cfg.gen_large));
  if (bytes <= small) {
    if (!generate_program("ring", coll, R, C, 4, out)) return false;
    out.proto = Proto::ll;
    out.min_bytes = 0;
    out.max_bytes = small;
  } else if (bytes <= mid) {
    if (!generate_program("ring", coll, R, C, 4, out)) return false;
    out.proto = Proto::ll128;
    out.min_bytes = small + 1;
    out.max_bytes = mid;
  } else if (bytes <= large) {
    if (!generate_program("ring", coll, R, 1, 1, out)) return false;
    out.min_bytes = mid + 1;
    out.max_bytes = large;
  } else {
    if (!generate_program("ring", coll, R, C, 4, out)) return false;
    out.min_bytes = large + 1;
    out.max_bytes = 1ull << 40;
  }
  return true;
}

// A call no registered IR matches runs the runtime's built-in program for its collective and size
// tier (builtin_for): registered here, before any launch of the group, on every communicator this
// process hosts in the clique, in rank order — every process meets the first such call of a
// collective and tier at the same point of the call sequence, so IR ids stay aligned across ranks.
ncclResult_t register_builtins(std::vector<Pending>& pend) {
  for (Pending& q : pend) {
    Comm* c = q.comm;
    if (!c->cfg.builtin || select_ir(c, q.coll, q.count, q.dtype) >= 0) continue;
    const std::string coll = coll_name(q.coll);
    const uint64_t bytes = selection_bytes(q.coll, q.count, dtype_size(q.dtype), c->nranks);
    for (int r = 0; r < c->nranks; ++r) {
      Comm* lc = c->clique->local[r];
      if (!lc) continue;
      bool have = false;
      for (const auto& ir : lc->irs)
        have = have || (ir->builtin && ir->prog.collective == coll && bytes >= ir->prog.min_bytes && bytes <= ir->prog.max_bytes);
      if (have) continue;
      auto ir = std::make_unique<RankIR>();
      if (!builtin_for(lc->cfg, coll, lc->nranks, bytes, ir->prog)) break;
      ir->builtin = true;
      NCCL_TRY(register_program(lc, std::move(ir), nullptr));
    }
  }
  return ncclSuccess;
}

ncclResult_t flush_group() {
  std::vector<Pending> pend;
  pend.swap(g_pending);
  NCCL_TRY(register_builtins(pend));
  std::map<std::pair<Clique*, int>, std::vector<Pending*>> by_dev;
  for (Pending& q : pend) by_dev[{q.comm->clique, q.comm->device}].push_back(&q);
  ncclResult_t rc = ncclSuccess;
  for (auto& [key, ops] : by_dev) {
    const ncclResult_t r = launch_device(key.first, key.second, ops);
    if (r != ncclSuccess && rc == ncclSuccess) rc = r;
  }
  return rc;
}

ncclResult_t enqueue(const Pending& q) {
  if (!q.comm || q.comm->destroyed) return set_error(ncclInvalidArgument, "invalid communicator");
  if (q.dtype < 0 || q.dtype >= ncclNumTypes) return set_error(ncclInvalidArgument, "invalid datatype %d", q.dtype);
  if (q.count > 0 && (!q.send || !q.recv)) return set_error(ncclInvalidArgument, "null buffer");
  if (q.coll == kAllReduce || q.coll == kReduceScatter) {
    if (q.redop == ncclAvg || q.redop < 0 || q.redop >= ncclNumOps) return set_error(ncclInvalidArgument, "unsupported reduction op %d", q.redop);
  }
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  g_pending.push_back(q);
  if (g_group_depth == 0) return flush_group();
  return ncclSuccess;
}

// ------------------------------------------------------------------------------- init
ncclResult_t make_comm(Clique* cl, int rank, int dev, Comm** out) {
  auto* c = new gc3Comm();
  c->clique = cl;
  c->rank = rank;
  c->nranks = cl->nranks;
  c->device = dev;
  c->cfg = config_from_env();
  cl->local[rank] = c;
  cl->rank_dev[rank] = dev;
  cl->rank_pid[rank] = getpid();
  cl->refs++;
  *out = c;
  return ncclSuccess;
}

}  // namespace
}  // namespace gc3

using namespace gc3;

// =============================================================================== C ABI
extern "C" {

ncclResult_t ncclGetVersion(int* version) {
  if (!version) return ncclInvalidArgument;
  *version = GC3_VERSION_CODE;
  return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t r) {
  switch (r) {
    case ncclSuccess: return "no error";
    case ncclUnhandledCudaError: return "unhandled cuda error (run with GC3_DEBUG=1 for details)";
    case ncclSystemError: return "unhandled system error (run with GC3_DEBUG=1 for details)";
    case ncclInternalError: return "internal error - please report this issue";
    case ncclInvalidArgument: return "invalid argument (run with GC3_DEBUG=1 for details)";
    case ncclInvalidUsage: return "invalid usage (run with GC3_DEBUG=1 for details)";
    case ncclRemoteError: return "remote process exited or there was a network error";
    case ncclInProgress: return "NCCL operation in progress";
    default: return "unknown result code";
  }
}

const char* ncclGetLastError(ncclComm_t) { return g_last_error.c_str(); }

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  if (!id) return ncclInvalidArgument;
  std::memset(id->internal, 0, sizeof(id->internal));
  std::memcpy(id->internal, "GC3", 4);
  FILE* f = std::fopen("/dev/urandom", "rb");
  size_t got = f ? std::fread(id->internal + 4, 1, 16, f) : 0;
  if (f) std::fclose(f);
  if (got != 16) {
    const uint64_t t = static_cast<uint64_t>(std::chrono::high_resolution_clock::now().time_since_epoch().count()) ^
                       (static_cast<uint64_t>(getpid()) << 32);
    std::memcpy(id->internal + 4, &t, 8);
  }
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  if (!comm || nranks < 1 || rank < 0 || rank >= nranks) return set_error(ncclInvalidArgument, "bad InitRank arguments");
  if (std::memcmp(id.internal, "GC3", 4) != 0) return set_error(ncclInvalidArgument, "unique id not created by ncclGetUniqueId");
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  const std::string key = uid_key(id);
  auto& slot = g_cliques[key];
  if (!slot) {
    slot = std::make_unique<Clique>();
    slot->key = key;
    slot->nranks = nranks;
    slot->local.assign(nranks, nullptr);
    slot->rank_dev.assign(nranks, -1);
    slot->rank_pid.assign(nranks, 0);
  }
  Clique* cl = slot.get();
  if (cl->nranks != nranks) return set_error(ncclInvalidArgument, "nranks mismatch for this unique id");
  if (cl->local[rank]) return set_error(ncclInvalidUsage, "rank %d initialised twice", rank);
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  Comm* c = nullptr;
  NCCL_TRY(make_comm(cl, rank, dev, &c));
  // publish (pid, device) and learn the peers'
  const std::string dir = shm_dir(key);
  if (!post_record(dir, "rank" + std::to_string(rank), std::to_string(getpid()) + " " + std::to_string(dev) + " " + device_bus_id(dev)))
    return set_error(ncclSystemError, "cannot write bootstrap record in %s", dir.c_str());
  *comm = c;
  return ncclSuccess;
}

ncclResult_t ncclCommInitAll(ncclComm_t* comms, int ndev, const int* devlist) {
  if (!comms || ndev < 1) return set_error(ncclInvalidArgument, "bad InitAll arguments");
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  const std::string key = uid_key(id);
  auto cl = std::make_unique<Clique>();
  cl->key = key;
  cl->nranks = ndev;
  cl->local.assign(ndev, nullptr);
  cl->rank_dev.assign(ndev, -1);
  cl->rank_pid.assign(ndev, getpid());
  std::set<int> devs;
  for (int r = 0; r < ndev; ++r) {
    const int dev = devlist ? devlist[r] : r;
    Comm* c = nullptr;
    NCCL_TRY(make_comm(cl.get(), r, dev, &c));
    comms[r] = c;
    devs.insert(dev);
  }
  // NVLink peer access between the distinct devices of this process
  for (int a : devs)
    for (int b : devs) {
      if (a == b) continue;
      int can = 0;
      CUDA_TRY(cudaDeviceCanAccessPeer(&can, a, b));
      if (!can) return set_error(ncclSystemError, "device %d cannot access peer %d", a, b);
      DeviceGuard g(a);
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CUDA_TRY(e);
      cudaGetLastError();
    }
  g_cliques[key] = std::move(cl);
  return ncclSuccess;
}

static void release_comm(Comm* c) {
  Clique* cl = c->clique;
  DeviceGuard g(c->device);
  for (void* p : c->opened_ipc) cudaIpcCloseMemHandle(p);
  for (auto& ir : c->irs)
    if (ir->arena) cudaFree(ir->arena);
  if (c->scratch) cudaFree(c->scratch);
  if (c->work) cudaFree(c->work);
  if (c->work2) cudaFree(c->work2);
  cl->local[c->rank] = nullptr;
  const std::string dir = shm_dir(cl->key);
  unlink((dir + "/rank" + std::to_string(c->rank)).c_str());
  for (size_t i = 0; i < c->irs.size(); ++i) unlink((dir + "/ir" + std::to_string(i) + ".rank" + std::to_string(c->rank)).c_str());
  for (size_t i = 0; i < c->regs.size(); ++i) unlink((dir + "/buf" + std::to_string(c->rank) + "." + std::to_string(i)).c_str());
  if (cl->refs == 1 && cl->calls) {  // the process's last rank of the clique: drop the call table
    munmap(cl->calls, cl->calls_bytes);
    cl->calls = nullptr;
    unlink((dir + "/calls").c_str());
  }
  rmdir(dir.c_str());  // succeeds for the last rank only
  c->destroyed = true;
  if (--cl->refs == 0) {
    for (auto& [dev, ds] : cl->devs) {
      DeviceGuard gd(dev);
      for (auto& p : ds.plans) {
        cudaFree(p.d_tbs);
        cudaFree(p.d_ops);
        cudaFree(p.d_deps);
        cudaFree(p.d_chans);
        cudaFree(p.d_sems);
        if (p.d_df_nodes) cudaFree(p.d_df_nodes);
        if (p.d_df_succ) cudaFree(p.d_df_succ);
        if (p.d_df_roots) cudaFree(p.d_df_roots);
        for (auto& [k, d] : p.wq_order) cudaFree(d);
      }
      cudaFree(ds.d_abort);
      if (ds.d_epoch) cudaFree(ds.d_epoch);
      if (ds.d_trace) cudaFree(ds.d_trace);
      if (ds.d_wq_next) cudaFree(ds.d_wq_next);
      if (ds.d_prog) cudaFree(ds.d_prog);
      if (ds.d_df_cnt) cudaFree(ds.d_df_cnt);
      if (ds.d_df_q) cudaFree(ds.d_df_q);
      if (ds.d_mail) cudaFree(ds.d_mail);
      if (ds.last_done) cudaEventDestroy(ds.last_done);
      if (ds.launch_done) cudaEventDestroy(ds.launch_done);
      for (auto& [st, ev] : ds.stream_events) cudaEventDestroy(ev);
      cudaFreeHost(ds.h_err);
    }
    g_cliques.erase(cl->key);
  }
  delete c;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  if (!comm) return ncclInvalidArgument;
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  {
    DeviceGuard g(comm->device);
    cudaDeviceSynchronize();
  }
  release_comm(comm);
  return ncclSuccess;
}

ncclResult_t ncclCommAbort(ncclComm_t comm) {
  if (!comm) return ncclInvalidArgument;
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  // raise the device abort flag so spinning blocks exit, then tear down
  auto it = comm->clique->devs.find(comm->device);
  if (it != comm->clique->devs.end() && it->second.d_abort) {
    DeviceGuard g(comm->device);
    const int one = 1;
    cudaMemcpy(it->second.d_abort, &one, sizeof(one), cudaMemcpyHostToDevice);
    cudaDeviceSynchronize();
  }
  release_comm(comm);
  return ncclSuccess;
}

ncclResult_t ncclCommGetAsyncError(ncclComm_t comm, ncclResult_t* err) {
  if (!comm || !err) return ncclInvalidArgument;
  *err = comm->async_error;
  auto it = comm->clique->devs.find(comm->device);
  if (*err == ncclSuccess && it != comm->clique->devs.end() && it->second.h_err) {
    volatile uint64_t* e = it->second.h_err;
    if (e[0]) {
      static const char* what[] = {"?", "dependency semaphore", "send slot credit", "receive slot", "LL line"};
      const uint64_t w = e[5] < 5 ? e[5] : 0;
      comm->async_error = ncclSystemError;
      set_error(ncclSystemError, "watchdog: launch rank-slot %llu tb %llu step %llu tile %llu timed out waiting on %s",
                (unsigned long long)e[1], (unsigned long long)e[2], (unsigned long long)e[3], (unsigned long long)e[4], what[w]);
      comm->last_error = g_last_error;
      *err = ncclSystemError;
    }
  }
  return ncclSuccess;
}

ncclResult_t ncclCommCount(const ncclComm_t comm, int* count) {
  if (!comm || !count) return ncclInvalidArgument;
  *count = comm->nranks;
  return ncclSuccess;
}
ncclResult_t ncclCommCuDevice(const ncclComm_t comm, int* device) {
  if (!comm || !device) return ncclInvalidArgument;
  *device = comm->device;
  return ncclSuccess;
}
ncclResult_t ncclCommUserRank(const ncclComm_t comm, int* rank) {
  if (!comm || !rank) return ncclInvalidArgument;
  *rank = comm->rank;
  return ncclSuccess;
}

ncclResult_t ncclGroupStart(void) {
  ++g_group_depth;
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd(void) {
  if (g_group_depth <= 0) return set_error(ncclInvalidUsage, "ncclGroupEnd without ncclGroupStart");
  if (--g_group_depth > 0) return ncclSuccess;
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  return flush_group();
}

ncclResult_t ncclAllReduce(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t datatype, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t stream) {
  return enqueue(Pending{comm, kAllReduce, sendbuff, recvbuff, count, datatype, op, stream});
}
ncclResult_t ncclReduceScatter(const void* sendbuff, void* recvbuff, size_t recvcount, ncclDataType_t datatype,
                               ncclRedOp_t op, ncclComm_t comm, cudaStream_t stream) {
  return enqueue(Pending{comm, kReduceScatter, sendbuff, recvbuff, recvcount, datatype, op, stream});
}
ncclResult_t ncclAllGather(const void* sendbuff, void* recvbuff, size_t sendcount, ncclDataType_t datatype, ncclComm_t comm,
                           cudaStream_t stream) {
  return enqueue(Pending{comm, kAllGather, sendbuff, recvbuff, sendcount, datatype, -1, stream});
}
ncclResult_t ncclAlltoAll(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t datatype, ncclComm_t comm,
                          cudaStream_t stream) {
  return enqueue(Pending{comm, kAllToAll, sendbuff, recvbuff, count, datatype, -1, stream});
}
ncclResult_t ncclAllToAll(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t datatype, ncclComm_t comm,
                          cudaStream_t stream) {
  return ncclAlltoAll(sendbuff, recvbuff, count, datatype, comm, stream);
}

ncclResult_t gc3RegisterIR(ncclComm_t comm, const char* path_or_json, int instances, int* ir_id) {
  if (!comm || !path_or_json) return set_error(ncclInvalidArgument, "null argument");
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  std::string text;
  if (!read_ir_text(path_or_json, text)) return set_error(ncclSystemError, "io: cannot open IR file %s", path_or_json);
  auto ir = std::make_unique<RankIR>();
  size_t first = text.find_first_not_of(" \t\r\n");
  if (first != std::string::npos && text[first] == '<') {  // MSCCL algorithm file (msccl_xml.hpp)
    std::string e;
    if (!parse_msccl_xml(text, ir->prog, e)) return set_error(ncclInvalidArgument, "%s", e.c_str());
  } else {
    SchemaError se;
    if (!parse_program(text, ir->prog, se)) return set_error(ncclInvalidArgument, "%s", se.what().c_str());
  }
  if (instances > 1) {
    if (!uniform_counts(ir->prog))
      return set_error(ncclInvalidUsage, "instances=%d: the runtime rewrite needs ops of one count (SURVEY.md Finding 5)", instances);
    ir->prog = replicate_instances(ir->prog, instances);
  }
  return register_program(comm, std::move(ir), ir_id);
}


ncclResult_t gc3SetProtocolOverride(ncclComm_t comm, int ir_id, int proto) {
  if (!comm || ir_id < 0 || ir_id >= static_cast<int>(comm->irs.size()) || proto < -1 || proto > 2)
    return set_error(ncclInvalidArgument, "bad protocol override");
  comm->irs[ir_id]->proto_override = proto;
  comm->irs[ir_id]->predicted.clear();
  return ncclSuccess;
}

ncclResult_t gc3SetConfig(ncclComm_t comm, const char* key, int64_t value) {
  if (!comm || !key) return ncclInvalidArgument;
  const std::string k = key;
  Config& c = comm->cfg;
  if (k == "slots") c.slots = static_cast<int>(value);
  else if (k == "slot_bytes") c.slot_bytes = value;
  else if (k == "max_lanes") c.max_lanes = static_cast<int>(value);
  else if (k == "lanes") c.lanes = static_cast<int>(value);
  else if (k == "tile_bytes") c.tile_bytes = value;
  else if (k == "timeout_ms") c.timeout_ms = value;
  else if (k == "trace") c.trace = static_cast<int>(value);
  else if (k == "direct") c.direct = static_cast<int>(value);
  else if (k == "source") c.source = static_cast<int>(value);
  else if (k == "unit_warps") c.unit_warps = static_cast<int>(value);
  else if (k == "group") c.group = static_cast<int>(value);
  else if (k == "tma") c.tma = static_cast<int>(value);
  else if (k == "balance") c.balance = static_cast<int>(value);
  else if (k == "mult_cap") c.mult_cap = static_cast<int>(value);
  else if (k == "taper") c.taper = static_cast<int>(value);
  else if (k == "l2hint") c.l2hint = static_cast<int>(value);
  else if (k == "wq") c.wq = static_cast<int>(value);
  else if (k == "tma_min") c.tma_min = value;
  else if (k == "ll_max_bytes") c.ll_max_bytes = value;
  else if (k == "ll128_max_bytes") c.ll128_max_bytes = value;
  else if (k == "ll_wide_tbs") c.ll_wide_tbs = static_cast<int>(value);
  else if (k == "ll_narrow_max_bytes") c.ll_narrow_max_bytes = value;
  else if (k == "builtin") c.builtin = static_cast<int>(value);
  else if (k == "clip") c.clip = static_cast<int>(value);
  else if (k == "gen") c.gen = static_cast<int>(value);
  else if (k == "gen_small") c.gen_small = value;
  else if (k == "gen_large") c.gen_large = value;
  else if (k == "gen_ll128") c.gen_ll128 = value;
  else if (k == "smem_kb") c.smem_kb = value;
  else if (k == "select") c.select = static_cast<int>(value);
  else if (k == "stage_kb") c.stage_kb = value;
  else if (k == "wq_items") c.wq_items = static_cast<int>(value);
  else if (k == "wq_lag") c.wq_lag = static_cast<int>(value);
  else if (k == "discard") c.discard = static_cast<int>(value);
  else if (k == "df") c.df = static_cast<int>(value);
  else if (k == "remote") c.remote = static_cast<int>(value);
  else if (k == "df_policy") c.df_policy = static_cast<int>(value);
  else if (k == "df_window") c.df_window = static_cast<int>(value);
  else if (k == "df_big_bytes") c.df_big_bytes = value;
  else if (k == "df_big_tile") c.df_big_tile = value;
  else if (k == "tma_remote") c.tma_remote = static_cast<int>(value);
  else if (k == "force_sys") c.force_sys = static_cast<int>(value);
  else if (k == "df_items") c.df_items = static_cast<int>(value);
  else if (k == "df_max_tile") c.df_max_tile = value;
  else if (k == "df_min_tile") c.df_min_tile = value;
  else if (k == "df_waves") c.df_waves = static_cast<int>(value);
  else if (k == "df_wave_min_tile") c.df_wave_min_tile = value;
  else if (k == "df_wave_max_lanes") c.df_wave_max_lanes = static_cast<int>(value);
  else return set_error(ncclInvalidArgument, "unknown config key %s", key);
  return ncclSuccess;
}

ncclResult_t gc3GetTrace(ncclComm_t comm, uint64_t* out, size_t max_words, int* grid, int* ops_per_block, int* lanes) {
  if (!comm || !grid || !ops_per_block || !lanes) return ncclInvalidArgument;
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  auto it = comm->clique->devs.find(comm->device);
  if (it == comm->clique->devs.end() || !it->second.d_trace) return set_error(ncclInvalidUsage, "no traced launch on this device");
  DeviceState& ds = it->second;
  *grid = ds.trace_grid;
  *ops_per_block = ds.trace_ops;
  *lanes = ds.trace_lanes;
  const size_t words = static_cast<size_t>(ds.trace_grid) * ds.trace_ops * 4;
  if (out) {
    DeviceGuard g(comm->device);
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpy(out, ds.d_trace, std::min(words, max_words) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  }
  return ncclSuccess;
}

ncclResult_t gc3QueryPlan(ncclComm_t comm, int collective, size_t count, ncclDataType_t datatype, gc3PlanInfo* info) {
  if (!comm || !info || collective < 0 || collective > 3) return ncclInvalidArgument;
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  std::memset(info, 0, sizeof(*info));
  info->ir_id = select_ir(comm, collective, count, datatype);
  if (info->ir_id < 0) return ncclSuccess;
  DeviceState* ds = nullptr;
  NCCL_TRY(device_state(comm->clique, comm->device, ds));
  int ntbs = 0, nlocal = 0;
  const RankIR& ir = *comm->irs[info->ir_id];
  for (int r = 0; r < comm->nranks; ++r)
    if (comm->clique->local[r] && comm->clique->local[r]->device == comm->device) {
      for (int m : ir.mult[r]) ntbs += m;
      ++nlocal;
    }
  CallPlan cp;
  {  // the device plan decides the execution mode: build it now when every rank lives in this process
     // and has registered the IR (never blocks on other processes)
    bool ready = true;
    for (int r = 0; r < comm->nranks; ++r) {
      Comm* lc = comm->clique->local[r];
      ready = ready && lc && lc->irs.size() > static_cast<size_t>(info->ir_id);
    }
    if (ready) NCCL_TRY(build_plan(comm->clique, *ds, info->ir_id));
  }
  const bool built = ds->plans.size() > static_cast<size_t>(info->ir_id) && ds->plans[info->ir_id].built;
  NCCL_TRY(plan_call(comm, *ds, info->ir_id, collective, count, datatype, collective == kAllReduce || collective == kReduceScatter ? 0 : -1,
                     built ? ds->plans[info->ir_id].weight : ntbs, built && ds->plans[info->ir_id].sys_scope, cp));
  info->protocol = cp.proto;
  info->mode = cp.df ? 2 : cp.wq ? 1 : 0;
  info->mail_messages = cp.df ? ds->plans[info->ir_id].df_mail_msgs : 0;
  info->remote_messages = built ? ds->plans[info->ir_id].remote_msgs : 0;
  info->sys_scope = built && ds->plans[info->ir_id].sys_scope ? 1 : 0;
  info->tma_stages = cp.tma_stages;
  info->lanes = cp.lanes;
  info->unit_warps = cp.unit_warps;
  info->group = cp.group;
  info->grid = cp.grid;
  info->local_ranks = nlocal;
  info->slots = ir.slots;
  info->chunk_elems = cp.chunk_elems * cp.kesize / static_cast<int64_t>(dtype_size(datatype));
  info->tile_elems = cp.tile_elems * cp.kesize / static_cast<int64_t>(dtype_size(datatype));
  info->ntiles = cp.ntiles;
  info->slot_bytes = ir.slot_bytes;
  const int64_t chunk_bytes = cp.chunk_elems * cp.kesize;
  int64_t wire = 0, hbm = 0;
  for (int r = 0; r < comm->nranks; ++r) {
    int64_t s, rv, h;
    traffic(ir.prog, r, chunk_bytes, s, rv, h);
    wire = std::max({wire, s, rv});
    if (comm->clique->local[r] && comm->clique->local[r]->device == comm->device) hbm += h;
  }
  info->wire_bytes = wire;
  info->hbm_bytes = hbm;
  std::snprintf(info->name, sizeof(info->name), "%s", ir.prog.name.c_str());
  return ncclSuccess;
}

// ------------------------------------------------------------------------------- IR library
struct gc3Ir {
  Program p;
};

static char* dup_cstr(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

ncclResult_t gc3IrParse(const char* text, gc3Ir_t* ir, char** err) {
  if (!text || !ir) return ncclInvalidArgument;
  auto h = std::make_unique<gc3Ir>();
  SchemaError se;
  if (!parse_program(text, h->p, se)) {
    if (err) *err = dup_cstr(se.path + "\t" + se.message);
    *ir = nullptr;
    return ncclInvalidArgument;
  }
  if (err) *err = nullptr;
  *ir = h.release();
  return ncclSuccess;
}

ncclResult_t gc3IrParseXml(const char* text, int fold_nops, gc3Ir_t* ir, char** err) {
  if (!text || !ir) return ncclInvalidArgument;
  auto h = std::make_unique<gc3Ir>();
  std::string e;
  if (!parse_msccl_xml(text, h->p, e, fold_nops != 0)) {
    if (err) *err = dup_cstr(e);
    *ir = nullptr;
    return ncclInvalidArgument;
  }
  if (err) *err = nullptr;
  *ir = h.release();
  return ncclSuccess;
}
ncclResult_t gc3IrToXml(gc3Ir_t ir, char** text) {
  if (!ir || !text) return ncclInvalidArgument;
  *text = dup_cstr(to_msccl_xml(ir->p));
  return ncclSuccess;
}
ncclResult_t gc3IrSerialize(gc3Ir_t ir, char** text) {
  if (!ir || !text) return ncclInvalidArgument;
  *text = dup_cstr(serialize(ir->p));
  return ncclSuccess;
}

ncclResult_t gc3IrValidate(gc3Ir_t ir, int nodes, int gpus_per_node, int max_threadblocks, int max_channels, char** issues) {
  if (!ir || !issues) return ncclInvalidArgument;
  Topology t;
  t.nodes = nodes;
  t.gpus_per_node = gpus_per_node;
  if (max_threadblocks > 0) t.max_threadblocks = max_threadblocks;
  if (max_channels > 0) t.max_channels = max_channels;
  std::string s;
  for (const auto& i : validate(ir->p, t)) s += i + "\n";
  *issues = dup_cstr(s);
  return ncclSuccess;
}

ncclResult_t gc3IrCheckSlots(gc3Ir_t ir, int slots, char** violations) {
  if (!ir || !violations) return ncclInvalidArgument;
  std::string s;
  for (const auto& v : check_slots(ir->p, slots)) s += v.what + "\n";
  *violations = dup_cstr(s);
  return ncclSuccess;
}

ncclResult_t gc3IrReplicate(gc3Ir_t ir, int instances, gc3Ir_t* out) {
  if (!ir || !out || instances < 1) return ncclInvalidArgument;
  if (instances > 1 && !uniform_counts(ir->p)) return ncclInvalidUsage;
  auto h = std::make_unique<gc3Ir>();
  h->p = replicate_instances(ir->p, instances);
  *out = h.release();
  return ncclSuccess;
}

ncclResult_t gc3IrArenaLayout(gc3Ir_t ir, int rank, int lanes, int slots, int64_t slot_unit, char** json) {
  if (!ir || !json || rank < 0 || rank >= ir->p.ranks() || lanes < 1 || slots < 1 || slot_unit < 1) return ncclInvalidArgument;
  const ArenaLayout a = make_layout(ir->p, rank, lanes, slots, slot_unit, {});
  std::ostringstream os;
  os << "{\"n_in\": " << a.n_in << ", \"n_out\": " << a.n_out << ", \"bytes\": " << a.bytes << ", \"off_head\": " << a.off_head
     << ", \"off_tail\": " << a.off_tail << ", \"off_mine_in\": " << a.off_mine_in << ", \"off_mine_out\": " << a.off_mine_out
     << ", \"fifo_off\": [";
  for (size_t i = 0; i < a.fifo_off[0].size(); ++i) os << (i ? ", " : "") << a.fifo_off[0][i];
  os << "], \"slot_stride\": [";
  for (size_t i = 0; i < a.slot_stride[0].size(); ++i) os << (i ? ", " : "") << a.slot_stride[0][i];
  static const char* pn[] = {"simple", "ll", "ll128"};
  for (int pr = 1; pr < kNumProtos; ++pr) {
    os << "], \"fifo_off_" << pn[pr] << "\": [";
    for (size_t i = 0; i < a.fifo_off[pr].size(); ++i) os << (i ? ", " : "") << a.fifo_off[pr][i];
    os << "], \"slot_stride_" << pn[pr] << "\": [";
    for (size_t i = 0; i < a.slot_stride[pr].size(); ++i) os << (i ? ", " : "") << a.slot_stride[pr][i];
  }
  os << "]}";
  *json = dup_cstr(os.str());
  return ncclSuccess;
}

ncclResult_t gc3IrDirectMessages(gc3Ir_t ir, char** json) {
  if (!ir || !json) return ncclInvalidArgument;
  const auto f = direct_messages(ir->p, true, nullptr);
  std::ostringstream os;
  os << "[";
  for (size_t r = 0; r < f.size(); ++r) {
    os << (r ? ", " : "") << "[";
    for (size_t t = 0; t < f[r].size(); ++t) {
      os << (t ? ", " : "") << "[";
      for (size_t s = 0; s < f[r][t].size(); ++s) os << (s ? ", " : "") << static_cast<int>(f[r][t][s]);
      os << "]";
    }
    os << "]";
  }
  os << "]";
  *json = dup_cstr(os.str());
  return ncclSuccess;
}

ncclResult_t gc3IrOrderCheck(gc3Ir_t ir, int64_t tiles, int group, int slots, int* deadlock_free) {
  if (!ir || !deadlock_free || tiles < 0 || group < 1 || slots < 1) return ncclInvalidArgument;
  *deadlock_free = order_is_deadlock_free(ir->p, {}, tiles, 1, {}, group, slots) ? 1 : 0;
  return ncclSuccess;
}

ncclResult_t gc3BootstrapExchange(const ncclUniqueId* id, int rank, int nranks, const void* payload, size_t bytes, void* out,
                                  int timeout_ms) {
  if (!id || rank < 0 || rank >= nranks || (bytes && (!payload || !out))) return ncclInvalidArgument;
  if (std::memcmp(id->internal, "GC3", 4) != 0) return set_error(ncclInvalidArgument, "unique id not created by ncclGetUniqueId");
  const std::string dir = shm_dir(uid_key(*id));
  const std::string mine(static_cast<const char*>(payload), bytes);
  if (!post_record(dir, "x.rank" + std::to_string(rank), mine)) return set_error(ncclSystemError, "cannot post bootstrap record");
  for (int r = 0; r < nranks; ++r) {
    std::string rec;
    if (!read_record(dir, "x.rank" + std::to_string(r), rec, timeout_ms))
      return set_error(ncclSystemError, "timed out waiting for rank %d's bootstrap record", r);
    if (rec.size() != bytes) return set_error(ncclInvalidUsage, "rank %d posted %zu bytes, expected %zu", r, rec.size(), bytes);
    std::memcpy(static_cast<char*>(out) + static_cast<size_t>(r) * bytes, rec.data(), bytes);
  }
  return ncclSuccess;
}

ncclResult_t gc3IrSourceReads(gc3Ir_t ir, int* complete, char** json) {
  if (!ir || !json || !complete) return ncclInvalidArgument;
  bool c = false;
  const auto f = source_reads(ir->p, c);
  *complete = c ? 1 : 0;
  std::string o = "[";
  for (size_t r = 0; r < f.size(); ++r) {
    o += r ? ",[" : "[";
    for (size_t t = 0; t < f[r].size(); ++t) {
      o += t ? ",[" : "[";
      for (size_t k = 0; k < f[r][t].size(); ++k) o += (k ? "," : "") + std::to_string(f[r][t][k]);
      o += "]";
    }
    o += "]";
  }
  *json = dup_cstr(o + "]");
  return ncclSuccess;
}
ncclResult_t gc3IrResultWrites(gc3Ir_t ir, int* complete, char** json) {
  if (!ir || !json || !complete) return ncclInvalidArgument;
  bool c = false;
  const auto f = result_writes(ir->p, c);
  *complete = c ? 1 : 0;
  std::string o = "[";
  for (size_t r = 0; r < f.size(); ++r) {
    o += r ? ",[" : "[";
    for (size_t t = 0; t < f[r].size(); ++t) {
      o += t ? ",[" : "[";
      for (size_t k = 0; k < f[r][t].size(); ++k) o += (k ? "," : "") + std::to_string(f[r][t][k]);
      o += "]";
    }
    o += "]";
  }
  *json = dup_cstr(o + "]");
  return ncclSuccess;
}
ncclResult_t gc3IrLaneMultipliers(gc3Ir_t ir, char** json) {
  if (!ir || !json) return ncclInvalidArgument;
  const auto m = lane_multipliers(ir->p, 1, 4, transport_mask(3));
  std::string o = "[";
  for (size_t r = 0; r < m.size(); ++r) {
    o += r ? ",[" : "[";
    for (size_t t = 0; t < m[r].size(); ++t) o += (t ? "," : "") + std::to_string(m[r][t]);
    o += "]";
  }
  *json = dup_cstr(o + "]");
  return ncclSuccess;
}
ncclResult_t gc3IrPredict(gc3Ir_t ir, int64_t chunk_bytes, int protocol, int lanes, double* us) {
  if (!ir || !us || chunk_bytes < 0) return ncclInvalidArgument;
  TimedModel m;  // calibration overrides (GC3_MODEL_ALPHA / _BETA / _BW, per protocol)
  const int pr = protocol == 1 ? 1 : 0;
  if (const char* v = std::getenv(pr ? "GC3_MODEL_ALPHA_LL" : "GC3_MODEL_ALPHA")) m.alpha_us[pr] = std::atof(v);
  if (const char* v = std::getenv(pr ? "GC3_MODEL_BETA_LL" : "GC3_MODEL_BETA")) m.beta_unit_gbs[pr] = std::atof(v);
  if (const char* v = std::getenv(pr ? "GC3_MODEL_BW_LL" : "GC3_MODEL_BW")) m.bw_gbs[pr] = std::atof(v);
  *us = predict_us(ir->p, chunk_bytes, protocol, lanes, m);
  return ncclSuccess;
}
ncclResult_t gc3IrBuiltin(const char* collective, int nranks, gc3Ir_t* ir) {
  if (!collective || !ir) return ncclInvalidArgument;
  auto h = std::make_unique<gc3Ir>();
  if (!builtin_program(collective, nranks, h->p)) return ncclInvalidArgument;
  *ir = h.release();
  return ncclSuccess;
}
ncclResult_t gc3SimDefaults(gc3SimConfig* cfg) {
  if (!cfg) return ncclInvalidArgument;
  std::memset(cfg, 0, sizeof(*cfg));
  const SimParams d;
  cfg->gpus_per_node = d.gpus_per_node;
  for (int k = 0; k < 3; ++k) {
    cfg->alpha_us[k] = d.alpha_us[k];
    cfg->gbps[k] = d.gbps[k];
  }
  cfg->gamma_gbps = d.gamma_gbps;
  cfg->copy_gbps = d.copy_gbps;
  cfg->chunk_bytes = d.chunk_bytes;
  cfg->launch_us = d.launch_us;
  cfg->msg_read_passes = d.msg_read_passes;
  return ncclSuccess;
}
static SimParams sim_params(const gc3SimConfig* cfg) {
  SimParams sp;
  if (cfg->nranks_gpu > 0 && cfg->rank_gpu) sp.rank_gpu.assign(cfg->rank_gpu, cfg->rank_gpu + cfg->nranks_gpu);
  sp.gpus_per_node = cfg->gpus_per_node > 0 ? cfg->gpus_per_node : 8;
  for (int k = 0; k < 3; ++k) {
    sp.alpha_us[k] = cfg->alpha_us[k];
    sp.gbps[k] = cfg->gbps[k];
  }
  sp.gamma_gbps = cfg->gamma_gbps;
  sp.copy_gbps = cfg->copy_gbps;
  sp.proto = cfg->protocol;
  if (cfg->slots > 0)
    for (int& s : sp.slots) s = cfg->slots;
  sp.chunk_bytes = cfg->chunk_bytes;
  sp.tile_bytes = cfg->tile_bytes;
  sp.launch_us = cfg->launch_us;
  sp.hbm_gbps = cfg->hbm_gbps;
  sp.lanes = std::max(1, cfg->lanes);
  sp.group = std::max(1, cfg->group);
  sp.op_us = cfg->op_us;
  sp.msg_read_passes = cfg->msg_read_passes;
  sp.workers = cfg->workers;
  return sp;
}
ncclResult_t gc3IrSimulate(gc3Ir_t ir, const gc3SimConfig* cfg, gc3SimReport* report) {
  if (!ir || !cfg || !report) return ncclInvalidArgument;
  if (cfg->gamma_gbps <= 0 || cfg->copy_gbps <= 0 || cfg->chunk_bytes < 0) return ncclInvalidArgument;
  const SimReport r = simulate(ir->p, sim_params(cfg));
  std::memset(report, 0, sizeof(*report));
  report->completed = r.completed ? 1 : 0;
  report->makespan_us = r.makespan_us;
  for (int k = 0; k < 3; ++k) report->util[k] = r.util[k];
  report->messages = r.messages;
  report->tiles = r.tiles;
  std::snprintf(report->deadlock, sizeof(report->deadlock), "%s", r.deadlock.c_str());
  return ncclSuccess;
}
ncclResult_t gc3IrSweep(gc3Ir_t ir, const gc3SimConfig* cfg, const int64_t* sizes, int nsizes, int64_t tile_bytes, char** csv) {
  if (!ir || !cfg || !csv || nsizes < 0 || (nsizes > 0 && !sizes)) return ncclInvalidArgument;
  if (cfg->gamma_gbps <= 0 || cfg->copy_gbps <= 0) return ncclInvalidArgument;
  const std::string s = sweep_csv(ir->p, sim_params(cfg), std::vector<int64_t>(sizes, sizes + nsizes), tile_bytes);
  *csv = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(*csv, s.c_str(), s.size() + 1);
  return ncclSuccess;
}
ncclResult_t gc3IrGenerate(const char* algo, const char* collective, int nranks, int channels, int instances, gc3Ir_t* ir) {
  if (!algo || !collective || !ir) return ncclInvalidArgument;
  auto h = std::make_unique<gc3Ir>();
  if (!generate_program(algo, collective, nranks, channels, instances, h->p)) return ncclInvalidArgument;
  *ir = h.release();
  return ncclSuccess;
}
ncclResult_t gc3IrBuiltinSized(const char* collective, int nranks, uint64_t bytes, gc3Ir_t* ir) {
  if (!collective || !ir) return ncclInvalidArgument;
  auto h = std::make_unique<gc3Ir>();
  if (!builtin_for(config_from_env(), collective, nranks, bytes, h->p)) return ncclInvalidArgument;
  *ir = h.release();
  return ncclSuccess;
}
ncclResult_t gc3IrFree(gc3Ir_t ir) {
  delete ir;
  return ncclSuccess;
}

void gc3Free(void* p) { std::free(p); }

}  // extern "C"
