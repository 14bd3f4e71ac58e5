// Timed simulator of GC3-IR programs (SPEC.md:464-481 run_timed / sweep): a discrete-event
// alpha-beta model with chunk tiling. Used by the runtime to choose among candidate programs
// (config "select", comm-time generated programs) and exposed as gc3IrSimulate / gc3IrSweep.
//
//   * every IR thread block steps through its ops tile by tile (Fig. 4 tiling loop outermost,
//     PAPER.md:419), an op starting when its deps are done for that tile, its
//     incoming message has been delivered and (for a send) its connection has a free slot of the
//     `slots` FIFO slots;
//   * a message of b bytes on the ordered GPU pair (g, h) costs alpha(class) + b * beta(class),
//     concurrent messages on one ordered pair sharing its bandwidth equally (processor sharing:
//     SPEC.md:470, "DESIGN DECISIONS"); alpha is paid per message;
//   * local work: a reduction costs b / gamma, a local copy b / copy rate; fused ops pay their local
//     part, then one transfer;
//   * link classes: 0 the same GPU (loopback ranks), 1 another GPU of the node (NVLink/NVSwitch),
//     2 another node; protocols scale alpha and beta (SPEC's placeholders: Simple 1/1, LL 0.25/2,
//     LL128 0.5/1.07) and set the FIFO depth.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ir.hpp"

namespace gc3 {

struct SimParams {
  std::vector<int> rank_gpu;          // GPU of every rank (empty: rank r on GPU r)
  int gpus_per_node = 8;              // GPUs g and h share a node iff g / gpus_per_node == h / gpus_per_node
  double alpha_us[3] = {1.0, 2.0, 8.0};        // per message, per link class
  double gbps[3] = {3000.0, 770.0, 50.0};      // bandwidth of one ordered GPU pair, per link class
  double gamma_gbps = 3000.0;                  // local reduction rate
  double copy_gbps = 3000.0;                   // local copy rate
  int proto = 0;                               // 0 simple, 1 ll, 2 ll128
  double alpha_mult[3] = {1.0, 0.25, 0.5};
  double beta_mult[3] = {1.0, 2.0, 1.07};
  int slots[3] = {2, 8, 4};
  int64_t chunk_bytes = 1 << 20;
  int64_t tile_bytes = 0;                      // 0: one tile per chunk
  double launch_us = 0.0;                      // added to the makespan
  // Optional device-memory resource (0: off, SPEC semantics). On: every op's local reads and writes
  // (send 1, recv 1, copy 2, reduce 3, rrc 2, rcs 1, rrcs 2, rrs 1 passes of its bytes: the
  // runtime's algorithmic bytes) are flows on one processor-shared resource per GPU of this rate;
  // same-GPU messages then pay only their alpha -- the loopback calibration, where all ranks share
  // one GPU's HBM.
  double hbm_gbps = 0.0;
  double op_us = 0.0;          // fixed cost of every op per tile (device-memory mode): the interpreter's
                               // per-op synchronisation (barriers, release fence, flags)
  int msg_read_passes = 1;     // device-memory mode: extra passes of a reducing receive (rrc / rrcs / rrs)
                               // that reads its message from a FIFO slot or the sender's span
  // Lanes (the runtime's parallelism): every thread block runs as `lanes` independent
  // units, lane l taking tiles l, l + lanes, ...; each connection has its FIFO slots per lane.
  int lanes = 1;
  int group = 1;  // tiles per op-major group inside a lane (the runtime's tile groups; 1: tile-major)
  int workers = 0;  // > 0: dataflow execution (the runtime's dataflow executor) with this many units
};

struct SimReport {
  bool completed = false;
  std::string deadlock;       // blocked thread blocks when !completed
  double makespan_us = 0.0;
  double util[3] = {0, 0, 0};  // per link class: mean busy fraction of the ordered pairs used
  int64_t messages = 0;
  int64_t tiles = 0;
};

SimReport simulate(const Program& p, const SimParams& sp);

// One timed run per size (bytes per rank buffer, i.e. chunk_bytes = size / nchunks(input));
// CSV "size_bytes,makespan_us,util_intra,util_inter". util_intra covers
// link classes 0 and 1, util_inter class 2.
std::string sweep_csv(const Program& p, const SimParams& sp, const std::vector<int64_t>& sizes, int64_t tile_bytes);

}  // namespace gc3
