// Timed simulator: see timed.hpp.
#include "timed.hpp"

#include <algorithm>
#include <cmath>
#include <deque>
#include <cstdio>
#include <limits>
#include <map>
#include <sstream>
#include <tuple>

namespace gc3 {

namespace {

struct SimTb {
  int rank = 0;
  const ThreadBlock* tb = nullptr;
  int conn_in = -1, conn_out = -1;
  int lane = 0;
  int64_t pos = 0;    // (tile of the lane, step) positions completed, tile-major
  int64_t total = 0;  // tiles x ops
  bool running = false;
};

struct SimConn {
  int link = -1;
  int64_t sent = 0;       // sends started (slots taken)
  int64_t delivered = 0;  // transfers finished
  int64_t received = 0;   // receives started
  int64_t consumed = 0;   // receives finished (slots freed)
};

struct SimLink {
  int cls = 0;
  double gbps = 1.0;
  double alpha_us = 0.0;
  std::vector<int> flows;  // running tb indices in the transfer phase
  double busy_us = 0.0;
};

enum Phase { kLocal, kLocalFlow, kAlpha, kXfer };

struct Running {
  int tb;
  Phase phase;
  double end_us;     // kLocal / kAlpha: phase end
  double remaining;  // kLocalFlow / kXfer: bytes left on resource `res`
  double bytes;      // message bytes
  int link;          // transfer resource (-1: the op sends nothing)
  int res;           // resource of the current flow
  double local;      // local bytes (device-memory resource on)
  int hbm;           // device-memory resource of the op's GPU (-1: off)
  bool local_done;   // the local flow (device-memory mode) has run
};

int local_passes(Opcode o) {
  switch (o) {
    case Opcode::send: case Opcode::recv: case Opcode::rcs: case Opcode::rrs: return 1;
    case Opcode::copy: case Opcode::rrc: case Opcode::rrcs: return 2;
    case Opcode::reduce: return 3;
    default: return 0;
  }
}

}  // namespace

// Dataflow execution (SimParams::workers > 0): the runtime's dataflow executor. Every (op, tile) is a
// task, ready once all of the op's predecessors (previous op of its thread block, declared deps, the
// sender of its message) have finished that tile; `workers` units take ready tasks in order (roots
// tile-major). A task costs op_us, then its local bytes on its GPU's device-memory resource
// (processor sharing), then alpha if it sends.
static SimReport simulate_dataflow(const Program& p, const SimParams& sp) {
  SimReport rep;
  const int R = p.ranks();
  const int pr = std::max(0, std::min(2, sp.proto));
  const int64_t chunk = std::max<int64_t>(sp.chunk_bytes, 0);
  const int64_t tile = (sp.tile_bytes <= 0 || sp.tile_bytes > chunk) ? chunk : sp.tile_bytes;
  const int64_t ntiles = chunk == 0 ? 0 : (chunk + tile - 1) / tile;
  rep.tiles = ntiles;
  std::vector<int> gpu(R);
  for (int r = 0; r < R; ++r) gpu[r] = sp.rank_gpu.empty() ? r : sp.rank_gpu[static_cast<size_t>(r) % sp.rank_gpu.size()];
  struct Node {
    int rank;
    const Op* op;
    bool sends;
  };
  std::vector<Node> nodes;
  std::vector<std::vector<int>> first(R);
  for (int r = 0; r < R; ++r)
    for (const ThreadBlock& tb : p.gpus[r].tbs) {
      first[r].push_back(static_cast<int>(nodes.size()));
      for (const Op& op : tb.ops) nodes.push_back({r, &op, op_sends(op.op) && tb.send_peer >= 0});
    }
  const int N = static_cast<int>(nodes.size());
  std::vector<std::vector<int>> succ(N);
  std::vector<int> indeg(N, 0);
  auto edge = [&](int u, int v) {
    succ[u].push_back(v);
    indeg[v]++;
  };
  std::map<std::tuple<int, int, int>, std::pair<std::vector<int>, std::vector<int>>> conns;
  for (int r = 0; r < R; ++r)
    for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) {
      const ThreadBlock& tb = p.gpus[r].tbs[t];
      for (size_t s = 0; s < tb.ops.size(); ++s) {
        const int v = first[r][t] + static_cast<int>(s);
        if (s > 0) edge(v - 1, v);
        for (const Dep& d : tb.ops[s].deps)
          for (size_t t2 = 0; t2 < p.gpus[r].tbs.size(); ++t2)
            if (p.gpus[r].tbs[t2].id == d.tb && d.step < static_cast<int>(p.gpus[r].tbs[t2].ops.size()))
              edge(first[r][t2] + d.step, v);
        if (op_sends(tb.ops[s].op) && tb.send_peer >= 0) conns[{r, tb.send_peer, tb.channel}].first.push_back(v);
        if (op_receives(tb.ops[s].op) && tb.recv_peer >= 0) conns[{tb.recv_peer, r, tb.channel}].second.push_back(v);
      }
    }
  for (auto& [k, c] : conns) {
    for (size_t i = 0; i < std::min(c.first.size(), c.second.size()); ++i) edge(c.first[i], c.second[i]);
    for (size_t i = c.first.size(); i < c.second.size(); ++i) indeg[c.second[i]]++;  // never delivered
  }
  // message link class of every sending node (its thread block's send peer)
  std::vector<int> link_class(N, 0), peer(N, -1);
  for (int r = 0; r < R; ++r)
    for (size_t t = 0; t < p.gpus[r].tbs.size(); ++t) {
      const ThreadBlock& tb = p.gpus[r].tbs[t];
      for (size_t s = 0; s < tb.ops.size(); ++s) {
        const int v = first[r][t] + static_cast<int>(s);
        if (!nodes[v].sends) continue;
        const int g = gpu[r], h = gpu[tb.send_peer];
        const int gpn = std::max(1, sp.gpus_per_node);
        link_class[v] = g == h ? 0 : (g / gpn == h / gpn ? 1 : 2);
        peer[v] = h;
      }
    }
  // processor-shared resources: the device memory of a GPU (local bytes; device-memory mode, else the
  // local copy rate) and the ordered GPU pairs (message bytes; same-GPU messages in device-memory mode
  // pay only alpha, their bytes are the receiver's local pass)
  std::map<std::pair<int, int>, int> res_id;
  std::vector<double> rate, busy;
  std::vector<int> res_class;
  std::vector<std::vector<int>> flows;
  auto resource = [&](int kind, int key, double gbps, int cls) {
    auto f = res_id.find({kind, key});
    if (f != res_id.end()) return f->second;
    flows.emplace_back();
    rate.push_back(gbps * 1e3);  // bytes per us
    busy.push_back(0.0);
    res_class.push_back(cls);
    return res_id[{kind, key}] = static_cast<int>(flows.size()) - 1;
  };
  struct Task {
    int64_t id;
    int phase;  // 0 fixed cost, 1 local flow, 2 alpha, 3 message transfer
    double end, remaining;
    int res;
  };
  std::vector<int64_t> left(static_cast<size_t>(N) * ntiles);
  for (int64_t t = 0; t < ntiles; ++t)
    for (int v = 0; v < N; ++v) left[static_cast<size_t>(t) * N + v] = indeg[v];
  std::deque<int64_t> ready;
  for (int64_t t = 0; t < ntiles; ++t)
    for (int v = 0; v < N; ++v)
      if (indeg[v] == 0) ready.push_back(t * N + v);
  std::vector<Task> run;
  const int W = std::max(1, sp.workers);
  double now = 0.0;
  int64_t done = 0;
  const int64_t total = static_cast<int64_t>(N) * ntiles;
  auto tile_of = [&](int64_t id) {
    const int64_t t = id / N;
    return static_cast<double>(std::min(tile, chunk - t * tile)) * nodes[id % N].op->count;
  };
  auto local_bytes = [&](int64_t id) {
    const Opcode o = nodes[id % N].op->op;
    const int passes = local_passes(o) + ((o == Opcode::rrc || o == Opcode::rrcs || o == Opcode::rrs) ? sp.msg_read_passes : 0);
    if (sp.hbm_gbps > 0) return tile_of(id) * passes;
    return o == Opcode::copy || op_reduces(o) ? tile_of(id) : 0.0;  // SPEC: b / copy rate, b / gamma
  };
  auto local_res = [&](int64_t id) {
    const int g = gpu[nodes[id % N].rank];
    if (sp.hbm_gbps > 0) return resource(0, g, sp.hbm_gbps, 0);
    return op_reduces(nodes[id % N].op->op) ? resource(2, g, sp.gamma_gbps, 0) : resource(3, g, sp.copy_gbps, 0);
  };
  auto alpha_of = [&](int64_t id) {
    const int v = static_cast<int>(id % N);
    return nodes[v].sends ? sp.alpha_us[link_class[v]] * sp.alpha_mult[pr] : 0.0;
  };
  auto xfer_res = [&](int64_t id) {
    const int v = static_cast<int>(id % N);
    if (!nodes[v].sends || (link_class[v] == 0 && sp.hbm_gbps > 0)) return -1;
    const int c = link_class[v];
    return resource(1, gpu[nodes[v].rank] * 65536 + peer[v], sp.gbps[c] / sp.beta_mult[pr], c);
  };
  // advance a task whose current phase ended at `now`; returns true when the task is finished
  auto next_phase = [&](Task& x) {
    for (;;) {
      if (x.phase == 0) {
        x.phase = 1;
        x.remaining = local_bytes(x.id);
        if (x.remaining > 0) {
          x.res = local_res(x.id);
          return false;
        }
      } else if (x.phase == 1) {
        x.phase = 2;
        x.end = now + alpha_of(x.id);
        if (x.end > now) return false;
      } else if (x.phase == 2) {
        x.phase = 3;
        x.res = xfer_res(x.id);
        x.remaining = x.res >= 0 ? tile_of(x.id) : 0.0;
        if (x.remaining > 0) return false;
      } else {
        return true;
      }
    }
  };
  const double kInf = std::numeric_limits<double>::infinity();
  while (done < total) {
    while (static_cast<int>(run.size()) < W && !ready.empty()) {
      const int64_t id = ready.front();
      ready.pop_front();
      run.push_back({id, 0, now + sp.op_us, 0.0, -1});
    }
    if (run.empty()) {
      rep.deadlock = "deadlock: tasks wait for predecessors or messages that never complete";
      rep.makespan_us = now;
      return rep;
    }
    // phase ends at `now`, then completions
    bool finished = false;
    for (size_t k = 0; k < run.size();) {
      Task& x = run[k];
      const bool ended = (x.phase == 0 || x.phase == 2) ? x.end <= now : x.remaining <= 1e-9 * std::max(1.0, tile_of(x.id));
      if (ended && next_phase(x)) {
        const int64_t id = x.id;
        const int64_t t = id / N;
        for (int v2 : succ[id % N])
          if (--left[static_cast<size_t>(t) * N + v2] == 0) ready.push_back(t * N + v2);
        if (nodes[id % N].sends) rep.messages++;
        ++done;
        run.erase(run.begin() + static_cast<long>(k));
        finished = true;
      } else {
        ++k;
      }
    }
    if (finished) continue;
    for (auto& f : flows) f.clear();
    for (size_t k = 0; k < run.size(); ++k)
      if (run[k].phase == 1 || run[k].phase == 3) flows[run[k].res].push_back(static_cast<int>(k));
    double dt = kInf;
    for (const Task& x : run) {
      if (x.phase == 1 || x.phase == 3) dt = std::min(dt, x.remaining / (rate[x.res] / static_cast<double>(flows[x.res].size())));
      else dt = std::min(dt, x.end - now);
    }
    if (!(dt < kInf)) dt = 0.0;
    dt = std::max(dt, 0.0);
    for (size_t r2 = 0; r2 < flows.size(); ++r2)
      if (!flows[r2].empty()) busy[r2] += dt;
    for (Task& x : run)
      if (x.phase == 1 || x.phase == 3) x.remaining -= dt * rate[x.res] / static_cast<double>(flows[x.res].size());
    now += dt;
  }
  rep.completed = true;
  rep.makespan_us = now + (ntiles > 0 ? sp.launch_us : 0.0);
  // utilisation: mean busy fraction per link class of the ordered pairs used (device memory: class 0)
  double sum[3] = {0, 0, 0};
  int cnt[3] = {0, 0, 0};
  for (size_t r2 = 0; r2 < rate.size(); ++r2)
    if (busy[r2] > 0) {
      sum[res_class[r2]] += now > 0 ? busy[r2] / now : 0.0;
      cnt[res_class[r2]]++;
    }
  for (int c = 0; c < 3; ++c) rep.util[c] = cnt[c] ? sum[c] / cnt[c] : 0.0;
  return rep;
}

SimReport simulate(const Program& p, const SimParams& sp) {
  if (sp.workers > 0) return simulate_dataflow(p, sp);
  SimReport rep;
  const int R = p.ranks();
  const int pr = std::max(0, std::min(2, sp.proto));
  std::vector<int> gpu(R);
  for (int r = 0; r < R; ++r) gpu[r] = sp.rank_gpu.empty() ? r : sp.rank_gpu[static_cast<size_t>(r) % sp.rank_gpu.size()];
  const int64_t chunk = std::max<int64_t>(sp.chunk_bytes, 0);
  const int64_t tile = (sp.tile_bytes <= 0 || sp.tile_bytes > chunk) ? chunk : sp.tile_bytes;
  const int64_t ntiles = chunk == 0 ? 0 : (chunk + tile - 1) / tile;
  rep.tiles = ntiles;
  auto tile_len = [&](int64_t i) { return static_cast<double>(std::min(tile, chunk - i * tile)); };
  // thread blocks, connections, links
  std::vector<SimTb> tbs;
  std::vector<std::vector<int>> first(R);  // (rank, tb index) -> sim tb
  std::map<std::tuple<int, int, int>, int> conn_id;
  std::vector<SimConn> conns;
  std::map<std::pair<int, int>, int> link_id;
  std::vector<SimLink> links;
  auto link_of = [&](int src, int dst) {
    const auto key = std::make_pair(gpu[src], gpu[dst]);
    auto f = link_id.find(key);
    if (f != link_id.end()) return f->second;
    SimLink l;
    const int gpn = std::max(1, sp.gpus_per_node);
    l.cls = gpu[src] == gpu[dst] ? 0 : (gpu[src] / gpn == gpu[dst] / gpn ? 1 : 2);
    l.gbps = std::max(1e-9, sp.gbps[l.cls] / sp.beta_mult[pr]);
    l.alpha_us = sp.alpha_us[l.cls] * sp.alpha_mult[pr];
    links.push_back(l);
    return link_id[key] = static_cast<int>(links.size()) - 1;
  };
  std::map<int, int> hbm_id;  // GPU -> device-memory resource
  auto hbm_of = [&](int g) {
    if (sp.hbm_gbps <= 0) return -1;
    auto f = hbm_id.find(g);
    if (f != hbm_id.end()) return f->second;
    SimLink l;
    l.cls = 3;
    l.gbps = sp.hbm_gbps;
    l.alpha_us = sp.alpha_us[0] * sp.alpha_mult[pr];  // same-GPU messages routed here keep their alpha
    links.push_back(l);
    return hbm_id[g] = static_cast<int>(links.size()) - 1;
  };
  auto conn_of = [&](int src, int dst, int ch) {
    const auto key = std::make_tuple(src, dst, ch);
    auto f = conn_id.find(key);
    if (f != conn_id.end()) return f->second;
    SimConn c;
    c.link = link_of(src, dst);
    conns.push_back(c);
    return conn_id[key] = static_cast<int>(conns.size()) - 1;
  };
  const int L = std::max(1, sp.lanes);
  for (int r = 0; r < R; ++r)
    for (const ThreadBlock& tb : p.gpus[r].tbs) {
      first[r].push_back(static_cast<int>(tbs.size()));
      for (int l = 0; l < L; ++l) {  // sim tb index = first + lane
        SimTb s;
        s.rank = r;
        s.tb = &tb;
        s.lane = l;
        if (tb.send_peer >= 0 && tb.send_peer < R) s.conn_out = conn_of(r, tb.send_peer, tb.channel * L + l);
        if (tb.recv_peer >= 0 && tb.recv_peer < R) s.conn_in = conn_of(tb.recv_peer, r, tb.channel * L + l);
        const int64_t lane_tiles = ntiles > l ? (ntiles - 1 - l) / L + 1 : 0;
        s.total = lane_tiles * static_cast<int64_t>(tb.ops.size());
        tbs.push_back(s);
      }
    }
  auto tb_by_id = [&](int r, int id) {
    const auto& v = p.gpus[r].tbs;
    for (size_t t = 0; t < v.size(); ++t)
      if (v[t].id == id) return first[r][t];
    return -1;
  };
  // a lane's order: groups of G tiles, op-major inside a group (G = 1: the paper's tile-major loop)
  const int64_t G = std::max<int64_t>(1, sp.group);
  auto lane_tiles = [&](const SimTb& s) { return s.total / static_cast<int64_t>(std::max<size_t>(1, s.tb->ops.size())); };
  auto decode = [&](const SimTb& s, int64_t pos, int64_t& lt, int& step) {  // pos -> (tile of the lane, step)
    const int64_t nops = static_cast<int64_t>(s.tb->ops.size());
    const int64_t g0 = pos / (G * nops) * G;
    const int64_t gs = std::min<int64_t>(G, lane_tiles(s) - g0);
    const int64_t in = pos - g0 * nops;
    step = static_cast<int>(in / gs);
    lt = g0 + in % gs;
  };
  auto encode = [&](const SimTb& s, int64_t lt, int step) {  // (tile of the lane, step) -> pos
    const int64_t nops = static_cast<int64_t>(s.tb->ops.size());
    const int64_t g0 = lt / G * G;
    const int64_t gs = std::min<int64_t>(G, lane_tiles(s) - g0);
    return g0 * nops + step * gs + (lt - g0);
  };
  const int slots = std::max(1, sp.slots[pr]);
  std::vector<Running> run;
  double now = 0.0;
  auto ready = [&](const SimTb& s) {
    const int nops = static_cast<int>(s.tb->ops.size());
    int64_t i;
    int step;
    decode(s, s.pos, i, step);
    (void)nops;
    const Op& op = s.tb->ops[step];
    for (const Dep& d : op.deps) {
      const int dt0 = tb_by_id(s.rank, d.tb);
      if (dt0 < 0) continue;
      const int dt = dt0 + s.lane;
      const int64_t dn = static_cast<int64_t>(tbs[dt].tb->ops.size());
      (void)dn;
      if (tbs[dt].pos < encode(tbs[dt], i, d.step) + 1) return false;
    }
    if (op_receives(op.op) && s.conn_in >= 0 && conns[s.conn_in].delivered <= conns[s.conn_in].received) return false;
    if (op_sends(op.op) && s.conn_out >= 0 && conns[s.conn_out].sent - conns[s.conn_out].consumed >= slots) return false;
    return true;
  };
  auto local_us = [&](const Op& op, double bytes) {
    const double b = bytes * op.count;
    switch (op.op) {
      case Opcode::copy: return b / (sp.copy_gbps * 1e3);
      case Opcode::reduce: case Opcode::rrc: case Opcode::rrcs: case Opcode::rrs: return b / (sp.gamma_gbps * 1e3);
      default: return 0.0;
    }
  };
  auto start = [&](int ti) {
    SimTb& s = tbs[ti];
    const int nops = static_cast<int>(s.tb->ops.size());
    int64_t lt;
    int step;
    decode(s, s.pos, lt, step);
    (void)nops;
    const int64_t i = s.lane + lt * L;  // the tile
    const Op& op = s.tb->ops[step];
    const double bytes = tile_len(i);
    if (op_receives(op.op) && s.conn_in >= 0) conns[s.conn_in].received++;
    if (op_sends(op.op) && s.conn_out >= 0) conns[s.conn_out].sent++;
    s.running = true;
    const int hbm = hbm_of(gpu[s.rank]);
    const int passes = local_passes(op.op) + ((op.op == Opcode::rrc || op.op == Opcode::rrcs || op.op == Opcode::rrs) ? sp.msg_read_passes : 0);
    Running x{ti, kLocal, hbm >= 0 ? now + sp.op_us : now + local_us(op, bytes), 0.0, bytes * op.count, -1, -1,
              bytes * op.count * passes, hbm, hbm < 0};
    if (op_sends(op.op) && s.conn_out >= 0) {
      x.link = conns[s.conn_out].link;
      if (hbm >= 0 && links[x.link].cls == 0) {  // same GPU: the message's bytes are the ops' local passes
        x.link = hbm;                            // (direct writes, pulled reads); it pays its alpha
        x.bytes = 0;
      }
    }
    if (hbm >= 0 && x.local <= 0) x.local_done = true;
    run.push_back(x);
  };
  auto finish = [&](int ti) {
    SimTb& s = tbs[ti];
    int64_t lt;
    int step;
    decode(s, s.pos, lt, step);
    const Op& op = s.tb->ops[step];
    if (op_receives(op.op) && s.conn_in >= 0) conns[s.conn_in].consumed++;
    if (op_sends(op.op) && s.conn_out >= 0) {
      conns[s.conn_out].delivered++;
      rep.messages++;
    }
    s.pos++;
    s.running = false;
  };
  const double kInf = std::numeric_limits<double>::infinity();
  for (;;) {
    bool all_done = true;
    for (size_t ti = 0; ti < tbs.size(); ++ti) {
      SimTb& s = tbs[ti];
      if (s.pos >= s.total) continue;
      all_done = false;
      if (!s.running && ready(s)) start(static_cast<int>(ti));
    }
    if (all_done) break;
    if (run.empty()) {
      std::ostringstream os;
      for (const SimTb& s : tbs)
        if (s.pos < s.total) {
          int64_t lt;
          int step;
          decode(s, s.pos, lt, step);
          os << " r" << s.rank << ".tb" << s.tb->id << "@t" << s.lane + lt * L << ".s" << step;
        }
      rep.deadlock = "deadlock: blocked" + os.str();
      rep.makespan_us = now;
      return rep;
    }
    // zero-length phases advance immediately; an op finishing now may enable others now
    bool moved = true, finished_now = false;
    while (moved) {
      moved = false;
      for (size_t k = 0; k < run.size(); ++k) {
        Running& x = run[k];
        if ((x.phase == kLocal || x.phase == kAlpha) && x.end_us <= now) {
          if (x.phase == kLocal && !x.local_done) {  // fixed per-op cost done: the local bytes flow
            x.phase = kLocalFlow;
            x.remaining = x.local;
            x.res = x.hbm;
            links[x.hbm].flows.push_back(x.tb);
          } else if (x.phase == kLocal && x.link >= 0) {
            x.phase = kAlpha;
            x.end_us = now + links[x.link].alpha_us;
          } else if (x.phase == kAlpha || x.link < 0) {
            if (x.link >= 0 && x.bytes > 0) {
              x.phase = kXfer;
              x.remaining = x.bytes;
              x.res = x.link;
              links[x.link].flows.push_back(x.tb);
            } else {
              finish(x.tb);
              run.erase(run.begin() + static_cast<long>(k));
              --k;
              finished_now = true;
            }
          }
          moved = true;
        }
      }
    }
    if (finished_now || run.empty()) continue;
    // next event: a phase end or a transfer completion (processor sharing on each ordered pair)
    double dt = kInf;
    auto rate = [&](int res) { return links[res].gbps * 1e3 / static_cast<double>(links[res].flows.size()); };
    for (const Running& x : run) {
      if (x.phase == kLocal || x.phase == kAlpha) dt = std::min(dt, x.end_us - now);
      else dt = std::min(dt, x.remaining / rate(x.res));
    }
    if (!(dt < kInf)) dt = 0.0;
    dt = std::max(dt, 0.0);
    for (SimLink& l : links)
      if (!l.flows.empty()) l.busy_us += dt;
    for (Running& x : run)
      if (x.phase == kXfer || x.phase == kLocalFlow) x.remaining -= dt * rate(x.res);
    now += dt;
    for (size_t k = 0; k < run.size(); ++k) {
      Running& x = run[k];
      const bool flow = x.phase == kXfer || x.phase == kLocalFlow;
      if (!flow || x.remaining > 1e-9 * std::max(1.0, x.phase == kXfer ? x.bytes : x.local)) continue;
      auto& f = links[x.res].flows;
      f.erase(std::find(f.begin(), f.end(), x.tb));
      if (x.phase == kLocalFlow) {  // local work done: the message (if any) follows
        x.phase = kLocal;
        x.end_us = now;
        x.local_done = true;
        continue;
      }
      finish(x.tb);
      run.erase(run.begin() + static_cast<long>(k));
      --k;
    }
  }
  rep.completed = true;
  rep.makespan_us = now + (ntiles > 0 ? sp.launch_us : 0.0);
  int used[3] = {0, 0, 0};
  for (const SimLink& l : links) {
    if (l.busy_us <= 0.0 || l.cls > 2) continue;
    used[l.cls]++;
    rep.util[l.cls] += now > 0 ? l.busy_us / now : 0.0;
  }
  for (int c = 0; c < 3; ++c)
    if (used[c]) rep.util[c] /= used[c];
  return rep;
}

std::string sweep_csv(const Program& p, const SimParams& sp, const std::vector<int64_t>& sizes, int64_t tile_bytes) {
  std::ostringstream os;
  os << "size_bytes,makespan_us,util_intra,util_inter\n";
  const int nin = std::max(1, p.nchunks[0]);
  for (int64_t size : sizes) {
    SimParams q = sp;
    q.chunk_bytes = size / nin;
    q.tile_bytes = tile_bytes;
    const SimReport r = simulate(p, q);
    char line[160];
    const double intra = (r.util[0] > 0 && r.util[1] > 0) ? 0.5 * (r.util[0] + r.util[1]) : std::max(r.util[0], r.util[1]);
    if (r.completed) std::snprintf(line, sizeof(line), "%lld,%.4f,%.4f,%.4f\n", static_cast<long long>(size), r.makespan_us, intra, r.util[2]);
    else std::snprintf(line, sizeof(line), "%lld,deadlock,,\n", static_cast<long long>(size));
    os << line;
  }
  return os.str();
}

}  // namespace gc3
