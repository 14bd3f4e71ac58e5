// Timed simulator: see timed.hpp.
#include "timed.hpp"

#include <algorithm>
#include <cmath>
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
  int64_t pos = 0;    // (tile, step) positions completed, tile-major
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

enum Phase { kLocal, kAlpha, kXfer };

struct Running {
  int tb;
  Phase phase;
  double end_us;     // kLocal / kAlpha: phase end
  double remaining;  // kXfer: bytes left
  double bytes;      // message bytes
  int link;
};

}  // namespace

SimReport simulate(const Program& p, const SimParams& sp) {
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
  auto conn_of = [&](int src, int dst, int ch) {
    const auto key = std::make_tuple(src, dst, ch);
    auto f = conn_id.find(key);
    if (f != conn_id.end()) return f->second;
    SimConn c;
    c.link = link_of(src, dst);
    conns.push_back(c);
    return conn_id[key] = static_cast<int>(conns.size()) - 1;
  };
  for (int r = 0; r < R; ++r)
    for (const ThreadBlock& tb : p.gpus[r].tbs) {
      SimTb s;
      s.rank = r;
      s.tb = &tb;
      if (tb.send_peer >= 0 && tb.send_peer < R) s.conn_out = conn_of(r, tb.send_peer, tb.channel);
      if (tb.recv_peer >= 0 && tb.recv_peer < R) s.conn_in = conn_of(tb.recv_peer, r, tb.channel);
      s.total = ntiles * static_cast<int64_t>(tb.ops.size());
      first[r].push_back(static_cast<int>(tbs.size()));
      tbs.push_back(s);
    }
  auto tb_by_id = [&](int r, int id) {
    const auto& v = p.gpus[r].tbs;
    for (size_t t = 0; t < v.size(); ++t)
      if (v[t].id == id) return first[r][t];
    return -1;
  };
  const int slots = std::max(1, sp.slots[pr]);
  std::vector<Running> run;
  double now = 0.0;
  auto ready = [&](const SimTb& s) {
    const int nops = static_cast<int>(s.tb->ops.size());
    const int64_t i = s.pos / nops;
    const Op& op = s.tb->ops[s.pos % nops];
    for (const Dep& d : op.deps) {
      const int dt = tb_by_id(s.rank, d.tb);
      if (dt < 0) continue;
      const int64_t dn = static_cast<int64_t>(tbs[dt].tb->ops.size());
      if (tbs[dt].pos < i * dn + d.step + 1) return false;
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
    const int64_t i = s.pos / nops;
    const Op& op = s.tb->ops[s.pos % nops];
    const double bytes = tile_len(i);
    if (op_receives(op.op) && s.conn_in >= 0) conns[s.conn_in].received++;
    if (op_sends(op.op) && s.conn_out >= 0) conns[s.conn_out].sent++;
    s.running = true;
    Running x{ti, kLocal, now + local_us(op, bytes), 0.0, bytes * op.count, -1};
    if (op_sends(op.op) && s.conn_out >= 0) x.link = conns[s.conn_out].link;
    run.push_back(x);
  };
  auto finish = [&](int ti) {
    SimTb& s = tbs[ti];
    const int nops = static_cast<int>(s.tb->ops.size());
    const Op& op = s.tb->ops[s.pos % nops];
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
          const int nops = static_cast<int>(s.tb->ops.size());
          os << " r" << s.rank << ".tb" << s.tb->id << "@t" << s.pos / nops << ".s" << s.pos % nops;
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
          if (x.phase == kLocal && x.link >= 0) {
            x.phase = kAlpha;
            x.end_us = now + links[x.link].alpha_us;
          } else if (x.phase == kAlpha || x.link < 0) {
            if (x.link >= 0 && x.bytes > 0) {
              x.phase = kXfer;
              x.remaining = x.bytes;
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
    for (const Running& x : run) {
      if (x.phase != kXfer) dt = std::min(dt, x.end_us - now);
      else dt = std::min(dt, x.remaining / (links[x.link].gbps * 1e3 / static_cast<double>(links[x.link].flows.size())));
    }
    if (!(dt < kInf)) dt = 0.0;
    dt = std::max(dt, 0.0);
    for (SimLink& l : links)
      if (!l.flows.empty()) l.busy_us += dt;
    for (Running& x : run)
      if (x.phase == kXfer) x.remaining -= dt * links[x.link].gbps * 1e3 / static_cast<double>(links[x.link].flows.size());
    now += dt;
    for (size_t k = 0; k < run.size(); ++k) {
      Running& x = run[k];
      if (x.phase == kXfer && x.remaining <= 1e-9 * std::max(1.0, x.bytes)) {
        auto& f = links[x.link].flows;
        f.erase(std::find(f.begin(), f.end(), x.tb));
        finish(x.tb);
        run.erase(run.begin() + static_cast<long>(k));
        --k;
      }
    }
  }
  rep.completed = true;
  rep.makespan_us = now + (ntiles > 0 ? sp.launch_us : 0.0);
  int used[3] = {0, 0, 0};
  for (const SimLink& l : links) {
    if (l.busy_us <= 0.0) continue;
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
