// GC3-IR host library (see ir.hpp for the reference interfaces each function replaces).
#include "ir.hpp"

#include <algorithm>
#include <deque>
#include <map>
#include <set>
#include <tuple>

#include "json.hpp"

namespace gc3 {

const char* opcode_name(Opcode op) {
  static const char* names[] = {"send", "recv", "copy", "reduce", "rrc", "rcs", "rrcs", "rrs", "nop"};
  const int i = static_cast<int>(op);
  return i >= 0 && i < 9 ? names[i] : "?";
}
const char* buf_name(Buf b) {
  static const char* names[] = {"input", "output", "scratch"};
  const int i = static_cast<int>(b);
  return i >= 0 && i < 3 ? names[i] : "?";
}
const char* proto_name(Proto p) {
  static const char* names[] = {"simple", "ll", "ll128"};
  const int i = static_cast<int>(p);
  return i >= 0 && i < 3 ? names[i] : "?";
}

bool known_collective(const std::string& name) {
  for (const char* k : {"allreduce", "allgather", "reducescatter", "alltoall", "alltonext", "custom"})
    if (name == k) return true;
  return false;
}

const ThreadBlock* Program::find_tb(int rank, int id) const {
  if (rank < 0 || rank >= ranks()) return nullptr;
  for (const auto& tb : gpus[rank].tbs)
    if (tb.id == id) return &tb;
  return nullptr;
}

// ---------------------------------------------------------------------------------------------
// Loader. Error paths/messages follow the reference deserializer (ir.hpp:188-310) and
// require_keys (core.hpp:478-491): missing keys are reported in schema order before unknown keys,
// unknown keys in sorted order.

namespace {

struct Fail {
  SchemaError e;
};

[[noreturn]] void fail(const std::string& path, const std::string& msg) { throw Fail{SchemaError{path, msg}}; }

std::string join(const std::string& path, const std::string& key) { return path.empty() ? key : path + "." + key; }

void need_keys(const json::Value& v, const std::string& path, std::initializer_list<const char*> keys) {
  if (!v.is_object()) fail(path, "expected an object");
  for (const char* k : keys)
    if (!v.contains(k)) fail(join(path, k), "missing required key");
  for (const auto& kv : v.o) {
    bool known = false;
    for (const char* k : keys) known = known || kv.first == k;
    if (!known) fail(join(path, kv.first), "unknown key");
  }
}

int get_int(const json::Value& v, const std::string& path) {
  if (!v.is_int()) fail(path, "expected an integer");
  return static_cast<int>(v.as_i64());
}

uint64_t get_u64(const json::Value& v, const std::string& path) {
  if (!v.is_int()) fail(path, "expected an integer");
  if (!v.is_unsigned() && v.as_i64() < 0) fail(path, "expected a non-negative integer");
  return v.as_u64();
}

bool get_bool(const json::Value& v, const std::string& path) {
  if (!v.is_bool()) fail(path, "expected a boolean");
  return v.b;
}

const std::string& get_str(const json::Value& v, const std::string& path) {
  if (!v.is_string()) fail(path, "expected a string");
  return v.s;
}

Buf get_buf(const json::Value& v, const std::string& path) {
  const auto& s = get_str(v, path);
  if (s == "input") return Buf::input;
  if (s == "output") return Buf::output;
  if (s == "scratch") return Buf::scratch;
  fail(path, "expected one of \"input\", \"output\", \"scratch\"");
}

bool opcode_from(const std::string& s, Opcode& out) {
  for (int i = 0; i < 9; ++i)
    if (s == opcode_name(static_cast<Opcode>(i))) {
      out = static_cast<Opcode>(i);
      return true;
    }
  return false;
}

const json::Value& array_at(const json::Value& parent, const char* key, const std::string& path) {
  const auto& v = parent.at(key);
  if (!v.is_array()) fail(path, "expected an array");
  return v;
}

void load(const json::Value& root, Program& p) {
  need_keys(root, "", {"name", "collective", "protocol", "inplace", "nchunks", "size_range", "gpus"});
  p.name = get_str(root.at("name"), "name");
  p.collective = get_str(root.at("collective"), "collective");
  if (!known_collective(p.collective)) fail("collective", "unknown collective \"" + p.collective + "\"");
  const auto& proto = get_str(root.at("protocol"), "protocol");
  if (proto == "simple") p.proto = Proto::simple;
  else if (proto == "ll") p.proto = Proto::ll;
  else if (proto == "ll128") p.proto = Proto::ll128;
  else fail("protocol", "expected one of \"simple\", \"ll\", \"ll128\"");
  p.inplace = get_bool(root.at("inplace"), "inplace");

  const auto& nc = root.at("nchunks");
  need_keys(nc, "nchunks", {"input", "output", "scratch"});
  p.nchunks[0] = get_int(nc.at("input"), "nchunks.input");
  p.nchunks[1] = get_int(nc.at("output"), "nchunks.output");
  p.nchunks[2] = get_int(nc.at("scratch"), "nchunks.scratch");

  const auto& sr = root.at("size_range");
  need_keys(sr, "size_range", {"min_bytes", "max_bytes"});
  p.min_bytes = get_u64(sr.at("min_bytes"), "size_range.min_bytes");
  p.max_bytes = get_u64(sr.at("max_bytes"), "size_range.max_bytes");

  const auto& gpus = array_at(root, "gpus", "gpus");
  p.gpus.resize(gpus.a.size());
  for (size_t g = 0; g < gpus.a.size(); ++g) {
    const std::string gp = "gpus[" + std::to_string(g) + "]";
    const auto& jg = gpus.a[g];
    need_keys(jg, gp, {"rank", "threadblocks"});
    Gpu& gpu = p.gpus[g];
    gpu.rank = get_int(jg.at("rank"), gp + ".rank");
    const auto& tbs = array_at(jg, "threadblocks", gp + ".threadblocks");
    gpu.tbs.resize(tbs.a.size());
    for (size_t t = 0; t < tbs.a.size(); ++t) {
      const std::string tp = gp + ".threadblocks[" + std::to_string(t) + "]";
      const auto& jt = tbs.a[t];
      need_keys(jt, tp, {"id", "send_peer", "recv_peer", "channel", "ops"});
      ThreadBlock& tb = gpu.tbs[t];
      tb.id = get_int(jt.at("id"), tp + ".id");
      tb.send_peer = get_int(jt.at("send_peer"), tp + ".send_peer");
      tb.recv_peer = get_int(jt.at("recv_peer"), tp + ".recv_peer");
      tb.channel = get_int(jt.at("channel"), tp + ".channel");
      const auto& ops = array_at(jt, "ops", tp + ".ops");
      tb.ops.resize(ops.a.size());
      for (size_t o = 0; o < ops.a.size(); ++o) {
        const std::string op_path = tp + ".ops[" + std::to_string(o) + "]";
        const auto& jo = ops.a[o];
        need_keys(jo, op_path, {"step", "opcode", "src_buf", "src_off", "dst_buf", "dst_off", "count", "deps", "has_dep"});
        Op& op = tb.ops[o];
        op.step = get_int(jo.at("step"), op_path + ".step");
        if (!opcode_from(get_str(jo.at("opcode"), op_path + ".opcode"), op.op)) fail(op_path + ".opcode", "unknown opcode");
        op.src_buf = get_buf(jo.at("src_buf"), op_path + ".src_buf");
        op.src_off = get_int(jo.at("src_off"), op_path + ".src_off");
        op.dst_buf = get_buf(jo.at("dst_buf"), op_path + ".dst_buf");
        op.dst_off = get_int(jo.at("dst_off"), op_path + ".dst_off");
        op.count = get_int(jo.at("count"), op_path + ".count");
        const auto& deps = array_at(jo, "deps", op_path + ".deps");
        op.deps.resize(deps.a.size());
        for (size_t d = 0; d < deps.a.size(); ++d) {
          const std::string dp = op_path + ".deps[" + std::to_string(d) + "]";
          need_keys(deps.a[d], dp, {"tb", "step"});
          op.deps[d].tb = get_int(deps.a[d].at("tb"), dp + ".tb");
          op.deps[d].step = get_int(deps.a[d].at("step"), dp + ".step");
        }
        op.has_dep = get_bool(jo.at("has_dep"), op_path + ".has_dep");
      }
    }
  }
}

json::Value jint(int64_t x) {
  json::Value v;
  if (x < 0) {
    v.kind = json::Kind::integer;
    v.i = x;
  } else {
    v.kind = json::Kind::unsigned_integer;
    v.u = static_cast<uint64_t>(x);
  }
  return v;
}
json::Value jstr(const std::string& s) {
  json::Value v;
  v.kind = json::Kind::string;
  v.s = s;
  return v;
}
json::Value jbool(bool b) {
  json::Value v;
  v.kind = json::Kind::boolean;
  v.b = b;
  return v;
}

}  // namespace

bool parse_program(const std::string& text, Program& out, SchemaError& err) {
  json::Value root;
  std::string perr;
  out = Program();
  if (!json::parse(text, root, perr)) {
    err = SchemaError{"", "invalid JSON: " + perr};
    return false;
  }
  try {
    load(root, out);
  } catch (const Fail& f) {
    err = f.e;
    return false;
  }
  return true;
}

std::string serialize(const Program& p) {
  json::Value root;
  root.kind = json::Kind::object;
  root.o["name"] = jstr(p.name);
  root.o["collective"] = jstr(p.collective);
  root.o["protocol"] = jstr(proto_name(p.proto));
  root.o["inplace"] = jbool(p.inplace);
  json::Value nc;
  nc.kind = json::Kind::object;
  nc.o["input"] = jint(p.nchunks[0]);
  nc.o["output"] = jint(p.nchunks[1]);
  nc.o["scratch"] = jint(p.nchunks[2]);
  root.o["nchunks"] = nc;
  json::Value sr;
  sr.kind = json::Kind::object;
  sr.o["min_bytes"].kind = json::Kind::unsigned_integer;
  sr.o["min_bytes"].u = p.min_bytes;
  sr.o["max_bytes"].kind = json::Kind::unsigned_integer;
  sr.o["max_bytes"].u = p.max_bytes;
  root.o["size_range"] = sr;
  json::Value gpus;
  gpus.kind = json::Kind::array;
  for (const auto& g : p.gpus) {
    json::Value jg;
    jg.kind = json::Kind::object;
    jg.o["rank"] = jint(g.rank);
    json::Value tbs;
    tbs.kind = json::Kind::array;
    for (const auto& tb : g.tbs) {
      json::Value jt;
      jt.kind = json::Kind::object;
      jt.o["id"] = jint(tb.id);
      jt.o["send_peer"] = jint(tb.send_peer);
      jt.o["recv_peer"] = jint(tb.recv_peer);
      jt.o["channel"] = jint(tb.channel);
      json::Value ops;
      ops.kind = json::Kind::array;
      for (const auto& op : tb.ops) {
        json::Value jo;
        jo.kind = json::Kind::object;
        jo.o["step"] = jint(op.step);
        jo.o["opcode"] = jstr(opcode_name(op.op));
        jo.o["src_buf"] = jstr(buf_name(op.src_buf));
        jo.o["src_off"] = jint(op.src_off);
        jo.o["dst_buf"] = jstr(buf_name(op.dst_buf));
        jo.o["dst_off"] = jint(op.dst_off);
        jo.o["count"] = jint(op.count);
        json::Value deps;
        deps.kind = json::Kind::array;
        for (const auto& d : op.deps) {
          json::Value jd;
          jd.kind = json::Kind::object;
          jd.o["tb"] = jint(d.tb);
          jd.o["step"] = jint(d.step);
          deps.a.push_back(jd);
        }
        jo.o["deps"] = deps;
        jo.o["has_dep"] = jbool(op.has_dep);
        ops.a.push_back(std::move(jo));
      }
      jt.o["ops"] = std::move(ops);
      tbs.a.push_back(std::move(jt));
    }
    jg.o["threadblocks"] = std::move(tbs);
    gpus.a.push_back(std::move(jg));
  }
  root.o["gpus"] = std::move(gpus);
  return json::dump(root, 2) + "\n";
}

// ---------------------------------------------------------------------------------------------
// Structural validation: the checks and messages of the reference validate() (ir.hpp:341-439),
// reported in the same order so the issue lists compare equal.

std::vector<std::string> validate(const Program& p, const Topology& topo) {
  std::vector<std::string> out;
  auto S = [](long long x) { return std::to_string(x); };
  const int R = p.ranks();
  if (R != topo.ranks()) out.push_back("program has " + S(R) + " gpus but topology has " + S(topo.ranks()));
  if (p.inplace && p.nchunks[0] != p.nchunks[1]) out.push_back("in-place program must have matching input/output chunk counts");
  if (p.nchunks[0] < 0 || p.nchunks[1] < 0 || p.nchunks[2] < 0) out.push_back("negative chunk count");

  for (int r = 0; r < R; ++r) {
    const Gpu& g = p.gpus[r];
    if (g.rank != r) out.push_back("gpus[" + S(r) + "] has rank " + S(g.rank) + ", expected " + S(r));
    if (static_cast<int>(g.tbs.size()) > topo.max_threadblocks)
      out.push_back("gpu " + S(r) + " uses " + S(g.tbs.size()) + " thread blocks, budget is " + S(topo.max_threadblocks));
    std::set<int> ids;
    std::set<std::pair<int, int>> senders, receivers;
    for (const auto& tb : g.tbs) {
      const std::string where = "gpu " + S(r) + " tb " + S(tb.id);
      if (!ids.insert(tb.id).second) out.push_back(where + ": duplicate thread block id");
      if (tb.channel < 0 || tb.channel >= topo.max_channels) out.push_back(where + ": channel " + S(tb.channel) + " out of budget");
      for (int peer : {tb.send_peer, tb.recv_peer})
        if (peer < -1 || peer >= R || peer == r) out.push_back(where + ": invalid peer " + S(peer));
      if (tb.send_peer >= 0 && !senders.emplace(tb.send_peer, tb.channel).second)
        out.push_back(where + ": a second thread block sends to peer " + S(tb.send_peer) + " on channel " + S(tb.channel));
      if (tb.recv_peer >= 0 && !receivers.emplace(tb.recv_peer, tb.channel).second)
        out.push_back(where + ": a second thread block receives from peer " + S(tb.recv_peer) + " on channel " + S(tb.channel));
      for (size_t s = 0; s < tb.ops.size(); ++s) {
        const Op& op = tb.ops[s];
        const std::string at = where + " step " + S(s);
        if (op.step != static_cast<int>(s)) out.push_back(at + ": step field is " + S(op.step));
        if (op.count < 1) out.push_back(at + ": count must be >= 1");
        if (op_sends(op.op) && tb.send_peer < 0) out.push_back(at + ": " + opcode_name(op.op) + " in a thread block without a send peer");
        if (op_receives(op.op) && tb.recv_peer < 0) out.push_back(at + ": " + opcode_name(op.op) + " in a thread block without a receive peer");
        const long long src_end = static_cast<long long>(op.src_off) + op.count;
        const long long dst_end = static_cast<long long>(op.dst_off) + op.count;
        if (op.src_off < 0 || src_end > p.nchunks[static_cast<int>(op.src_buf)])
          out.push_back(at + ": src span exceeds " + buf_name(op.src_buf) + " extent");
        if (op.dst_off < 0 || dst_end > p.nchunks[static_cast<int>(op.dst_buf)])
          out.push_back(at + ": dst span exceeds " + buf_name(op.dst_buf) + " extent");
        std::set<int> dep_tbs;
        for (const auto& d : op.deps) {
          if (!dep_tbs.insert(d.tb).second) out.push_back(at + ": duplicate dependency on tb " + S(d.tb));
          if (d.tb == tb.id) out.push_back(at + ": dependency on own thread block");
          const ThreadBlock* target = p.find_tb(r, d.tb);
          if (!target) out.push_back(at + ": dependency on nonexistent tb " + S(d.tb));
          else if (d.step < 0 || d.step >= static_cast<int>(target->ops.size()))
            out.push_back(at + ": dependency on nonexistent step " + S(d.step) + " of tb " + S(d.tb));
          else if (!target->ops[d.step].has_dep)
            out.push_back(at + ": dependency target tb " + S(d.tb) + " step " + S(d.step) + " lacks has_dep");
        }
      }
    }
  }
  // every sender needs exactly one receiving thread block with the same message-count sequence
  for (int r = 0; r < R; ++r) {
    for (const auto& tb : p.gpus[r].tbs) {
      if (tb.send_peer < 0 || tb.send_peer >= R) continue;
      std::vector<int> sent;
      for (const auto& op : tb.ops)
        if (op_sends(op.op)) sent.push_back(op.count);
      const ThreadBlock* rx = nullptr;
      for (const auto& other : p.gpus[tb.send_peer].tbs)
        if (other.recv_peer == r && other.channel == tb.channel) rx = &other;  // last match wins
      const std::string conn = "connection " + S(r) + "->" + S(tb.send_peer) + " ch " + S(tb.channel);
      if (!rx) {
        if (!sent.empty()) out.push_back(conn + " has no receiving thread block");
        continue;
      }
      std::vector<int> got;
      for (const auto& op : rx->ops)
        if (op_receives(op.op)) got.push_back(op.count);
      if (sent != got)
        out.push_back(conn + " is unbalanced: " + S(sent.size()) + " sends vs " + S(got.size()) + " receives (or counts differ)");
    }
  }
  return out;
}

// ---------------------------------------------------------------------------------------------
// Static slot check (scheduler.hpp:633-734): over the happens-before graph made of sequential
// execution, declared deps and the k-th send -> k-th receive matching, the k-th send on a
// connection must not precede (transitively) the receive k-s it waits for.

std::vector<SlotViolation> check_slots(const Program& p, int slots) {
  std::vector<SlotViolation> out;
  if (slots < 1) slots = 1;
  std::map<std::tuple<int, int, int>, int> unit_of;  // (gpu, tb id, step) -> unit
  struct Unit {
    int gpu, tb, step;
  };
  std::vector<Unit> units;
  for (const auto& g : p.gpus)
    for (const auto& tb : g.tbs)
      for (size_t s = 0; s < tb.ops.size(); ++s) {
        unit_of[{g.rank, tb.id, static_cast<int>(s)}] = static_cast<int>(units.size());
        units.push_back({g.rank, tb.id, static_cast<int>(s)});
      }
  const size_t n = units.size();
  std::vector<std::vector<int>> succ(n);
  struct Conn {
    std::vector<int> tx, rx;
  };
  std::map<std::tuple<int, int, int>, Conn> conns;
  for (const auto& g : p.gpus)
    for (const auto& tb : g.tbs)
      for (size_t s = 0; s < tb.ops.size(); ++s) {
        const int u = unit_of[{g.rank, tb.id, static_cast<int>(s)}];
        if (s + 1 < tb.ops.size()) succ[u].push_back(u + 1);
        for (const auto& d : tb.ops[s].deps) {
          auto it = unit_of.find({g.rank, d.tb, d.step});
          if (it != unit_of.end()) succ[it->second].push_back(u);
        }
        if (op_sends(tb.ops[s].op) && tb.send_peer >= 0) conns[{g.rank, tb.send_peer, tb.channel}].tx.push_back(u);
        if (op_receives(tb.ops[s].op) && tb.recv_peer >= 0) conns[{tb.recv_peer, g.rank, tb.channel}].rx.push_back(u);
      }
  for (auto& [key, c] : conns) {
    if (c.tx.size() != c.rx.size()) {
      out.push_back({std::get<0>(key), std::get<1>(key), std::get<2>(key), -1, -1, "unbalanced connection"});
      continue;
    }
    for (size_t k = 0; k < c.tx.size(); ++k) succ[c.tx[k]].push_back(c.rx[k]);
  }
  // reachability bitsets in reverse topological order
  const size_t words = (n + 63) / 64;
  std::vector<uint64_t> reach(n * words, 0);
  std::vector<int> indeg(n, 0), order;
  for (size_t u = 0; u < n; ++u)
    for (int v : succ[u]) ++indeg[v];
  std::deque<int> ready;
  for (size_t u = 0; u < n; ++u)
    if (!indeg[u]) ready.push_back(static_cast<int>(u));
  while (!ready.empty()) {
    const int u = ready.front();
    ready.pop_front();
    order.push_back(u);
    for (int v : succ[u])
      if (--indeg[v] == 0) ready.push_back(v);
  }
  for (auto it = order.rbegin(); it != order.rend(); ++it) {
    const int u = *it;
    uint64_t* ru = &reach[u * words];
    ru[u / 64] |= 1ull << (u % 64);
    for (int v : succ[u]) {
      const uint64_t* rv = &reach[v * words];
      for (size_t w = 0; w < words; ++w) ru[w] |= rv[w];
    }
  }
  for (const auto& [key, c] : conns) {
    if (c.tx.size() != c.rx.size()) continue;
    const auto [src, dst, ch] = key;
    for (size_t k = slots; k < c.tx.size(); ++k) {
      const int snd = c.tx[k], need = c.rx[k - slots];
      if ((reach[snd * words + need / 64] >> (need % 64)) & 1) {
        out.push_back({src, dst, ch, units[snd].tb, units[snd].step,
                       "send " + std::to_string(k) + " on connection " + std::to_string(src) + "->" + std::to_string(dst) + " ch " +
                           std::to_string(ch) + " needs slot " + std::to_string(k - slots) +
                           " freed, but that receive depends on this send"});
      }
    }
  }
  return out;
}

// ---------------------------------------------------------------------------------------------
bool uniform_counts(const Program& p) {
  int c = 0;
  for (const auto& g : p.gpus)
    for (const auto& tb : g.tbs)
      for (const auto& op : tb.ops) {
        if (op.op == Opcode::nop) continue;
        if (c && op.count != c) return false;
        c = op.count;
      }
  return true;
}

Program replicate_instances(const Program& p, int k) {
  if (k <= 1) return p;
  Program q = p;
  int nch = 1;
  for (const auto& g : p.gpus)
    for (const auto& tb : g.tbs) nch = std::max(nch, tb.channel + 1);
  for (int b = 0; b < 3; ++b) q.nchunks[b] = p.nchunks[b] * k;
  for (size_t r = 0; r < p.gpus.size(); ++r) {
    const Gpu& g = p.gpus[r];
    int ntb = 0;
    for (const auto& tb : g.tbs) ntb = std::max(ntb, tb.id + 1);
    Gpu& out = q.gpus[r];
    out.tbs.clear();
    for (int j = 0; j < k; ++j) {
      for (const auto& tb : g.tbs) {
        ThreadBlock t = tb;
        t.id = tb.id + j * ntb;
        t.channel = tb.channel + j * nch;
        for (auto& op : t.ops) {
          op.src_off = op.src_off * k + j * op.count;
          op.dst_off = op.dst_off * k + j * op.count;
          for (auto& d : op.deps) d.tb += j * ntb;
        }
        out.tbs.push_back(std::move(t));
      }
    }
  }
  return q;
}

bool builtin_program(const std::string& collective, int R, Program& out, int channels) {
  if (R < 2) return false;
  auto mod = [R](int x) { return ((x % R) + R) % R; };
  Program p;
  p.collective = collective;
  p.proto = Proto::simple;
  auto op = [](int step, Opcode o, Buf sb, int so, Buf db, int dof) {
    Op x;
    x.step = step;
    x.op = o;
    x.src_buf = sb;
    x.src_off = so;
    x.dst_buf = db;
    x.dst_off = dof;
    x.count = 1;
    return x;
  };
  for (int r = 0; r < R; ++r) {
    Gpu g;
    g.rank = r;
    if (collective == "alltoall") {  // direct: one thread block per peer, own chunk copied locally
      int id = 0;
      for (int q = 0; q < R; ++q) {
        if (q == r) continue;
        ThreadBlock tb;
        tb.id = id;
        tb.send_peer = tb.recv_peer = q;
        tb.channel = 0;
        int s = 0;
        tb.ops.push_back(op(s++, Opcode::send, Buf::input, q, Buf::output, r));
        if (id == 0) tb.ops.push_back(op(s++, Opcode::copy, Buf::input, r, Buf::output, r));
        tb.ops.push_back(op(s++, Opcode::recv, Buf::input, r, Buf::output, q));
        g.tbs.push_back(tb);
        ++id;
      }
    } else if (collective == "allreduce") {
      // ring, one thread block per channel: chunk k travels on channel k % C. Chunk k is sent raw by
      // rank k+1 and reduced along the ring (RS step s = (r - k - 1) mod R at rank r; the rank
      // before the owner forwards the sum without storing it: rrs), completed by its owner k
      // (rrcs) and forwarded around (AG step a = (r - k) mod R). A thread block runs its chunks'
      // ops in global ring-step order (RS steps 0..R-1, then AG steps R..2R-2): the order the
      // reference scheduler gives these programs.
      const int C = std::max(1, std::min(channels, R));
      for (int ch = 0; ch < C; ++ch) {
        ThreadBlock tb;
        tb.id = ch;
        tb.send_peer = mod(r + 1);
        tb.recv_peer = mod(r - 1);
        tb.channel = ch;
        std::vector<std::pair<int, Op>> steps;
        for (int k = ch; k < R; k += C) {
          const int s = mod(r - k - 1);
          const Opcode rs = s == 0 ? Opcode::send : (s == R - 2 && R >= 3) ? Opcode::rrs : Opcode::rrcs;
          steps.push_back({s, op(0, rs, Buf::input, k, Buf::input, k)});
          const int ag = mod(r - k);
          if (ag >= 1) steps.push_back({R - 1 + ag, op(0, ag == R - 1 ? Opcode::recv : Opcode::rcs, Buf::input, k, Buf::input, k)});
        }
        std::sort(steps.begin(), steps.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
        for (auto& [gs, o] : steps) {
          o.step = static_cast<int>(tb.ops.size());
          tb.ops.push_back(o);
        }
        g.tbs.push_back(tb);
      }
    } else {  // ring: send to r+1, receive from r-1
      ThreadBlock tb;
      tb.id = 0;
      tb.send_peer = mod(r + 1);
      tb.recv_peer = mod(r - 1);
      tb.channel = 0;
      int s = 0;
      auto same = [&](Opcode o, Buf b, int c) { tb.ops.push_back(op(s++, o, b, mod(c), b, mod(c))); };
      if (collective == "allgather") {
        tb.ops.push_back(op(s++, Opcode::copy, Buf::input, 0, Buf::output, r));
        same(Opcode::send, Buf::output, r);
        for (int k = 1; k <= R - 2; ++k) same(Opcode::rcs, Buf::output, r - k);
        same(Opcode::recv, Buf::output, r + 1);
      } else if (collective == "reducescatter") {
        same(Opcode::send, Buf::input, r - 1);
        for (int k = 1; k <= R - 2; ++k) same(Opcode::rrcs, Buf::input, r - 1 - k);
        same(Opcode::rrc, Buf::input, r);
      } else {
        return false;
      }
      g.tbs.push_back(tb);
    }
    p.gpus.push_back(std::move(g));
  }
  if (collective == "allreduce" || collective == "reducescatter") {
    p.inplace = true;
    p.nchunks[0] = p.nchunks[1] = R;
  } else if (collective == "allgather") {
    p.nchunks[0] = 1;
    p.nchunks[1] = R;
  } else {
    p.nchunks[0] = p.nchunks[1] = R;
  }
  p.name = "builtin_" + collective + "_" + std::to_string(R);
  out = std::move(p);
  return true;
}

// All-pairs AllReduce (two communication steps instead of Ring's 2R-2). Rank r
// owns chunk r; one thread block per peer q (send and receive peer q, channel 0) runs: send chunk q
// (r's contribution to q's chunk), rrc chunk r (q's contribution, reduced in), send chunk r (the
// final value, back to q), recv chunk q (q's final value). The reductions into chunk r are chained
// across the thread blocks with deps (one writer at a time) and every final send waits for the
// last one. Equivalent to the reference compiler's all-pairs program (same final state, race free:
// tests/test_builtin_irs.py), not its exact thread-block layout: that one fuses the last
// reduction with the first final send (rrcs) and orders blocks by its scheduler's heuristics.
static bool allpairs_allreduce(int R, Program& out) {
  if (R < 2) return false;
  Program p;
  p.collective = "allreduce";
  p.proto = Proto::simple;
  p.inplace = true;
  p.nchunks[0] = p.nchunks[1] = R;
  for (int r = 0; r < R; ++r) {
    Gpu g;
    g.rank = r;
    std::vector<int> peers;
    for (int q = 0; q < R; ++q)
      if (q != r) peers.push_back(q);
    const int last = static_cast<int>(peers.size()) - 1;
    for (int i = 0; i <= last; ++i) {
      const int q = peers[i];
      ThreadBlock tb;
      tb.id = i;
      tb.send_peer = tb.recv_peer = q;
      tb.channel = 0;
      auto mk = [&](Opcode o, int chunk) {
        Op x;
        x.step = static_cast<int>(tb.ops.size());
        x.op = o;
        x.src_buf = x.dst_buf = Buf::input;
        x.src_off = x.dst_off = chunk;
        x.count = 1;
        return x;
      };
      tb.ops.push_back(mk(Opcode::send, q));
      Op red = mk(Opcode::rrc, r);
      if (i > 0) red.deps.push_back({i - 1, 1});
      red.has_dep = true;  // the next reduction (or the final sends) wait on it
      tb.ops.push_back(red);
      Op fin = mk(Opcode::send, r);
      if (i != last) fin.deps.push_back({last, 1});
      tb.ops.push_back(fin);
      tb.ops.push_back(mk(Opcode::recv, q));
      g.tbs.push_back(tb);
    }
    p.gpus.push_back(std::move(g));
  }
  p.name = "builtin_allpairs_allreduce_" + std::to_string(R);
  out = std::move(p);
  return true;
}

// Hierarchical AllReduce over N nodes x G GPUs (rank = node * G + local index),
// R = N * G chunks per rank seen as G blocks of N chunks: (1) a ReduceScatter ring inside every
// node on channel 0 leaves local rank g owning block g reduced over its node; (2) on channel 1 a
// ring AllReduce across the N nodes among the ranks with local index g completes block g (its N
// chunks, one per node); (3) an AllGather ring inside every node on channel 2 distributes the
// blocks. Phase 2 waits for phase 1 (the owning rrc), phase 3's first send for phase 2's last op,
// both declared as deps. Our own layout of the reference's hier_ar program (same final state,
// race free: tests/test_builtin_irs.py), not its exact thread-block order.
static bool hierarchical_allreduce(int N, int G, Program& out) {
  if (N < 2 || G < 2) return false;
  const int R = N * G;
  Program p;
  p.collective = "allreduce";
  p.proto = Proto::simple;
  p.inplace = true;
  p.nchunks[0] = p.nchunks[1] = R;
  auto mk = [](Opcode o, int chunk, int count) {
    Op x;
    x.op = o;
    x.src_buf = x.dst_buf = Buf::input;
    x.src_off = x.dst_off = chunk;
    x.count = count;
    return x;
  };
  auto finish = [](ThreadBlock& tb, std::vector<std::pair<int, Op>>& steps) {
    std::stable_sort(steps.begin(), steps.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    for (auto& [k, o] : steps) {
      o.step = static_cast<int>(tb.ops.size());
      tb.ops.push_back(o);
    }
  };
  for (int r = 0; r < R; ++r) {
    const int n = r / G, l = r % G;
    Gpu g;
    g.rank = r;
    // (1) intra-node ReduceScatter of the G blocks (N chunks each): block b's chain starts at local
    // b + 1 and ends (rrc) at its owner b; RS step s = (l - b - 1) mod G
    ThreadBlock t1;
    t1.id = 0;
    t1.send_peer = n * G + (l + 1) % G;
    t1.recv_peer = n * G + (l + G - 1) % G;
    t1.channel = 0;
    std::vector<std::pair<int, Op>> s1;
    for (int b = 0; b < G; ++b) {
      const int s = ((l - b - 1) % G + G) % G;
      s1.push_back({s, mk(s == 0 ? Opcode::send : s == G - 1 ? Opcode::rrc : Opcode::rrcs, b * N, N)});
    }
    finish(t1, s1);
    t1.ops.back().has_dep = true;  // the owning rrc: phase 2 waits for it
    // (2) ring AllReduce across the nodes on block l: chunk l*N + k is owned by node k
    ThreadBlock t2;
    t2.id = 1;
    t2.send_peer = ((n + 1) % N) * G + l;
    t2.recv_peer = ((n + N - 1) % N) * G + l;
    t2.channel = 1;
    std::vector<std::pair<int, Op>> s2;
    for (int k = 0; k < N; ++k) {
      const int s = ((n - k - 1) % N + N) % N;  // RS step
      const Opcode rs = s == 0 ? Opcode::send : (s == N - 2 && N >= 3) ? Opcode::rrs : Opcode::rrcs;
      s2.push_back({s, mk(rs, l * N + k, 1)});
      const int a = ((n - k) % N + N) % N;  // AG step
      if (a >= 1) s2.push_back({N - 1 + a, mk(a == N - 1 ? Opcode::recv : Opcode::rcs, l * N + k, 1)});
    }
    finish(t2, s2);
    t2.ops.front().deps.push_back({0, static_cast<int>(t1.ops.size()) - 1});
    t2.ops.back().has_dep = true;  // phase 3's first send waits for it
    // (3) intra-node AllGather of the blocks: block b leaves its owner b; AG step a = (l - b) mod G
    ThreadBlock t3;
    t3.id = 2;
    t3.send_peer = t1.send_peer;
    t3.recv_peer = t1.recv_peer;
    t3.channel = 2;
    std::vector<std::pair<int, Op>> s3;
    for (int b = 0; b < G; ++b) {
      const int a = ((l - b) % G + G) % G;
      s3.push_back({a, mk(a == 0 ? Opcode::send : a == G - 1 ? Opcode::recv : Opcode::rcs, b * N, N)});
    }
    finish(t3, s3);
    t3.ops.front().deps.push_back({1, static_cast<int>(t2.ops.size()) - 1});
    g.tbs.push_back(t1);
    g.tbs.push_back(t2);
    g.tbs.push_back(t3);
    p.gpus.push_back(std::move(g));
  }
  p.name = "builtin_hier_allreduce_" + std::to_string(N) + "x" + std::to_string(G);
  out = std::move(p);
  return true;
}

bool generate_program(const std::string& algo, const std::string& collective, int R, int channels, int instances, Program& out) {
  if (R < 2 || channels < 1 || instances < 1 || instances > 64) return false;
  Program p;
  if (algo == "ring") {
    if (collective == "alltoall" || (channels > 1 && collective != "allreduce")) return false;
    if (!builtin_program(collective, R, p, channels)) return false;
  } else if (algo == "direct") {
    if (collective != "alltoall" || channels != 1) return false;
    if (!builtin_program(collective, R, p)) return false;
  } else if (algo == "allpairs") {
    if (collective != "allreduce" || channels != 1) return false;
    if (!allpairs_allreduce(R, p)) return false;
  } else if (algo == "hier") {  // channels = GPUs per node (R = nodes x channels)
    if (collective != "allreduce" || channels < 2 || R % channels) return false;
    if (!hierarchical_allreduce(R / channels, channels, p)) return false;
  } else {
    return false;
  }
  if (instances > 1) p = replicate_instances(p, instances);
  p.name = "builtin_" + algo + "_" + collective + "_" + std::to_string(R) + "_ch" + std::to_string(channels) + "_inst" +
           std::to_string(instances);
  out = std::move(p);
  return true;
}

}  // namespace gc3
