// MSCCL-XML adapter (see msccl_xml.hpp).
#include "msccl_xml.hpp"

#include <algorithm>
#include <cstdlib>
#include <map>
#include <set>
#include <sstream>
#include <utility>
#include <vector>

namespace gc3 {
namespace {

// ------------------------------------------------------------------ a small XML reader
// Elements, attributes ('..' or ".." with the five predefined entities and numeric references),
// self-closing tags, comments, processing instructions and <!DOCTYPE>. Character data between
// elements is ignored (MSCCL files carry none).
struct Elem {
  std::string tag;
  std::vector<std::pair<std::string, std::string>> attrs;
  std::vector<Elem> kids;
  int line = 0;
  const std::string* attr(const std::string& k) const {
    for (const auto& a : attrs)
      if (a.first == k) return &a.second;
    return nullptr;
  }
};

struct Reader {
  const std::string& s;
  size_t i = 0;
  int line = 1;
  std::string err;

  explicit Reader(const std::string& text) : s(text) {}
  bool eof() const { return i >= s.size(); }
  bool fail(const std::string& m) {
    if (err.empty()) err = "line " + std::to_string(line) + ": " + m;
    return false;
  }
  void adv(size_t n = 1) {
    for (size_t k = 0; k < n && i < s.size(); ++k, ++i)
      if (s[i] == '\n') ++line;
  }
  bool starts(const char* p) const { return s.compare(i, std::char_traits<char>::length(p), p) == 0; }
  void ws() {
    while (!eof() && (s[i] == ' ' || s[i] == '\t' || s[i] == '\n' || s[i] == '\r')) adv();
  }
  static bool name_char(char c) {
    return (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || (c >= '0' && c <= '9') || c == '_' || c == '-' || c == '.' ||
           c == ':';
  }
  bool name(std::string& out) {
    const size_t b = i;
    while (!eof() && name_char(s[i])) adv();
    if (i == b) return fail("expected a name");
    out = s.substr(b, i - b);
    return true;
  }
  bool skip_until(const char* end) {
    const size_t p = s.find(end, i);
    if (p == std::string::npos) return fail(std::string("unterminated construct, expected '") + end + "'");
    adv(p + std::char_traits<char>::length(end) - i);
    return true;
  }
  // comments, processing instructions, declarations and character data
  bool misc() {
    for (;;) {
      const size_t b = i;
      while (!eof() && s[i] != '<') adv();
      if (eof()) return true;
      if (starts("<!--")) {
        if (!skip_until("-->")) return false;
      } else if (starts("<?")) {
        if (!skip_until("?>")) return false;
      } else if (starts("<!")) {
        if (!skip_until(">")) return false;
      } else {
        return true;
      }
      (void)b;
    }
  }
  bool value(std::string& out) {
    if (eof() || (s[i] != '"' && s[i] != '\'')) return fail("expected a quoted attribute value");
    const char q = s[i];
    adv();
    out.clear();
    while (!eof() && s[i] != q) {
      if (s[i] == '<') return fail("'<' in attribute value");
      if (s[i] == '&') {
        const size_t semi = s.find(';', i);
        if (semi == std::string::npos || semi - i > 10) return fail("bad entity reference");
        const std::string ent = s.substr(i + 1, semi - i - 1);
        if (ent == "lt") out += '<';
        else if (ent == "gt") out += '>';
        else if (ent == "amp") out += '&';
        else if (ent == "quot") out += '"';
        else if (ent == "apos") out += '\'';
        else if (ent.size() > 1 && ent[0] == '#') {
          const long v = ent[1] == 'x' ? std::strtol(ent.c_str() + 2, nullptr, 16) : std::strtol(ent.c_str() + 1, nullptr, 10);
          if (v <= 0 || v > 127) return fail("unsupported character reference &" + ent + ";");
          out += static_cast<char>(v);
        } else {
          return fail("unknown entity &" + ent + ";");
        }
        adv(semi + 1 - i);
      } else {
        out += s[i];
        adv();
      }
    }
    if (eof()) return fail("unterminated attribute value");
    adv();
    return true;
  }
  bool element(Elem& e, int depth) {
    if (depth > 16) return fail("elements nested too deeply");
    if (eof() || s[i] != '<') return fail("expected '<'");
    e.line = line;
    adv();
    if (!name(e.tag)) return false;
    for (;;) {
      ws();
      if (eof()) return fail("unterminated tag <" + e.tag + ">");
      if (starts("/>")) {
        adv(2);
        return true;
      }
      if (s[i] == '>') {
        adv();
        break;
      }
      std::string k, v;
      if (!name(k)) return false;
      ws();
      if (eof() || s[i] != '=') return fail("expected '=' after attribute " + k);
      adv();
      ws();
      if (!value(v)) return false;
      if (e.attr(k)) return fail("duplicate attribute " + k + " on <" + e.tag + ">");
      e.attrs.emplace_back(k, v);
    }
    for (;;) {
      if (!misc()) return false;
      if (eof()) return fail("missing </" + e.tag + ">");
      if (starts("</")) {
        adv(2);
        std::string t;
        if (!name(t)) return false;
        if (t != e.tag) return fail("</" + t + "> closes <" + e.tag + ">");
        ws();
        if (eof() || s[i] != '>') return fail("expected '>'");
        adv();
        return true;
      }
      e.kids.emplace_back();
      if (!element(e.kids.back(), depth + 1)) return false;
    }
  }
  bool document(Elem& root) {
    if (!misc()) return false;
    if (eof()) return fail("no root element");
    if (!element(root, 0)) return false;
    if (!misc()) return false;
    if (!eof()) return fail("content after the root element");
    return true;
  }
};

// ------------------------------------------------------------------ MSCCL vocabulary
struct TypeName {
  const char* xml;
  Opcode op;
};
// MSCCL instruction names (msccl-tools Instruction): send 's', recv 'r', copy 'cpy', reduce 're',
// recv_reduce_copy 'rrc', recv_copy_send 'rcs', recv_reduce_copy_send 'rrcs', recv_reduce_send 'rrs'
const TypeName kTypes[] = {{"s", Opcode::send},   {"r", Opcode::recv},   {"cpy", Opcode::copy}, {"re", Opcode::reduce},
                           {"rrc", Opcode::rrc},  {"rcs", Opcode::rcs},  {"rrcs", Opcode::rrcs}, {"rrs", Opcode::rrs},
                           {"nop", Opcode::nop}};

const char* xml_type(Opcode op) {
  for (const auto& t : kTypes)
    if (t.op == op) return t.xml;
  return "nop";
}
char xml_buf(Buf b) { return b == Buf::input ? 'i' : (b == Buf::output ? 'o' : 's'); }
const char* xml_proto(Proto p) { return p == Proto::ll ? "LL" : (p == Proto::ll128 ? "LL128" : "Simple"); }
std::string xml_coll(const std::string& c) { return c == "reducescatter" ? "reduce_scatter" : c; }

struct Conv {
  std::string err;
  bool fail(const std::string& path, const std::string& m) {
    if (err.empty()) err = "xml: " + path + ": " + m;
    return false;
  }
  bool str(const Elem& e, const std::string& path, const char* k, std::string& out) {
    const std::string* v = e.attr(k);
    if (!v) return fail(path, std::string("missing attribute '") + k + "'");
    out = *v;
    return true;
  }
  bool integer(const Elem& e, const std::string& path, const char* k, long long& out, bool required = true,
               long long def = 0) {
    const std::string* v = e.attr(k);
    if (!v) {
      if (required) return fail(path, std::string("missing attribute '") + k + "'");
      out = def;
      return true;
    }
    if (v->empty()) return fail(path, std::string("attribute '") + k + "' is empty");
    char* end = nullptr;
    out = std::strtoll(v->c_str(), &end, 10);
    if (*end != '\0') return fail(path, std::string("attribute '") + k + "' is not an integer: \"" + *v + "\"");
    return true;
  }
  bool buffer(const Elem& e, const std::string& path, const char* k, Buf& out) {
    std::string v;
    if (!str(e, path, k, v)) return false;
    if (v == "i" || v == "input") out = Buf::input;
    else if (v == "o" || v == "output") out = Buf::output;
    else if (v == "s" || v == "scratch") out = Buf::scratch;
    else return fail(path, std::string("attribute '") + k + "' names an unknown buffer \"" + v + "\"");
    return true;
  }
};

}  // namespace

bool parse_msccl_xml(const std::string& text, Program& out, std::string& err, bool fold_nops) {
  Reader rd(text);
  Elem root;
  if (!rd.document(root)) {
    err = "xml: " + rd.err;
    return false;
  }
  Conv cv;
  auto done = [&](bool ok) {
    if (!ok) err = cv.err;
    return ok;
  };
  if (root.tag != "algo") return done(cv.fail("", "root element is <" + root.tag + ">, expected <algo>"));
  Program p;
  std::string v;
  long long x = 0;
  p.name = root.attr("name") ? *root.attr("name") : "";
  if (!cv.str(root, "algo", "coll", v)) return done(false);
  p.collective = v == "reduce_scatter" ? "reducescatter" : v;
  if (!known_collective(p.collective)) return done(cv.fail("algo", "unknown collective \"" + v + "\""));
  const std::string proto = root.attr("proto") ? *root.attr("proto") : "Simple";
  if (proto == "Simple" || proto == "simple") p.proto = Proto::simple;
  else if (proto == "LL" || proto == "ll") p.proto = Proto::ll;
  else if (proto == "LL128" || proto == "ll128") p.proto = Proto::ll128;
  else return done(cv.fail("algo", "unknown protocol \"" + proto + "\""));
  if (!cv.integer(root, "algo", "inplace", x, false, 0)) return done(false);
  p.inplace = x != 0;
  if (!cv.integer(root, "algo", "minBytes", x, false, 0)) return done(false);
  p.min_bytes = static_cast<uint64_t>(x);
  long long maxb = 0;
  if (!cv.integer(root, "algo", "maxBytes", maxb, false, 0)) return done(false);
  p.max_bytes = maxb > 0 ? static_cast<uint64_t>(maxb) : (1ull << 40);  // MSCCL: 0 = unbounded
  long long ngpus = -1;
  if (!cv.integer(root, "algo", "ngpus", ngpus, false, -1)) return done(false);

  // gpus in rank order
  std::map<int, const Elem*> by_rank;
  int gi = 0;
  for (const Elem& g : root.kids) {
    const std::string path = "algo.gpu[" + std::to_string(gi++) + "]";
    if (g.tag != "gpu") return done(cv.fail(path, "unexpected element <" + g.tag + ">"));
    long long id;
    if (!cv.integer(g, path, "id", id)) return done(false);
    if (id < 0 || by_rank.count(static_cast<int>(id))) return done(cv.fail(path, "bad or repeated gpu id " + std::to_string(id)));
    by_rank[static_cast<int>(id)] = &g;
  }
  if (by_rank.empty()) return done(cv.fail("algo", "no <gpu> elements"));
  if (by_rank.rbegin()->first != static_cast<int>(by_rank.size()) - 1)
    return done(cv.fail("algo", "gpu ids are not 0..R-1"));
  if (ngpus >= 0 && ngpus != static_cast<long long>(by_rank.size()))
    return done(cv.fail("algo", "ngpus=" + std::to_string(ngpus) + " but " + std::to_string(by_rank.size()) + " <gpu> elements"));

  // (rank, tb id, xml step) -> op; folded nops are recorded as absorbed into the next op
  struct Raw {
    Op op;
    int dep_tb = -1, dep_step = -1;
  };
  for (const auto& [rank, ge] : by_rank) {
    const std::string gpath = "algo.gpu[" + std::to_string(rank) + "]";
    Gpu gpu;
    gpu.rank = rank;
    const char* nk[3] = {"i_chunks", "o_chunks", "s_chunks"};
    for (int b = 0; b < 3; ++b) {
      if (!cv.integer(*ge, gpath, nk[b], x, false, 0)) return done(false);
      if (x < 0) return done(cv.fail(gpath, std::string(nk[b]) + " is negative"));
      p.nchunks[b] = std::max(p.nchunks[b], static_cast<int>(x));
    }
    int ti = 0;
    for (const Elem& te : ge->kids) {
      const std::string tpath = gpath + ".tb[" + std::to_string(ti++) + "]";
      if (te.tag != "tb") return done(cv.fail(tpath, "unexpected element <" + te.tag + ">"));
      ThreadBlock tb;
      long long a, b, c, d;
      if (!cv.integer(te, tpath, "id", a) || !cv.integer(te, tpath, "send", b) || !cv.integer(te, tpath, "recv", c) ||
          !cv.integer(te, tpath, "chan", d))
        return done(false);
      tb.id = static_cast<int>(a);
      tb.send_peer = static_cast<int>(b);
      tb.recv_peer = static_cast<int>(c);
      tb.channel = static_cast<int>(d);
      int si = 0;
      for (const Elem& se : te.kids) {
        const std::string spath = tpath + ".step[" + std::to_string(si) + "]";
        if (se.tag != "step" && se.tag != "op") return done(cv.fail(spath, "unexpected element <" + se.tag + ">"));
        Op op;
        long long s;
        if (!cv.integer(se, spath, se.tag == "step" ? "s" : "step", s)) return done(false);
        if (s != si) return done(cv.fail(spath, "step index " + std::to_string(s) + ", expected " + std::to_string(si)));
        op.step = si++;
        std::string ty;
        if (!cv.str(se, spath, "type", ty)) return done(false);
        bool known = false;
        for (const auto& t : kTypes)
          if (ty == t.xml) {
            op.op = t.op;
            known = true;
          }
        if (!known) return done(cv.fail(spath, "unsupported step type \"" + ty + "\""));
        long long so, dof, cnt, depid, deps, hasdep;
        if (!cv.buffer(se, spath, "srcbuf", op.src_buf) || !cv.integer(se, spath, "srcoff", so) ||
            !cv.buffer(se, spath, "dstbuf", op.dst_buf) || !cv.integer(se, spath, "dstoff", dof) ||
            !cv.integer(se, spath, "cnt", cnt) || !cv.integer(se, spath, "depid", depid, false, -1) ||
            !cv.integer(se, spath, "deps", deps, false, -1) || !cv.integer(se, spath, "hasdep", hasdep, false, 0))
          return done(false);
        op.src_off = so < 0 ? 0 : static_cast<int>(so);  // MSCCL writes -1 for an absent operand
        op.dst_off = dof < 0 ? 0 : static_cast<int>(dof);
        op.count = op.op == Opcode::nop && cnt < 1 ? 1 : static_cast<int>(cnt);  // a nop moves nothing
        if ((depid < 0) != (deps < 0)) return done(cv.fail(spath, "depid and deps must both be -1 or both set"));
        if (depid >= 0) op.deps.push_back(Dep{static_cast<int>(depid), static_cast<int>(deps)});
        op.has_dep = hasdep != 0;
        tb.ops.push_back(op);
      }
      gpu.tbs.push_back(std::move(tb));
    }
    p.gpus.push_back(std::move(gpu));
  }

  if (p.inplace && p.nchunks[1] == 0) p.nchunks[1] = p.nchunks[0];  // output aliases input
  if (fold_nops) {
    // nops that only wait (a dependency, nothing depends on them, not last) merge into the next op
    for (Gpu& g : p.gpus) {
      std::set<std::pair<int, int>> targets;
      for (const auto& tb : g.tbs)
        for (const auto& op : tb.ops)
          for (const auto& d : op.deps) targets.insert({d.tb, d.step});
      std::map<std::pair<int, int>, int> remap;  // (tb id, old step) -> new step
      for (ThreadBlock& tb : g.tbs) {
        std::vector<Op> kept;
        std::vector<Dep> pending;
        std::vector<int> absorbed;
        for (size_t k = 0; k < tb.ops.size(); ++k) {
          Op& op = tb.ops[k];
          const bool foldable = op.op == Opcode::nop && !op.has_dep && !op.deps.empty() && k + 1 < tb.ops.size() &&
                                !targets.count({tb.id, op.step});
          if (foldable) {
            pending.insert(pending.end(), op.deps.begin(), op.deps.end());
            absorbed.push_back(op.step);
            continue;
          }
          // a thread block runs its steps in order: of several dependencies on one thread block
          // only the latest step matters (the reference rejects duplicates, ir.hpp:341-439)
          for (const Dep& d : pending) {
            bool merged = false;
            for (Dep& e : op.deps)
              if (e.tb == d.tb) {
                e.step = std::max(e.step, d.step);
                merged = true;
              }
            if (!merged) op.deps.insert(op.deps.end() - static_cast<long>(op.deps.empty() ? 0 : 1), d);
          }
          pending.clear();
          const int ns = static_cast<int>(kept.size());
          for (int a : absorbed) remap[{tb.id, a}] = ns;
          absorbed.clear();
          remap[{tb.id, op.step}] = ns;
          op.step = ns;
          kept.push_back(op);
        }
        tb.ops = std::move(kept);
      }
      for (ThreadBlock& tb : g.tbs)
        for (Op& op : tb.ops)
          for (Dep& d : op.deps) {
            auto f = remap.find({d.tb, d.step});
            if (f != remap.end()) d.step = f->second;
          }
    }
  }
  out = std::move(p);
  return true;
}

std::string to_msccl_xml(const Program& p) {
  int nch = 0;
  for (const auto& g : p.gpus)
    for (const auto& tb : g.tbs) nch = std::max(nch, tb.channel + 1);
  std::ostringstream o;
  auto esc = [](const std::string& s) {
    std::string r;
    for (char c : s) {
      if (c == '<') r += "&lt;";
      else if (c == '>') r += "&gt;";
      else if (c == '&') r += "&amp;";
      else if (c == '"') r += "&quot;";
      else r += c;
    }
    return r;
  };
  o << "<algo name=\"" << esc(p.name) << "\" proto=\"" << xml_proto(p.proto) << "\" nchannels=\"" << nch
    << "\" nchunksperloop=\"" << std::max(p.nchunks[0], p.nchunks[1]) << "\" ngpus=\"" << p.ranks() << "\" coll=\""
    << xml_coll(p.collective) << "\" inplace=\"" << (p.inplace ? 1 : 0) << "\" outofplace=\"" << (p.inplace ? 0 : 1)
    << "\" minBytes=\"" << p.min_bytes << "\" maxBytes=\"" << p.max_bytes << "\">\n";
  for (const auto& g : p.gpus) {
    // new step index of every op after multi-dependency expansion
    std::map<std::pair<int, int>, int> pos;
    for (const auto& tb : g.tbs) {
      int n = 0;
      for (const auto& op : tb.ops) {
        n += op.deps.size() > 1 ? static_cast<int>(op.deps.size()) - 1 : 0;
        pos[{tb.id, op.step}] = n++;
      }
    }
    o << "  <gpu id=\"" << g.rank << "\" i_chunks=\"" << p.nchunks[0] << "\" o_chunks=\"" << p.nchunks[1] << "\" s_chunks=\""
      << p.nchunks[2] << "\">\n";
    for (const auto& tb : g.tbs) {
      o << "    <tb id=\"" << tb.id << "\" send=\"" << tb.send_peer << "\" recv=\"" << tb.recv_peer << "\" chan=\"" << tb.channel
        << "\">\n";
      int s = 0;
      auto step = [&](const char* type, Buf sb, int so, Buf db, int dof, int cnt, const Dep* d, bool hasdep) {
        int dt = -1, ds = -1;
        if (d) {
          dt = d->tb;
          auto f = pos.find({d->tb, d->step});
          ds = f != pos.end() ? f->second : d->step;
        }
        o << "      <step s=\"" << s++ << "\" type=\"" << type << "\" srcbuf=\"" << xml_buf(sb) << "\" srcoff=\"" << so
          << "\" dstbuf=\"" << xml_buf(db) << "\" dstoff=\"" << dof << "\" cnt=\"" << cnt << "\" depid=\"" << dt << "\" deps=\""
          << ds << "\" hasdep=\"" << (hasdep ? 1 : 0) << "\"/>\n";
      };
      for (const auto& op : tb.ops) {
        for (size_t k = 0; k + 1 < op.deps.size(); ++k)
          step("nop", op.src_buf, op.src_off, op.dst_buf, op.dst_off, op.count, &op.deps[k], false);
        step(xml_type(op.op), op.src_buf, op.src_off, op.dst_buf, op.dst_off, op.count, op.deps.empty() ? nullptr : &op.deps.back(),
             op.has_dep);
      }
      o << "    </tb>\n";
    }
    o << "  </gpu>\n";
  }
  o << "</algo>\n";
  return o.str();
}

}  // namespace gc3
