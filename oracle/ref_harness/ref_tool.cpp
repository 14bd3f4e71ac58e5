// Reference harness — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// Compiled by oracle/ref_harness/Makefile directly against the read-only reference headers in
// /root/reference/proj/include/cclforge (nlohmann/json 3.11.3 from the container's cudnn_frontend
// third-party tree stands in for the git-ignored vendor/ directory, proj/CMakeLists.txt:5).
// Nothing from the reference is copied here: this file only *calls* the reference API.
//
// Two build products, both written to oracle/_ref/ (git-ignored):
//   ref_tool   — `ref_tool gen <dir>` compiles the fixture IRs with the reference compiler
//                (program.hpp → chunk_dag.hpp → lowering.hpp → scheduler.hpp → ir.hpp), following
//                the recipe of SURVEY.md Appendix D, and writes canonical *.ir.json files.
//   libref.so  — C ABI used by tests/ to compare our own IR loader / validator / slot checker
//                with the reference implementations, and to pin the numeric oracle against the
//                reference's symbolic chunk algebra (core.hpp:94-161) and postconditions
//                (core.hpp:305-397, chunk_dag.hpp:133-149).
#include <cclforge/core.hpp>
#include <cclforge/chunk_dag.hpp>
#include <cclforge/program.hpp>
#include <cclforge/lowering.hpp>
#include <cclforge/ir.hpp>
#include <cclforge/scheduler.hpp>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <string>
#include <vector>

using namespace cclforge;

namespace {

topology make_topo(int nodes, int gpn) {
	topology t;
	t.nodes = nodes;
	t.gpus_per_node = gpn;
	return t;
}

directives ch_dir(int ch) {
	directives d;
	if(ch >= 0) d.ch = ch;
	return d;
}

// RS / AG helpers of SURVEY.md Appendix A.2 (PAPER.md "helper functions" listing).
void RS(program_builder& b, const std::vector<int>& ranks, int off, int cnt, int ch) {
	const int R = static_cast<int>(ranks.size());
	for(int r = 0; r < R; ++r) {
		const int idx = off + r * cnt;
		auto x = b.chunk(ranks[(r + 1) % R], buffer::input, idx, cnt);
		for(int step = 1; step < R; ++step) {
			x = b.chunk(ranks[(step + r + 1) % R], buffer::input, idx, cnt).reduce(x, ch_dir(ch));
		}
	}
}

void AG(program_builder& b, const std::vector<int>& ranks, int off, int cnt, int ch) {
	const int R = static_cast<int>(ranks.size());
	for(int r = 0; r < R; ++r) {
		const int idx = off + r * cnt;
		auto x = b.chunk(ranks[r], buffer::input, idx, cnt);
		for(int step = 1; step < R; ++step) {
			x = x.copy(ranks[(step + r) % R], buffer::input, idx, ch_dir(ch));
		}
	}
}

std::vector<int> iota_ranks(int n, int base = 0) {
	std::vector<int> v(n);
	for(int i = 0; i < n; ++i) v[i] = base + i;
	return v;
}

struct fixture {
	std::string name;
	std::string text;
};

std::string compile(program_builder& b, const topology& topo, bool fused, protocol proto) {
	auto dag = b.finalize();
	const auto rep = verify(dag);
	if(!rep.passed) throw std::runtime_error("verify failed: " + rep.summary());
	auto idag = lower(dag);
	auto f = fused ? fuse(idag) : idag;
	schedule_options opts;
	opts.proto = proto;
	auto ir = schedule(f, topo, opts);
	const auto issues = validate(ir, topo);
	if(!issues.empty()) throw std::runtime_error("validate failed: " + issues.front().what);
	return serialize(ir);
}

using gen_fn = std::function<std::string(bool fused, protocol proto)>;

std::map<std::string, gen_fn> generators() {
	std::map<std::string, gen_fn> g;

	// ring_ar_R_ch1: RS(all,0,1,ch=0); AG(all,0,1,ch=0); topo 1xR
	for(int R : {2, 4, 8}) {
		const std::string name = "ring_ar_" + std::to_string(R) + "_ch1";
		g[name] = [R, name](bool fused, protocol proto) {
			program_builder b(allreduce_spec(R, R), name);
			RS(b, iota_ranks(R), 0, 1, 0);
			AG(b, iota_ranks(R), 0, 1, 0);
			return compile(b, make_topo(1, R), fused, proto);
		};
	}
	// ring_ar_R_chR_instK: chunk r on channel r%8, wrapped in parallelize(K)
	for(int R : {2, 4, 8}) {
		for(int K : {1, 4}) {
			const std::string name = "ring_ar_" + std::to_string(R) + "_ch" + std::to_string(std::min(R, 8)) + "_inst" + std::to_string(K);
			g[name] = [R, K, name](bool fused, protocol proto) {
				program_builder b(allreduce_spec(R, R), name);
				b.parallelize(K, [&] {
					for(int r = 0; r < R; ++r) {
						auto x = b.chunk((r + 1) % R, buffer::input, r);
						for(int s = 1; s < R; ++s) x = b.chunk((s + r + 1) % R, buffer::input, r).reduce(x, ch_dir(r % 8));
					}
					for(int r = 0; r < R; ++r) {
						auto x = b.chunk(r, buffer::input, r);
						for(int s = 1; s < R; ++s) x = x.copy((s + r) % R, buffer::input, r, ch_dir(r % 8));
					}
				});
				return compile(b, make_topo(1, R), fused, proto);
			};
		}
	}
	// ring_ar_8_inst4_auto: parallelize(4, {RS; AG}) with no directives
	g["ring_ar_8_inst4_auto"] = [](bool fused, protocol proto) {
		program_builder b(allreduce_spec(8, 8), "ring_ar_8_inst4_auto");
		b.parallelize(4, [&] {
			RS(b, iota_ranks(8), 0, 1, -1);
			AG(b, iota_ranks(8), 0, 1, -1);
		});
		return compile(b, make_topo(1, 8), fused, proto);
	};
	// hier_ar_NxG_parP
	for(auto [N, G] : std::vector<std::pair<int, int>>{{2, 4}, {2, 2}}) {
		for(int par : {1, 2}) {
			if(G != 4 && par != 1) continue;
			const std::string name = "hier_ar_" + std::to_string(N) + "x" + std::to_string(G) + "_par" + std::to_string(par);
			g[name] = [N, G, par, name](bool fused, protocol proto) {
				const int a = 0, bch = par == 1 ? 1 : 2, c = par == 1 ? 2 : 4;
				program_builder b(allreduce_spec(N * G, N * G), name);
				for(int n = 0; n < N; ++n) b.parallelize(par, [&] { RS(b, iota_ranks(G, n * G), 0, N, a); });
				for(int gg = 0; gg < G; ++gg) {
					std::vector<int> cross;
					for(int n = 0; n < N; ++n) cross.push_back(n * G + gg);
					RS(b, cross, gg * N, 1, bch);
					AG(b, cross, gg * N, 1, bch);
				}
				for(int n = 0; n < N; ++n) b.parallelize(par, [&] { AG(b, iota_ranks(G, n * G), 0, N, c); });
				return compile(b, make_topo(N, G), fused, proto);
			};
		}
	}
	// twostep_a2a_NxG
	for(auto [N, G] : std::vector<std::pair<int, int>>{{2, 4}, {1, 8}, {1, 2}, {1, 4}, {2, 2}, {2, 1}}) {
		const std::string name = "twostep_a2a_" + std::to_string(N) + "x" + std::to_string(G);
		g[name] = [N, G, name](bool fused, protocol proto) {
			const int R = N * G;
			program_builder b(alltoall_spec(R), name);
			const auto rk = [G](int n, int gg) { return n * G + gg; };
			for(int n = 0; n < N; ++n)
				for(int gg = 0; gg < G; ++gg)
					for(int m = 0; m < N; ++m)
						for(int i = 0; i < G; ++i) {
							auto c = b.chunk(rk(m, i), buffer::input, rk(n, gg));
							if(n == m) c.copy(rk(n, gg), buffer::output, rk(m, i));
							else c.copy(rk(m, gg), buffer::scratch, rk(n, i));
						}
			for(int n = 0; n < N; ++n)
				for(int gg = 0; gg < G; ++gg)
					for(int m = 0; m < N; ++m) {
						if(m == n) continue;
						b.chunk(rk(m, gg), buffer::scratch, n * G, G).copy(rk(n, gg), buffer::output, m * G);
					}
			return compile(b, make_topo(N, G), fused, proto);
		};
	}
	// ring_ag_R / ring_rs_R / allpairs_ar_R
	for(int R : {2, 4, 8}) {
		const std::string ag = "ring_ag_" + std::to_string(R);
		g[ag] = [R, ag](bool fused, protocol proto) {
			program_builder b(allgather_spec(R, 1), ag);
			for(int r = 0; r < R; ++r) {
				auto x = b.chunk(r, buffer::input, 0).copy(r, buffer::output, r);
				for(int s = 1; s < R; ++s) x = x.copy((r + s) % R, buffer::output, r);
			}
			return compile(b, make_topo(1, R), fused, proto);
		};
		const std::string rs = "ring_rs_" + std::to_string(R);
		g[rs] = [R, rs](bool fused, protocol proto) {
			program_builder b(reducescatter_spec(R, 1), rs);
			for(int r = 0; r < R; ++r) {
				auto x = b.chunk((r + 1) % R, buffer::input, r);
				for(int s = 2; s <= R; ++s) x = b.chunk((r + s) % R, buffer::input, r).reduce(x);
			}
			return compile(b, make_topo(1, R), fused, proto);
		};
		const std::string ap = "allpairs_ar_" + std::to_string(R);
		g[ap] = [R, ap](bool fused, protocol proto) {
			program_builder b(allreduce_spec(R, R), ap);
			for(int r = 0; r < R; ++r)
				for(int q = 0; q < R; ++q)
					if(q != r) b.chunk(r, buffer::input, r).reduce(b.chunk(q, buffer::input, r));
			for(int r = 0; r < R; ++r)
				for(int q = 0; q < R; ++q)
					if(q != r) b.chunk(r, buffer::input, r).copy(q, buffer::input, r);
			return compile(b, make_topo(1, R), fused, proto);
		};
	}
	return g;
}

char* dup_string(const std::string& s) {
	char* p = static_cast<char*>(std::malloc(s.size() + 1));
	std::memcpy(p, s.c_str(), s.size() + 1);
	return p;
}

collective_spec spec_for(const ir_program& ir) {
	const int R = ir.ranks();
	const auto kind = parse_collective_kind(ir.collective);
	switch(*kind) {
	case collective_kind::allreduce: return allreduce_spec(R, ir.nchunks.input);
	case collective_kind::allgather: return allgather_spec(R, ir.nchunks.input);
	case collective_kind::reducescatter: return reducescatter_spec(R, ir.nchunks.input / R);
	case collective_kind::alltoall: return alltoall_spec(R, ir.nchunks.input / R);
	case collective_kind::alltonext: return alltonext_spec(R, ir.nchunks.input);
	default: return custom_spec(R, ir.nchunks.input, ir.nchunks.output, ir.inplace);
	}
}

// Symbolic execution of an IR over the reference's chunk algebra. The schedule is the simplest
// legal one (round-robin over thread blocks, unbounded FIFOs); the opcode semantics are those of
// lowering.hpp:68-77 + 96-119, deps/has_dep of scheduler.hpp:519-559, FIFO matching of
// scheduler.hpp:655-683.
std::string symbolic_run(const ir_program& ir, bool& passed, std::string& err) {
	const auto spec = spec_for(ir);
	buffer_state st(spec, ir.nchunks.scratch);
	struct tb_state {
		size_t pc = 0;
		int sem = -1;
	};
	const int R = ir.ranks();
	std::vector<std::vector<tb_state>> tbs(R);
	for(int r = 0; r < R; ++r) tbs[r].resize(ir.gpus[r].threadblocks.size());
	std::map<std::tuple<int, int, int>, std::deque<std::vector<chunk_value>>> fifo;
	const auto tb_index = [&](int r, int id) {
		for(size_t i = 0; i < ir.gpus[r].threadblocks.size(); ++i)
			if(ir.gpus[r].threadblocks[i].id == id) return static_cast<int>(i);
		return -1;
	};
	bool progress = true;
	try {
		while(progress) {
			progress = false;
			for(int r = 0; r < R; ++r) {
				for(size_t t = 0; t < ir.gpus[r].threadblocks.size(); ++t) {
					const auto& tb = ir.gpus[r].threadblocks[t];
					auto& ts = tbs[r][t];
					while(ts.pc < tb.ops.size()) {
						const auto& op = tb.ops[ts.pc];
						bool ready = true;
						for(const auto& d : op.deps)
							if(tbs[r][tb_index(r, d.tb)].sem < d.step) ready = false;
						const auto in_key = std::make_tuple(tb.recv_peer, r, tb.channel);
						const auto out_key = std::make_tuple(r, tb.send_peer, tb.channel);
						if(receives(op.op) && fifo[in_key].empty()) ready = false;
						if(!ready) break;
						std::vector<chunk_value> msg;
						if(receives(op.op)) {
							msg = fifo[in_key].front();
							fifo[in_key].pop_front();
						}
						std::vector<chunk_value> out(op.count);
						for(int i = 0; i < op.count; ++i) {
							switch(op.op) {
							case opcode::send: out[i] = st.at(r, op.src_buf, op.src_off + i); break;
							case opcode::recv: st.set(r, op.dst_buf, op.dst_off + i, msg[i]); break;
							case opcode::copy: st.set(r, op.dst_buf, op.dst_off + i, st.at(r, op.src_buf, op.src_off + i)); break;
							case opcode::reduce:
								st.set(r, op.dst_buf, op.dst_off + i, reduce_values(st.at(r, op.dst_buf, op.dst_off + i), st.at(r, op.src_buf, op.src_off + i)));
								break;
							case opcode::recv_reduce_copy: st.set(r, op.dst_buf, op.dst_off + i, reduce_values(st.at(r, op.src_buf, op.src_off + i), msg[i])); break;
							case opcode::recv_copy_send:
								st.set(r, op.src_buf, op.src_off + i, msg[i]);
								out[i] = msg[i];
								break;
							case opcode::recv_reduce_copy_send: {
								auto v = reduce_values(st.at(r, op.src_buf, op.src_off + i), msg[i]);
								st.set(r, op.src_buf, op.src_off + i, v);
								out[i] = v;
								break;
							}
							case opcode::recv_reduce_send: out[i] = reduce_values(st.at(r, op.src_buf, op.src_off + i), msg[i]); break;
							case opcode::nop: break;
							}
						}
						if(sends(op.op)) fifo[out_key].push_back(out);
						if(op.has_dep) ts.sem = static_cast<int>(ts.pc);
						ts.pc++;
						progress = true;
					}
				}
			}
		}
	} catch(const std::exception& e) {
		err = e.what();
		passed = false;
		return "";
	}
	for(int r = 0; r < R; ++r)
		for(size_t t = 0; t < tbs[r].size(); ++t)
			if(tbs[r][t].pc < ir.gpus[r].threadblocks[t].ops.size()) {
				err = "deadlock";
				passed = false;
				return st.canonical_json();
			}
	passed = check_postcondition(st, spec).passed;
	return st.canonical_json();
}

std::string json_escape(const std::string& s) {
	nlohmann::json j = s;
	return j.dump();
}

} // namespace

extern "C" {

/// deserialize + validate + canonical re-serialize with the reference (ir.hpp:145-439).
char* ref_load(const char* text, int nodes, int gpn, int max_tb, int max_ch) {
	nlohmann::json out;
	try {
		const auto ir = deserialize(text);
		auto topo = make_topo(nodes, gpn);
		if(max_tb > 0) topo.max_threadblocks = max_tb;
		if(max_ch > 0) topo.max_channels = max_ch;
		nlohmann::json issues = nlohmann::json::array();
		for(const auto& i : validate(ir, topo)) issues.push_back(i.what);
		out["schema_error"] = nullptr;
		out["issues"] = issues;
		out["canonical"] = serialize(ir);
	} catch(const schema_error& e) {
		out["schema_error"] = {{"path", e.path()}, {"what", e.what()}};
	} catch(const std::exception& e) {
		out["schema_error"] = {{"path", "?"}, {"what", e.what()}};
	}
	return dup_string(out.dump());
}

/// check_slots(ir, s) (scheduler.hpp:633-734): list of violation messages.
char* ref_check_slots(const char* text, int slots) {
	nlohmann::json out = nlohmann::json::array();
	try {
		for(const auto& v : check_slots(deserialize(text), slots)) out.push_back(v.what);
	} catch(const std::exception& e) {
		out.push_back(std::string("error: ") + e.what());
	}
	return dup_string(out.dump());
}

/// Symbolic run + reference postcondition: {"passed": bool, "error": str, "state": canonical_json}.
char* ref_symbolic(const char* text) {
	nlohmann::json out;
	try {
		const auto ir = deserialize(text);
		bool passed = true;
		std::string err;
		const auto state = symbolic_run(ir, passed, err);
		out["passed"] = passed;
		out["error"] = err;
		out["state"] = state.empty() ? nlohmann::json(nullptr) : nlohmann::json::parse(state);
	} catch(const std::exception& e) {
		out["passed"] = false;
		out["error"] = e.what();
		out["state"] = nullptr;
	}
	return dup_string(out.dump());
}

// Parametric generators for the runtime's built-in program families (tests/test_builtin_irs.py):
//   gen_ring_ar_R_C_K   ring AllReduce, chunk r on channel r % C, parallelize(K)
//   gen_allpairs_ar_R   all-pairs AllReduce
//   gen_hier_ar_N_G_P   hierarchical AllReduce N nodes x G GPUs, parallelize(P)
//   gen_ring_ag_R_K / gen_ring_rs_R_K   ring AllGather / ReduceScatter, parallelize(K)
gen_fn param_generator(const std::string& name) {
	std::vector<int> v;
	std::string kind;
	{
		std::string s = name.substr(4);
		size_t i = 0;
		while(i < s.size() && !std::isdigit(static_cast<unsigned char>(s[i]))) kind += s[i++];
		while(i < s.size()) {
			size_t j = i;
			while(j < s.size() && std::isdigit(static_cast<unsigned char>(s[j]))) ++j;
			v.push_back(std::stoi(s.substr(i, j - i)));
			i = j + 1;
		}
	}
	if(kind == "ring_ar_" && v.size() == 3) {
		const int R = v[0], C = v[1], K = v[2];
		return [R, C, K, name](bool fused, protocol proto) {
			program_builder b(allreduce_spec(R, R), name);
			b.parallelize(K, [&] {
				for(int r = 0; r < R; ++r) {
					auto x = b.chunk((r + 1) % R, buffer::input, r);
					for(int s = 1; s < R; ++s) x = b.chunk((s + r + 1) % R, buffer::input, r).reduce(x, ch_dir(r % C));
				}
				for(int r = 0; r < R; ++r) {
					auto x = b.chunk(r, buffer::input, r);
					for(int s = 1; s < R; ++s) x = x.copy((s + r) % R, buffer::input, r, ch_dir(r % C));
				}
			});
			return compile(b, make_topo(1, R), fused, proto);
		};
	}
	if(kind == "allpairs_ar_" && v.size() == 1) {
		const int R = v[0];
		return [R, name](bool fused, protocol proto) {
			program_builder b(allreduce_spec(R, R), name);
			for(int r = 0; r < R; ++r)
				for(int q = 0; q < R; ++q)
					if(q != r) b.chunk(r, buffer::input, r).reduce(b.chunk(q, buffer::input, r));
			for(int r = 0; r < R; ++r)
				for(int q = 0; q < R; ++q)
					if(q != r) b.chunk(r, buffer::input, r).copy(q, buffer::input, r);
			return compile(b, make_topo(1, R), fused, proto);
		};
	}
	if(kind == "hier_ar_" && v.size() == 3) {
		const int N = v[0], G = v[1], par = v[2];
		return [N, G, par, name](bool fused, protocol proto) {
			const int a = 0, bch = par, c = 2 * par;
			program_builder b(allreduce_spec(N * G, N * G), name);
			for(int n = 0; n < N; ++n) b.parallelize(par, [&] { RS(b, iota_ranks(G, n * G), 0, N, a); });
			for(int gg = 0; gg < G; ++gg) {
				std::vector<int> cross;
				for(int n = 0; n < N; ++n) cross.push_back(n * G + gg);
				RS(b, cross, gg * N, 1, bch);
				AG(b, cross, gg * N, 1, bch);
			}
			for(int n = 0; n < N; ++n) b.parallelize(par, [&] { AG(b, iota_ranks(G, n * G), 0, N, c); });
			return compile(b, make_topo(N, G), fused, proto);
		};
	}
	if((kind == "ring_ag_" || kind == "ring_rs_") && v.size() == 2) {
		const int R = v[0], K = v[1];
		const bool ag = kind == "ring_ag_";
		return [R, K, ag, name](bool fused, protocol proto) {
			program_builder b(ag ? allgather_spec(R, 1) : reducescatter_spec(R, 1), name);
			b.parallelize(K, [&] {
				for(int r = 0; r < R; ++r) {
					if(ag) {
						auto x = b.chunk(r, buffer::input, 0).copy(r, buffer::output, r);
						for(int s = 1; s < R; ++s) x = x.copy((r + s) % R, buffer::output, r);
					} else {
						auto x = b.chunk((r + 1) % R, buffer::input, r);
						for(int s = 2; s <= R; ++s) x = b.chunk((r + s) % R, buffer::input, r).reduce(x);
					}
				}
			});
			return compile(b, make_topo(1, R), fused, proto);
		};
	}
	return nullptr;
}

/// Compiles one named fixture with the reference compiler. proto: 0 simple, 1 ll, 2 ll128.
char* ref_compile(const char* name, int fused, int proto) {
	const auto gens = generators();
	auto it = gens.find(name);
	gen_fn param;
	if(it == gens.end() && std::string(name).rfind("gen_", 0) == 0) param = param_generator(name);
	if(it == gens.end() && !param) return nullptr;
	if(param) {
		try {
			return dup_string(param(fused != 0, static_cast<protocol>(proto)));
		} catch(const std::exception& e) {
			return dup_string(std::string("ERROR: ") + e.what());
		}
	}
	try {
		return dup_string(it->second(fused != 0, static_cast<protocol>(proto)));
	} catch(const std::exception& e) {
		return dup_string(std::string("ERROR: ") + e.what());
	}
}

/// Newline-separated list of fixture generator names.
char* ref_fixture_names() {
	std::string s;
	for(const auto& [k, v] : generators()) s += k + "\n";
	return dup_string(s);
}

void ref_free(char* p) { std::free(p); }

} // extern "C"

#ifndef REF_LIB
int main(int argc, char** argv) {
	if(argc < 3 || std::string(argv[1]) != "gen") {
		std::fprintf(stderr, "usage: ref_tool gen <outdir>\n");
		return 2;
	}
	const std::string dir = argv[2];
	for(const auto& [name, gen] : generators()) {
		try {
			write_file_atomic(dir + "/" + name + ".ir.json", gen(true, protocol::simple));
			write_file_atomic(dir + "/" + name + ".unfused.ir.json", gen(false, protocol::simple));
		} catch(const std::exception& e) {
			std::fprintf(stderr, "%s: %s\n", name.c_str(), e.what());
			return 1;
		}
	}
	return 0;
}
#endif
