"""Timed simulator (csrc/timed.cpp, gc3IrSimulate / gc3IrSweep): SPEC.md:464-481's run_timed and
sweep examples and invariants -- a discrete-event alpha-beta model with chunk tiling, processor
sharing on ordered GPU pairs, per-protocol multipliers."""
import json

import pytest

from conftest import read_ir

gc3 = pytest.importorskip("paper_2201_11840_b200.gc3")

A, BW = 3.0, 100.0  # alpha (us) and GB/s used by the closed-form checks (1 GB/s = 1e3 bytes/us)


def _ir(gpus, nchunks=(4, 4, 0), inplace=False, coll="custom"):
    j = {"name": "hand", "collective": coll, "protocol": "simple", "inplace": inplace,
         "nchunks": {"input": nchunks[0], "output": nchunks[1], "scratch": nchunks[2]},
         "size_range": {"min_bytes": 0, "max_bytes": 1 << 40},
         "gpus": [{"rank": r, "threadblocks": tbs} for r, tbs in enumerate(gpus)]}
    return gc3.IR(json.dumps(j))


def _op(step, opcode, off=0, count=1, buf="input"):
    return {"step": step, "opcode": opcode, "src_buf": buf, "src_off": off, "dst_buf": buf, "dst_off": off,
            "count": count, "has_dep": False, "deps": []}


def _tb(i, ops, send=-1, recv=-1, ch=0):
    return {"id": i, "send_peer": send, "recv_peer": recv, "channel": ch, "ops": ops}


def _flat(**kw):
    # one link class with alpha A, bandwidth BW; free local work
    kw.setdefault("alpha_us", [A, A, A])
    kw.setdefault("gbps", [BW, BW, BW])
    kw.setdefault("gamma_gbps", 1e12)
    kw.setdefault("copy_gbps", 1e12)
    return kw


def test_one_send_is_alpha_plus_bytes_over_bandwidth():
    ir = _ir([[_tb(0, [_op(0, "send")], send=1)], [_tb(0, [_op(0, "recv")], recv=0)]])
    B = 1 << 20
    r = ir.simulate(B, **_flat())
    assert r["completed"] and r["messages"] == 1
    assert r["makespan_us"] == pytest.approx(A + B / (BW * 1e3))


def test_aggregation_saves_g_minus_one_alphas():
    G, B = 4, 1 << 18
    agg = _ir([[_tb(0, [_op(0, "send", 0, G)], send=1)], [_tb(0, [_op(0, "recv", 0, G)], recv=0)]])
    sep = _ir([[_tb(0, [_op(s, "send", s) for s in range(G)], send=1)],
               [_tb(0, [_op(s, "recv", s) for s in range(G)], recv=0)]])
    ta = agg.simulate(B, **_flat(slots=G))["makespan_us"]
    ts = sep.simulate(B, **_flat(slots=G))["makespan_us"]
    assert ts - ta == pytest.approx((G - 1) * A)


def test_processor_sharing_on_an_ordered_pair():
    # two channels between the same GPUs: the messages share the pair's bandwidth
    B = 1 << 20
    two = _ir([[_tb(0, [_op(0, "send", 0)], send=1, ch=0), _tb(1, [_op(0, "send", 1)], send=1, ch=1)],
               [_tb(0, [_op(0, "recv", 0)], recv=0, ch=0), _tb(1, [_op(0, "recv", 1)], recv=0, ch=1)]])
    r = two.simulate(B, **_flat())
    assert r["makespan_us"] == pytest.approx(A + 2 * B / (BW * 1e3))
    # on different GPU pairs (ranks on distinct GPUs, opposite directions) they do not interfere
    opp = _ir([[_tb(0, [_op(0, "send", 0)], send=1), _tb(1, [_op(0, "recv", 1)], recv=1)],
               [_tb(0, [_op(0, "recv", 0)], recv=0), _tb(1, [_op(0, "send", 1)], send=0)]])
    r = opp.simulate(B, **_flat())
    assert r["makespan_us"] == pytest.approx(A + B / (BW * 1e3))


def test_hierarchical_pipelining_with_tiles():
    """SPEC: hierarchical AllReduce N=2, G=2: makespan with 4 tiles < with 1 tile (alpha small)."""
    ir = gc3.IR(read_ir("hier_ar_2x2_par1"))
    C = 4 << 20
    one = ir.simulate(C, 0, **_flat(alpha_us=[0.1, 0.1, 0.1]), gpus_per_node=2)["makespan_us"]
    four = ir.simulate(C, C // 4, **_flat(alpha_us=[0.1, 0.1, 0.1]), gpus_per_node=2)["makespan_us"]
    assert four < one


def test_allpairs_vs_ring_alpha_terms_at_small_sizes():
    """SPEC: at small sizes the critical path of All-Pairs has 2 message steps vs Ring's 2R-2."""
    R = 8
    ring = gc3.IR(read_ir("ring_ar_8_ch1"))
    ap = gc3.IR.generate("allpairs", "allreduce", R)
    kw = _flat(gbps=[1e12, 1e12, 1e12])  # alpha only
    t_ring = ring.simulate(64, **kw)["makespan_us"]
    t_ap = ap.simulate(64, **kw)["makespan_us"]
    assert t_ring == pytest.approx((2 * R - 2) * A)
    assert t_ap == pytest.approx(2 * A)
    # the compiler's all-pairs fuses the last reduction with the first final send (rrcs); the other
    # final sends depend on that op, which completes when its message is delivered: one alpha more
    t_fused = gc3.IR(read_ir("allpairs_ar_8")).simulate(64, **kw)["makespan_us"]
    assert t_fused == pytest.approx(3 * A)


def test_monotone_in_alpha_and_beta_and_fused_not_slower():
    ir = gc3.IR(read_ir("ring_ar_8_ch8_inst4"))
    unf = gc3.IR(read_ir("ring_ar_8_ch8_inst4.unfused"))
    base = ir.simulate(1 << 20, 1 << 18, **_flat())["makespan_us"]
    assert ir.simulate(1 << 20, 1 << 18, **_flat(alpha_us=[2 * A] * 3))["makespan_us"] > base
    assert ir.simulate(1 << 20, 1 << 18, **_flat(gbps=[BW / 2] * 3))["makespan_us"] > base
    assert unf.simulate(1 << 20, 1 << 18, **_flat())["makespan_us"] >= base


def test_alpha_zero_single_hop_is_tile_invariant():
    ir = _ir([[_tb(0, [_op(0, "send")], send=1)], [_tb(0, [_op(0, "recv")], recv=0)]])
    B = 1 << 20
    ts = [ir.simulate(B, B // k, **_flat(alpha_us=[0, 0, 0]))["makespan_us"] for k in (1, 4, 16)]
    assert ts == pytest.approx([ts[0]] * 3)


def test_protocol_multipliers():
    ir = _ir([[_tb(0, [_op(0, "send")], send=1)], [_tb(0, [_op(0, "recv")], recv=0)]])
    B = 1 << 20
    ll = ir.simulate(B, protocol="ll", **_flat())["makespan_us"]
    assert ll == pytest.approx(0.25 * A + 2 * B / (BW * 1e3))


def test_deadlock_reported():
    # s = 1 deadlock of SURVEY.md Finding 1 (the oracle's test_s1_deadlock_despite_static_check IRs)
    ir = _ir([[_tb(0, [_op(0, "send", 0), _op(1, "send", 1)], send=1), _tb(1, [_op(0, "recv", 2)], recv=1, ch=1)],
              [_tb(0, [_op(0, "recv", 0), _op(1, "recv", 1)], recv=0), _tb(1, [_op(0, "send", 2)], send=0, ch=1)]])
    ok = ir.simulate(1024, **_flat(slots=2))
    assert ok["completed"]
    # receiver waits for a message that is never sent: blocked
    bad = _ir([[_tb(0, [_op(0, "recv", 0)], recv=1)], [_tb(0, [_op(0, "recv", 0)], recv=0)]])
    r = bad.simulate(1024, **_flat())
    assert not r["completed"] and r["deadlock"].startswith("deadlock")


def test_empty_program_and_sweep_csv():
    ir = _ir([[_tb(0, [])], [_tb(0, [])]])
    assert ir.simulate(1 << 20)["makespan_us"] == 0.0
    ring = gc3.IR(read_ir("ring_ar_8_ch1"))
    csv = ring.sweep([1 << 10, 1 << 20, 64 << 20], tile_bytes=1 << 18, rank_gpu=list(range(8)))
    lines = csv.strip().split("\n")
    assert lines[0] == "size_bytes,makespan_us,util_intra,util_inter"
    rows = [list(map(float, l.split(","))) for l in lines[1:]]
    assert [int(r[0]) for r in rows] == [1 << 10, 1 << 20, 64 << 20]
    assert rows[0][1] < rows[1][1] < rows[2][1]
    assert all(0 < r[2] <= 1 for r in rows) and all(r[3] == 0 for r in rows)  # one node: no inter-node links
    assert csv == ring.sweep([1 << 10, 1 << 20, 64 << 20], tile_bytes=1 << 18, rank_gpu=list(range(8)))  # deterministic


def test_link_classes_follow_placement():
    ring = gc3.IR(read_ir("ring_ar_8_ch1"))
    loop = ring.simulate(1 << 20, rank_gpu=[0] * 8)
    nv = ring.simulate(1 << 20, rank_gpu=list(range(8)))
    two_nodes = ring.simulate(1 << 20, rank_gpu=list(range(8)), gpus_per_node=4)
    assert loop["util"][0] > 0 and loop["util"][1] == 0
    assert nv["util"][1] > 0 and nv["util"][0] == 0
    assert two_nodes["util"][2] > 0
    assert two_nodes["makespan_us"] > nv["makespan_us"]


def test_unknown_parameter_rejected():
    ir = _ir([[_tb(0, [_op(0, "send")], send=1)], [_tb(0, [_op(0, "recv")], recv=0)]])
    with pytest.raises(TypeError):
        ir.simulate(1024, alpah_us=[1, 1, 1])


def _dev(**kw):
    # device-memory mode, all ranks on one GPU (the loopback calibration's setting)
    kw.setdefault("alpha_us", [A, A, A])
    kw.setdefault("gbps", [1e9, 1e9, 1e9])
    kw.setdefault("gamma_gbps", 1e9)
    kw.setdefault("copy_gbps", 1e9)
    kw.setdefault("hbm_gbps", BW)
    return kw


def test_dataflow_single_send_closed_form():
    """workers > 0 (dataflow executor): a send's local bytes on the device-memory resource, then alpha;
    the receive's local bytes after delivery."""
    ir = _ir([[_tb(0, [_op(0, "send")], send=1)], [_tb(0, [_op(0, "recv")], recv=0)]])
    B = 1 << 20
    r = ir.simulate(B, rank_gpu=[0, 0], workers=4, **_dev())
    assert r["completed"] and r["messages"] == 1
    # send reads B, recv writes B (one pass each), serialised by the dependency; alpha in between
    assert r["makespan_us"] == pytest.approx(A + 2 * B / (BW * 1e3))


def test_dataflow_more_workers_not_slower_and_matches_static_on_one_tile():
    ir = gc3.IR(read_ir("ring_ar_8_ch8_inst4"))
    C, T = 4 << 20, 1 << 18
    ts = [ir.simulate(C, T, rank_gpu=[0] * 8, workers=w, **_dev(alpha_us=[0.5] * 3, hbm_gbps=4000.0))
          for w in (1, 8, 64, 592)]
    assert all(t["completed"] for t in ts)
    ms = [t["makespan_us"] for t in ts]
    assert ms[0] >= ms[1] >= ms[2] >= ms[3] * 0.999
    assert ms[0] > 2 * ms[3]  # one unit serialises everything


def test_dataflow_reports_deadlock():
    bad = _ir([[_tb(0, [_op(0, "recv", 0)], recv=1)], [_tb(0, [_op(0, "recv", 0)], recv=0)]])
    r = bad.simulate(1024, rank_gpu=[0, 0], workers=4, **_dev())
    assert not r["completed"] and r["deadlock"].startswith("deadlock")


def test_dataflow_link_mode_matches_static_single_hop():
    """Without the device-memory resource, a dataflow message pays alpha + bytes / pair bandwidth,
    processor-shared on its ordered GPU pair like the static model."""
    B = 1 << 20
    one = _ir([[_tb(0, [_op(0, "send")], send=1)], [_tb(0, [_op(0, "recv")], recv=0)]])
    assert one.simulate(B, workers=2, **_flat())["makespan_us"] == pytest.approx(A + B / (BW * 1e3))
    two = _ir([[_tb(0, [_op(0, "send", 0)], send=1, ch=0), _tb(1, [_op(0, "send", 1)], send=1, ch=1)],
               [_tb(0, [_op(0, "recv", 0)], recv=0, ch=0), _tb(1, [_op(0, "recv", 1)], recv=0, ch=1)]])
    r = two.simulate(B, workers=4, **_flat())
    assert r["makespan_us"] == pytest.approx(A + 2 * B / (BW * 1e3))
    xfer = 2 * B / (BW * 1e3)
    assert r["util"][1] == pytest.approx(xfer / (A + xfer))  # busy after the alpha
