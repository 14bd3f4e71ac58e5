"""Message transports (direct / pulled / FIFO) checked operationally, independently of the C++
happens-before analysis that chose them (runtime.cpp direct_messages).

An interleaving interpreter in plain Python executes the IR with ops as atomic steps in a random
order (any op whose deps are done and whose incoming message has been sent may run), moving each
message the way its flags say:
  * FIFO:   the sender pushes its value, the receiver pops it;
  * direct: the sender writes its value into the receiver's span (its op's dst fields) when it runs;
            the receiver finds it in place;
  * pulled: the sender stores nothing extra; the receiver reads the sender's span (the sending op's
            src span) when it runs.
If a transport were unsafe, some interleaving would let a direct write clobber a live span, or let
a pulled read see a span that changed after the send; the result would then differ from the
all-FIFO execution. Integer sums make every difference visible.
"""
import json
import random

import numpy as np
import pytest

from conftest import read_ir

gc3 = pytest.importorskip("paper_2201_11840_b200.gc3")

BUFS = {"input": 0, "output": 1, "scratch": 2}
SENDS = {"send", "rcs", "rrcs", "rrs"}
RECVS = {"recv", "rrc", "rcs", "rrcs", "rrs"}


def run(irj, flags, seed, use_flags=True, source=None, result=None):
    """source: flags of the const-source analysis; the working input then starts as garbage and
    flagged reads see the caller's (initial) data instead."""
    R = len(irj["gpus"])
    nin, nout, nsc = irj["nchunks"]["input"], irj["nchunks"]["output"], irj["nchunks"]["scratch"]
    rng = np.random.default_rng(1234)
    bufs, const = [], []
    for r in range(R):
        inp = rng.integers(-1000, 1000, nin).astype(np.int64)
        const.append(inp.copy())
        if source is not None:
            inp[:] = 77777  # the working buffer is not initialised
        out = inp if irj["inplace"] else np.zeros(max(nout, 1), np.int64)
        bufs.append([inp, out, np.zeros(max(nsc, 1), np.int64)])
    res = [np.full(max(nin, 1), 55555, np.int64) for _ in range(R)]  # the result buffers (recvbuff)

    def span(r, b, off, cnt):
        return bufs[r][BUFS[b]][off:off + cnt]

    def rspan(r, b, off, cnt, t, s, bit):  # a read: from the caller's buffer when flagged
        if source is not None and source[r][t][s] & bit:
            return const[r][off:off + cnt]
        return span(r, b, off, cnt)

    tbs = [(r, t, tb) for r, g in enumerate(irj["gpus"]) for t, tb in enumerate(g["threadblocks"])]
    ids = {(r, tb["id"]): t for r, g in enumerate(irj["gpus"]) for t, tb in enumerate(g["threadblocks"])}
    pc = {(r, t): 0 for r, t, _ in tbs}
    fifo = {}     # (src, dst, ch) -> list of values (FIFO transport)
    posted = {}   # (src, dst, ch) -> list of (sender rank, sender op) in send order
    taken = {}    # (src, dst, ch) -> messages consumed
    rnd = random.Random(seed)
    while True:
        ready = []
        for r, t, tb in tbs:
            s = pc[(r, t)]
            if s >= len(tb["ops"]):
                continue
            op = tb["ops"][s]
            if any(pc[(r, ids[(r, d["tb"])])] <= d["step"] for d in op["deps"]):
                continue
            if op["opcode"] in RECVS:
                key = (tb["recv_peer"], r, tb["channel"])
                if len(posted.get(key, [])) <= taken.get(key, 0):
                    continue
            ready.append((r, t, tb))
        if not ready:
            break
        r, t, tb = rnd.choice(ready)
        s = pc[(r, t)]
        op = tb["ops"][s]
        f = flags[r][t][s] if use_flags else 0
        oc, cnt = op["opcode"], op["count"]
        src = span(r, op["src_buf"], op["src_off"], cnt)
        dst = span(r, op["dst_buf"], op["dst_off"], cnt)
        if result is not None and result[r][t][s]:  # final owned write: straight to recvbuff
            dst = res[r][op["dst_off"]:op["dst_off"] + cnt]
        srcr = rspan(r, op["src_buf"], op["src_off"], cnt, t, s, 1)
        dstr = rspan(r, op["dst_buf"], op["dst_off"], cnt, t, s, 2)
        msg = None
        if oc in RECVS:
            key = (tb["recv_peer"], r, tb["channel"])
            k = taken.get(key, 0)
            taken[key] = k + 1
            sr, sop = posted[key][k]
            if f & 1:      # direct: already in place
                msg = None
            elif f & 4:    # pulled: the sender's span now (its read buffer when it is a send)
                st, ss = sop["_pos"]
                msg = (rspan(sr, sop["src_buf"], sop["src_off"], cnt, st, ss, 1) if sop["opcode"] == "send"
                       else span(sr, sop["src_buf"], sop["src_off"], cnt)).copy()
            else:
                msg = fifo[key].pop(0)
        out = None
        if oc == "send":
            out = srcr.copy()
        elif oc == "recv":
            if msg is not None:
                dst[:] = msg
        elif oc == "copy":
            dst[:] = srcr
        elif oc == "reduce":
            dst[:] = dstr + srcr
        elif oc == "rrc":
            dst[:] = srcr + msg
        elif oc == "rcs":
            if msg is not None:
                src[:] = msg
            out = src.copy()
        elif oc == "rrcs":
            src[:] = srcr + msg
            out = src.copy()
        elif oc == "rrs":
            out = srcr + msg
        if oc in SENDS:
            key = (r, tb["send_peer"], tb["channel"])
            posted.setdefault(key, []).append((r, dict(op, _pos=(t, s))))
            if f & 2:      # direct: into the receiver's span named by this op's dst fields
                span(tb["send_peer"], op["dst_buf"], op["dst_off"], cnt)[:] = out
            elif not f & 8:
                fifo.setdefault(key, []).append(out)
        pc[(r, t)] += 1
    assert all(pc[(r, t)] == len(tb["ops"]) for r, t, tb in tbs), "deadlock"
    if result is not None:
        return [x.copy() for x in res]
    return [b[1].copy() for b in bufs]


NAMES = ["ring_ar_8_ch1", "ring_ar_4_ch4_inst4", "hier_ar_2x4_par1", "hier_ar_2x4_par2", "allpairs_ar_8", "ring_rs_8",
         "ring_ag_8", "twostep_a2a_2x4", "twostep_a2a_1x8", "ring_ar_8_inst4_auto", "hier_ar_2x4_par1.unfused",
         "ring_ar_8_ch8_inst1.unfused", "ring_ag_8@3", "twostep_a2a_1x8@3", "ring_ar_8_ch1@2", "ring_rs_4@2",
         "hier_ar_2x4_par1@1"]


def _load(spec):
    name, _, k = spec.partition("@")
    ir = gc3.IR(read_ir(name))
    if k and int(k) > 1:
        ir = ir.replicate(int(k))
    return json.loads(ir.serialize()), ir.direct_messages()


@pytest.mark.parametrize("name", NAMES)
def test_transports_match_fifo_semantics_under_random_interleavings(name):
    irj, flags = _load(name)
    ref = run(irj, flags, 0, use_flags=False)
    for seed in range(40):
        # the program itself is schedule-independent (FIFO transports only) ...
        if seed < 5:
            assert all(np.array_equal(a, b) for a, b in zip(ref, run(irj, flags, seed, use_flags=False)))
        got = run(irj, flags, seed)
        assert all(np.array_equal(a, b) for a, b in zip(ref, got)), f"seed {seed}"


def test_ring_allreduce_needs_no_fifo_except_after_rrs():
    """Ring AllReduce: broadcast receives are direct, reduce-phase messages are pulled; only the
    message an rrs sends (a value it never stores) still travels through a FIFO."""
    name = "ring_ar_8_ch1"
    irj = json.loads(read_ir(name))
    flags = gc3.IR(read_ir(name)).direct_messages()
    for r, g in enumerate(irj["gpus"]):
        for t, tb in enumerate(g["threadblocks"]):
            for s, op in enumerate(tb["ops"]):
                f = flags[r][t][s]
                if op["opcode"] in SENDS:
                    assert (f & 2) or (f & 8) or op["opcode"] == "rrs", (r, s, op["opcode"], f)
                if op["opcode"] in RECVS and not (f & 1) and not (f & 4):
                    # the FIFO receive must come from an rrs
                    assert op["opcode"] in ("rrcs", "rrc"), (r, s, op["opcode"], f)


def test_a_racy_pull_would_be_caught():
    """The checker is not vacuous: forcing a pull where the sender later overwrites its span
    before the receive may run changes the result in some interleaving."""
    text = json.dumps({
        "name": "racy", "collective": "custom", "protocol": "simple", "inplace": False,
        "nchunks": {"input": 1, "output": 1, "scratch": 0},
        "size_range": {"min_bytes": 0, "max_bytes": 1 << 40},
        "gpus": [
            {"rank": 0, "threadblocks": [
                {"id": 0, "send_peer": 1, "recv_peer": -1, "channel": 0, "ops": [
                    {"step": 0, "opcode": "send", "src_buf": "input", "src_off": 0, "dst_buf": "output", "dst_off": 0,
                     "count": 1, "deps": [], "has_dep": False},
                    {"step": 1, "opcode": "copy", "src_buf": "output", "src_off": 0, "dst_buf": "input", "dst_off": 0,
                     "count": 1, "deps": [], "has_dep": False}]}]},
            {"rank": 1, "threadblocks": [
                {"id": 0, "send_peer": -1, "recv_peer": 0, "channel": 0, "ops": [
                    {"step": 0, "opcode": "recv", "src_buf": "input", "src_off": 0, "dst_buf": "output", "dst_off": 0,
                     "count": 1, "deps": [], "has_dep": False}]}]}]})
    irj = json.loads(text)
    flags = gc3.IR(text).direct_messages()
    assert not flags[1][0][0] & 4, "the analysis must not pull: rank 0 overwrites the span after sending"
    forced = [[[8, 0]], [[4]]]
    ref = run(irj, flags, 0, use_flags=False)
    assert any(not np.array_equal(run(irj, forced, s)[1], ref[1]) for s in range(40))


@pytest.mark.parametrize("name", ["ring_ar_8_ch1", "ring_rs_8", "ring_rs_4@2", "hier_ar_2x4_par1", "allpairs_ar_8",
                                  "ring_ar_8_inst4_auto", "hier_ar_2x4_par1.unfused", "allpairs_ar_4.unfused",
                                  "ring_ar_4_ch4_inst4"])
def test_const_source_reads_need_no_precopy(name):
    """In-place AllReduce / ReduceScatter IRs read the caller's const buffer where no write comes
    first (runtime.cpp source_reads): with the working buffer left uninitialised, every
    interleaving (with the chosen transports) still gives the all-FIFO, pre-copied result."""
    spec, _, k = name.partition("@")
    ir = gc3.IR(read_ir(spec))
    if k:
        ir = ir.replicate(int(k))
    irj, flags = json.loads(ir.serialize()), ir.direct_messages()
    complete, source = ir.source_reads()
    assert complete, name
    assert any(x for g in source for tb in g for x in tb)
    ref = run(irj, flags, 0, use_flags=False)
    R = len(irj["gpus"])
    c = irj["nchunks"]["input"] // R
    for seed in range(30):
        got = run(irj, flags, seed, source=source)
        for r, (a, b) in enumerate(zip(ref, got)):
            if irj["collective"] == "reducescatter":  # only the owned block is the result
                a, b = a[r * c:(r + 1) * c], b[r * c:(r + 1) * c]
            assert np.array_equal(a, b), f"seed {seed} rank {r}"


@pytest.mark.parametrize("name", ["ring_rs_8", "ring_rs_4@2", "ring_rs_2"])
def test_reducescatter_final_writes_to_recvbuff(name):
    """ReduceScatter owned blocks written straight into recvbuff (runtime.cpp result_writes) with an
    uninitialised working buffer and the chosen transports: every interleaving leaves the reduced
    owned block in the result buffer."""
    spec, _, k = name.partition("@")
    ir = gc3.IR(read_ir(spec))
    if k:
        ir = ir.replicate(int(k))
    irj, flags = json.loads(ir.serialize()), ir.direct_messages()
    complete, source = ir.source_reads()
    rcomplete, result = ir.result_writes()
    assert complete and rcomplete
    ref = run(irj, flags, 0, use_flags=False)
    R = len(irj["gpus"])
    c = irj["nchunks"]["input"] // R
    for seed in range(30):
        got = run(irj, flags, seed, source=source, result=result)
        for r in range(R):
            assert np.array_equal(ref[r][r * c:(r + 1) * c], got[r][r * c:(r + 1) * c]), f"seed {seed} rank {r}"
