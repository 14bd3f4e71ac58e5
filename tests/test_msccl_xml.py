"""MSCCL-XML adapter (csrc/msccl_xml.cpp).

* GC3-IR -> MSCCL XML -> GC3-IR is the identity (byte-identical canonical JSON) on every golden IR.
* The XML is checked with Python's own xml.etree, independently of the C++ reader: one dependency
  per step, nop chains carrying the extra dependencies of multi-dependency ops, renumbered steps.
* With nop folding off, the nop-expanded program is a different but equivalent program: the CPU
  oracle gives identical outputs for both.
* Reader errors carry the element path.
"""
import json
import xml.etree.ElementTree as ET

import numpy as np
import pytest

from conftest import golden_names, ir_path, read_ir
from oracle.oracle import FlatIR

gc3 = pytest.importorskip("paper_2201_11840_b200.gc3")

TYPES = {"send": "s", "recv": "r", "copy": "cpy", "reduce": "re", "rrc": "rrc", "rcs": "rcs", "rrcs": "rrcs",
         "rrs": "rrs", "nop": "nop"}


@pytest.mark.parametrize("name", golden_names(include_unfused=True, include_ll=True))
def test_round_trip_is_identity(name):
    text = read_ir(name)
    ir = gc3.IR(text)
    back = gc3.IR.from_xml(ir.to_xml())
    assert back.serialize() == ir.serialize()


@pytest.mark.parametrize("name", ["twostep_a2a_2x4", "hier_ar_2x4_par1", "ring_ar_8_ch1", "ring_ag_4"])
def test_xml_structure_with_etree(name):
    irj = json.loads(read_ir(name))
    root = ET.fromstring(gc3.IR(read_ir(name)).to_xml())
    assert root.tag == "algo" and int(root.get("ngpus")) == len(irj["gpus"])
    assert root.get("coll") == {"reducescatter": "reduce_scatter"}.get(irj["collective"], irj["collective"])
    assert root.get("inplace") == ("1" if irj["inplace"] else "0")
    for g, ge in zip(irj["gpus"], root.findall("gpu")):
        assert int(ge.get("id")) == g["rank"]
        assert int(ge.get("i_chunks")) == irj["nchunks"]["input"]
        for tb, te in zip(g["threadblocks"], ge.findall("tb")):
            assert (int(te.get("send")), int(te.get("recv")), int(te.get("chan"))) == \
                (tb["send_peer"], tb["recv_peer"], tb["channel"])
            steps = te.findall("step")
            assert [int(s.get("s")) for s in steps] == list(range(len(steps)))
            real = [s for s in steps if not (s.get("type") == "nop" and s.get("hasdep") == "0")]
            assert len(real) == len(tb["ops"])
            nops = sum(max(len(o["deps"]) - 1, 0) for o in tb["ops"])
            assert len(steps) - len(real) == nops
            for o, s in zip(tb["ops"], real):
                assert s.get("type") == TYPES[o["opcode"]]
                assert int(s.get("cnt")) == o["count"] and int(s.get("srcoff")) == o["src_off"]
                assert s.get("srcbuf") == o["src_buf"][0] and s.get("dstbuf") == o["dst_buf"][0]
                assert (s.get("depid") == "-1") == (not o["deps"])
                if o["deps"]:
                    assert int(s.get("depid")) == o["deps"][-1]["tb"]


def _run_oracle(irj, seed=1, chunk=16):
    ir = FlatIR(irj)
    R, (nin, nout, nsc) = ir.nranks, ir.nchunks
    rng = np.random.default_rng(seed)
    bufs = []
    for r in range(R):
        inp = rng.integers(-2 ** 20, 2 ** 20, nin * chunk).astype(np.int32)
        out = inp if ir.inplace else np.zeros(max(nout, 1) * chunk, np.int32)
        bufs.append([inp, out, np.zeros(max(nsc, 1) * chunk, np.int32)])
    rc, err = ir.run(bufs, chunk, "int32", mode="random", seed=seed, slots=2, tile_elems=4)
    assert rc == 0, err
    return [b[1].copy() for b in bufs]


@pytest.mark.parametrize("name", ["twostep_a2a_2x4", "twostep_a2a_2x4.unfused"])
def test_nop_expanded_program_is_equivalent(name):
    ir = gc3.IR(read_ir(name))
    expanded = gc3.IR.from_xml(ir.to_xml(), fold_nops=False)
    ej = json.loads(expanded.serialize())
    n_nops = sum(o["opcode"] == "nop" for g in ej["gpus"] for t in g["threadblocks"] for o in t["ops"])
    assert n_nops > 0
    assert all(len(o["deps"]) <= 1 for g in ej["gpus"] for t in g["threadblocks"] for o in t["ops"])
    assert expanded.validate(2, 4) == []
    irj = json.loads(ir.serialize())
    for seed in range(3):
        a, b = _run_oracle(irj, seed), _run_oracle(ej, seed)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))


# A hand-written MSCCL-style file: 2-GPU all-pairs all-reduce where rank 0's final copy waits on two
# thread blocks through a nop (MSCCL's one-dependency-per-step encoding), with comments and a prolog.
HAND = """<?xml version="1.0"?>
<!-- two ranks, two chunks; each rank reduces the chunk it owns, then sends it back -->
<algo name="allpairs_2_hand" proto="Simple" nchannels="1" nchunksperloop="2" ngpus="2" coll="allreduce" inplace="1">
  <gpu id="0" i_chunks="2" o_chunks="0" s_chunks="0">
    <tb id="0" send="1" recv="1" chan="0">
      <step s="0" type="s" srcbuf="i" srcoff="1" dstbuf="i" dstoff="1" cnt="1" depid="-1" deps="-1" hasdep="0"/>
      <step s="1" type="rrc" srcbuf="i" srcoff="0" dstbuf="i" dstoff="0" cnt="1" depid="-1" deps="-1" hasdep="0"/>
      <step s="2" type="s" srcbuf="i" srcoff="0" dstbuf="i" dstoff="0" cnt="1" depid="-1" deps="-1" hasdep="0"/>
      <step s="3" type="r" srcbuf="i" srcoff="1" dstbuf="i" dstoff="1" cnt="1" depid="-1" deps="-1" hasdep="0"/>
    </tb>
  </gpu>
  <gpu id="1" i_chunks="2" o_chunks="0" s_chunks="0">
    <tb id="0" send="0" recv="0" chan="0">
      <step s="0" type="s" srcbuf="i" srcoff="0" dstbuf="i" dstoff="0" cnt="1" depid="-1" deps="-1" hasdep="0"/>
      <step s="1" type="rrc" srcbuf="i" srcoff="1" dstbuf="i" dstoff="1" cnt="1" depid="-1" deps="-1" hasdep="1"/>
      <step s="2" type="s" srcbuf="i" srcoff="1" dstbuf="i" dstoff="1" cnt="1" depid="-1" deps="-1" hasdep="0"/>
      <step s="3" type="r" srcbuf="i" srcoff="0" dstbuf="i" dstoff="0" cnt="1" depid="-1" deps="-1" hasdep="1"/>
    </tb>
    <tb id="1" send="-1" recv="-1" chan="0">
      <step s="0" type="nop" srcbuf="i" srcoff="-1" dstbuf="i" dstoff="-1" cnt="0" depid="0" deps="1" hasdep="0"/>
      <step s="1" type="nop" srcbuf="i" srcoff="-1" dstbuf="i" dstoff="-1" cnt="0" depid="0" deps="3" hasdep="0"/>
    </tb>
  </gpu>
</algo>
"""


def test_hand_written_msccl_file():
    ir = gc3.IR.from_xml(HAND)
    j = json.loads(ir.serialize())
    assert j["name"] == "allpairs_2_hand" and j["collective"] == "allreduce" and j["inplace"]
    assert j["nchunks"] == {"input": 2, "output": 2, "scratch": 0}  # in place: output aliases input
    tb1 = j["gpus"][1]["threadblocks"][1]["ops"]
    # the first nop folds into the second (the last step of a thread block is never folded); two
    # dependencies on one thread block keep the later step
    assert len(tb1) == 1 and tb1[0]["opcode"] == "nop" and tb1[0]["deps"] == [{"step": 3, "tb": 0}]
    assert ir.validate(1, 2) == []
    out = _run_oracle(j, chunk=8)
    ir0 = FlatIR(j)
    rng = np.random.default_rng(1)
    x = [rng.integers(-2 ** 20, 2 ** 20, 16).astype(np.int32) for _ in range(2)]
    assert np.array_equal(out[0], x[0] + x[1]) and np.array_equal(out[1], x[0] + x[1])
    assert ir0.nranks == 2


@pytest.mark.parametrize("text,needle", [
    ("<algo coll='allreduce'><gpu id='0'><tb id='0' send='-1' recv='-1' chan='0'></gpu></algo>", "closes"),
    ("<algo coll='allreduce'><gpu id='0'><tb id='0' send='-1' recv='-1'/></gpu></algo>", "algo.gpu[0].tb[0]: missing attribute 'chan'"),
    ("<algo coll='allreduce'><gpu id='0'><tb id='0' send='-1' recv='-1' chan='0'><step s='0' type='zz' srcbuf='i' "
     "srcoff='0' dstbuf='i' dstoff='0' cnt='1'/></tb></gpu></algo>", "unsupported step type \"zz\""),
    ("<algo coll='allreduce'><gpu id='0'><tb id='0' send='-1' recv='-1' chan='0'><step s='1' type='cpy' srcbuf='i' "
     "srcoff='0' dstbuf='i' dstoff='0' cnt='1'/></tb></gpu></algo>", "algo.gpu[0].tb[0].step[0]: step index 1"),
    ("<algo coll='allreduce'><gpu id='0'><tb id='0' send='-1' recv='-1' chan='0'><step s='0' type='cpy' srcbuf='q' "
     "srcoff='0' dstbuf='i' dstoff='0' cnt='1'/></tb></gpu></algo>", "unknown buffer \"q\""),
    ("<algo coll='broadcastish'><gpu id='0'/></algo>", "unknown collective"),
    ("<algo coll='allreduce'><gpu id='0'/><gpu id='0'/></algo>", "repeated gpu id"),
    ("<algo coll='allreduce' ngpus='2'><gpu id='0'/></algo>", "ngpus=2"),
    ("<notalgo/>", "expected <algo>"),
    ("<algo coll='allreduce'><gpu id='x'/></algo>", "not an integer"),
    ("<algo coll='allreduce' name='a &bogus; b'><gpu id='0'/></algo>", "unknown entity"),
])
def test_reader_errors(text, needle):
    with pytest.raises(gc3.NcclError) as e:
        gc3.IR.from_xml(text)
    assert needle in str(e.value)
