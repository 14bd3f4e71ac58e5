"""IR loader / writer / validator / slot-check parity with the reference (ir.hpp, scheduler.hpp).

Product side: libgc3.so gc3Ir* (paper_2201_11840_b200/csrc/ir.cpp).  Reference side:
oracle/_ref/libref.so (the reference headers compiled by oracle/ref_harness) where available,
plus the exact strings recorded in SURVEY.md Appendix C so the tests also pin behaviour without it.
"""
import copy
import json

import pytest

from conftest import golden_names, read_ir


def mutate(fn, base="ring_rs_2"):
    d = json.loads(read_ir(base))
    fn(d)
    return json.dumps(d, indent=2, sort_keys=True)


def op0(d, g=0, t=0, o=0):
    return d["gpus"][g]["threadblocks"][t]["ops"][o]


# (name, mutation, expected path, expected message) — Appendix C of SURVEY.md and more
SCHEMA_MUTATIONS = [
    ("missing channel", lambda d: d["gpus"][0]["threadblocks"][0].pop("channel"), "gpus[0].threadblocks[0].channel", "missing required key"),
    ("count string", lambda d: op0(d).__setitem__("count", "1"), "gpus[0].threadblocks[0].ops[0].count", "expected an integer"),
    ("count float", lambda d: op0(d).__setitem__("count", 1.5), "gpus[0].threadblocks[0].ops[0].count", "expected an integer"),
    ("count 1.0", lambda d: op0(d).__setitem__("count", 1.0), "gpus[0].threadblocks[0].ops[0].count", "expected an integer"),
    ("count 2^70", lambda d: op0(d).__setitem__("count", 2 ** 70), "gpus[0].threadblocks[0].ops[0].count", "expected an integer"),
    ("bad opcode", lambda d: op0(d).__setitem__("opcode", "rrsc"), "gpus[0].threadblocks[0].ops[0].opcode", "unknown opcode"),
    ("opcode int", lambda d: op0(d).__setitem__("opcode", 3), "gpus[0].threadblocks[0].ops[0].opcode", "expected a string"),
    ("extra gpu key", lambda d: d["gpus"][1].__setitem__("extra", 1), "gpus[1].extra", "unknown key"),
    ("protocol case", lambda d: d.__setitem__("protocol", "LL"), "protocol", 'expected one of "simple", "ll", "ll128"'),
    ("collective", lambda d: d.__setitem__("collective", "broadcast"), "collective", 'unknown collective "broadcast"'),
    ("max_bytes -1", lambda d: d["size_range"].__setitem__("max_bytes", -1), "size_range.max_bytes", "expected a non-negative integer"),
    ("min_bytes float", lambda d: d["size_range"].__setitem__("min_bytes", 1.0), "size_range.min_bytes", "expected an integer"),
    ("src_buf", lambda d: op0(d).__setitem__("src_buf", "in"), "gpus[0].threadblocks[0].ops[0].src_buf", 'expected one of "input", "output", "scratch"'),
    ("dst_buf int", lambda d: op0(d).__setitem__("dst_buf", 0), "gpus[0].threadblocks[0].ops[0].dst_buf", "expected a string"),
    ("dep without step", lambda d: op0(d).__setitem__("deps", [{"tb": 0}]), "gpus[0].threadblocks[0].ops[0].deps[0].step", "missing required key"),
    ("dep tb string", lambda d: op0(d).__setitem__("deps", [{"tb": "0", "step": 0}]), "gpus[0].threadblocks[0].ops[0].deps[0].tb", "expected an integer"),
    ("dep extra key", lambda d: op0(d).__setitem__("deps", [{"tb": 0, "step": 0, "x": 1}]), "gpus[0].threadblocks[0].ops[0].deps[0].x", "unknown key"),
    ("inplace int", lambda d: d.__setitem__("inplace", 1), "inplace", "expected a boolean"),
    ("has_dep string", lambda d: op0(d).__setitem__("has_dep", "false"), "gpus[0].threadblocks[0].ops[0].has_dep", "expected a boolean"),
    ("gpus object", lambda d: d.__setitem__("gpus", {}), "gpus", "expected an array"),
    ("threadblocks object", lambda d: d["gpus"][0].__setitem__("threadblocks", {}), "gpus[0].threadblocks", "expected an array"),
    ("ops scalar", lambda d: d["gpus"][0]["threadblocks"][0].__setitem__("ops", 3), "gpus[0].threadblocks[0].ops", "expected an array"),
    ("op scalar", lambda d: d["gpus"][0]["threadblocks"][0]["ops"].__setitem__(0, 5), "gpus[0].threadblocks[0].ops[0]", "expected an object"),
    ("deps object", lambda d: op0(d).__setitem__("deps", {}), "gpus[0].threadblocks[0].ops[0].deps", "expected an array"),
    ("name int", lambda d: d.__setitem__("name", 5), "name", "expected a string"),
    ("missing name+gpus", lambda d: (d.pop("name"), d.pop("gpus")), "name", "missing required key"),
    ("missing scratch", lambda d: d["nchunks"].pop("scratch"), "nchunks.scratch", "missing required key"),
    ("nchunks string", lambda d: d["nchunks"].__setitem__("input", "2"), "nchunks.input", "expected an integer"),
    ("nchunks array", lambda d: d.__setitem__("nchunks", [1, 2]), "nchunks", "expected an object"),
    ("rank string", lambda d: d["gpus"][0].__setitem__("rank", "0"), "gpus[0].rank", "expected an integer"),
    ("unknown top keys sorted", lambda d: (d.__setitem__("zzz", 1), d.__setitem__("aaa", 1)), "aaa", "unknown key"),
    ("missing before unknown", lambda d: (d.__setitem__("aaa", 1), d.pop("protocol")), "protocol", "missing required key"),
    ("send_peer null", lambda d: d["gpus"][0]["threadblocks"][0].__setitem__("send_peer", None), "gpus[0].threadblocks[0].send_peer", "expected an integer"),
]


@pytest.mark.parametrize("case", SCHEMA_MUTATIONS, ids=[c[0] for c in SCHEMA_MUTATIONS])
def test_schema_mutation(gc3lib, case):
    _, fn, path, msg = case
    text = mutate(fn)
    with pytest.raises(gc3lib.NcclError) as e:
        gc3lib.IR(text)
    assert (e.value.path, e.value.message) == (path, msg)


@pytest.mark.parametrize("case", SCHEMA_MUTATIONS, ids=[c[0] for c in SCHEMA_MUTATIONS])
def test_schema_mutation_matches_reference(gc3lib, reflib, case):
    text = mutate(case[1])
    ref = reflib.load(text, 1, 2)["schema_error"]
    with pytest.raises(gc3lib.NcclError) as e:
        gc3lib.IR(text)
    assert ref is not None
    assert ref["path"] == e.value.path
    assert ref["what"] == f"schema: {e.value.path}: {e.value.message}"


@pytest.mark.parametrize("text", ["{not json", "", "[1,2", '{"a": 1,}', "nul", '{"name": "x"} trailing', "01"])
def test_invalid_json(gc3lib, text):
    with pytest.raises(gc3lib.NcclError) as e:
        gc3lib.IR(text)
    assert e.value.path == ""
    assert e.value.message.startswith("invalid JSON: ")


def test_top_level_not_object(gc3lib):
    with pytest.raises(gc3lib.NcclError) as e:
        gc3lib.IR("[1, 2]")
    assert (e.value.path, e.value.message) == ("", "expected an object")


def test_duplicate_key_last_wins(gc3lib, reflib):
    text = read_ir("ring_rs_2").replace('"protocol": "simple"', '"protocol": "ll", "protocol": "simple"')
    assert gc3lib.IR(text).serialize() == reflib.load(text, 1, 2)["canonical"]


@pytest.mark.parametrize("name", golden_names(include_unfused=True, include_ll=True))
def test_roundtrip_byte_identical(gc3lib, name):
    text = read_ir(name)
    assert gc3lib.IR(text).serialize() == text  # canonical bytes (ir.hpp:185)


@pytest.mark.parametrize("name", golden_names(include_unfused=True))
def test_golden_validate_clean(gc3lib, name):
    d = json.loads(read_ir(name))
    nodes, gpn = topo_of(name, len(d["gpus"]))
    assert gc3lib.IR(read_ir(name)).validate(nodes, gpn) == []


def topo_of(name, ranks):
    import re
    m = re.search(r"_(\d+)x(\d+)", name)
    if m:
        return int(m.group(1)), int(m.group(2))
    return 1, ranks


def vmut(fn, base="ring_rs_2"):
    return mutate(fn, base)


def _dup_tb(d):
    d["gpus"][0]["threadblocks"].append(copy.deepcopy(d["gpus"][0]["threadblocks"][0]))


VALIDATE_MUTATIONS = [
    ("dep nonexistent tb", lambda d: op0(d).__setitem__("deps", [{"tb": 5, "step": 0}]), ["gpu 0 tb 0 step 0: dependency on nonexistent tb 5"]),
    ("src span", lambda d: op0(d).__setitem__("src_off", 5), ["gpu 0 tb 0 step 0: src span exceeds input extent"]),
    ("unbalanced", lambda d: op0(d).__setitem__("count", 2), None),
    ("self dep", lambda d: op0(d).__setitem__("deps", [{"tb": 0, "step": 1}]), None),
    ("dup deps", lambda d: op0(d, o=1).__setitem__("deps", [{"tb": 1, "step": 0}, {"tb": 1, "step": 0}]), None),
    ("dup tb", _dup_tb, None),
    ("channel budget", lambda d: d["gpus"][0]["threadblocks"][0].__setitem__("channel", 40), None),
    ("invalid peer", lambda d: d["gpus"][0]["threadblocks"][0].__setitem__("send_peer", 0), None),
    ("peer out of range", lambda d: d["gpus"][0]["threadblocks"][0].__setitem__("recv_peer", 7), None),
    ("step field", lambda d: op0(d).__setitem__("step", 3), None),
    ("count zero", lambda d: op0(d).__setitem__("count", 0), None),
    ("rank field", lambda d: d["gpus"][1].__setitem__("rank", 0), None),
    ("inplace mismatch", lambda d: d["nchunks"].__setitem__("output", 3), None),
    ("negative chunks", lambda d: d["nchunks"].__setitem__("scratch", -1), None),
    ("send without peer", lambda d: d["gpus"][0]["threadblocks"][0].__setitem__("send_peer", -1), None),
    ("dst span scratch", lambda d: op0(d).__setitem__("dst_buf", "scratch"), None),
    ("dep lacks has_dep", lambda d: (d["gpus"][0]["threadblocks"].append(
        {"id": 1, "send_peer": -1, "recv_peer": -1, "channel": 0,
         "ops": [dict(op0(d), step=0, opcode="copy", deps=[{"tb": 0, "step": 1}], has_dep=False)]})), None),
]


@pytest.mark.parametrize("case", VALIDATE_MUTATIONS, ids=[c[0] for c in VALIDATE_MUTATIONS])
def test_validate_mutation(gc3lib, case):
    _, fn, expected = case
    issues = gc3lib.IR(vmut(fn)).validate(1, 2)
    assert issues, "mutation must be reported"
    if expected is not None:
        assert issues[: len(expected)] == expected


@pytest.mark.parametrize("case", VALIDATE_MUTATIONS, ids=[c[0] for c in VALIDATE_MUTATIONS])
def test_validate_mutation_matches_reference(gc3lib, reflib, case):
    text = vmut(case[1])
    assert gc3lib.IR(text).validate(1, 2) == reflib.load(text, 1, 2)["issues"]


def test_validate_unbalanced_message(gc3lib):
    text = vmut(lambda d: op0(d).__setitem__("count", 2))
    assert "connection 0->1 ch 0 is unbalanced: 1 sends vs 1 receives (or counts differ)" in gc3lib.IR(text).validate(1, 2)


def test_validate_topology_budgets(gc3lib, reflib):
    text = read_ir("ring_ar_8_ch8_inst4")
    for args in [(1, 4, 0, 0), (1, 8, 16, 0), (1, 8, 0, 8), (2, 4, 31, 31)]:
        assert gc3lib.IR(text).validate(*args) == reflib.load(text, *args)["issues"]


@pytest.mark.parametrize("name", golden_names(include_unfused=True))
@pytest.mark.parametrize("slots", [1, 2])
def test_check_slots_matches_reference(gc3lib, reflib, name, slots):
    text = read_ir(name)
    assert gc3lib.IR(text).check_slots(slots) == reflib.check_slots(text, slots)


def test_check_slots_flags_pathological(gc3lib, reflib):
    # receiver consumes only after the sender's second send depends on it -> needs 2 slots
    ir = {
        "name": "patho", "collective": "custom", "protocol": "simple", "inplace": False,
        "nchunks": {"input": 2, "output": 2, "scratch": 0},
        "size_range": {"min_bytes": 0, "max_bytes": 1 << 40},
        "gpus": [
            {"rank": 0, "threadblocks": [{"id": 0, "send_peer": 1, "recv_peer": 1, "channel": 0, "ops": [
                {"step": 0, "opcode": "send", "src_buf": "input", "src_off": 0, "dst_buf": "output", "dst_off": 0, "count": 1, "deps": [], "has_dep": False},
                {"step": 1, "opcode": "send", "src_buf": "input", "src_off": 1, "dst_buf": "output", "dst_off": 1, "count": 1, "deps": [], "has_dep": False},
                {"step": 2, "opcode": "recv", "src_buf": "input", "src_off": 0, "dst_buf": "output", "dst_off": 0, "count": 1, "deps": [], "has_dep": False}]}]},
            {"rank": 1, "threadblocks": [{"id": 0, "send_peer": 0, "recv_peer": 0, "channel": 0, "ops": [
                {"step": 0, "opcode": "send", "src_buf": "input", "src_off": 0, "dst_buf": "output", "dst_off": 0, "count": 1, "deps": [], "has_dep": False},
                {"step": 1, "opcode": "recv", "src_buf": "input", "src_off": 0, "dst_buf": "output", "dst_off": 0, "count": 1, "deps": [], "has_dep": False},
                {"step": 2, "opcode": "recv", "src_buf": "input", "src_off": 1, "dst_buf": "output", "dst_off": 1, "count": 1, "deps": [], "has_dep": False}]}]},
        ],
    }
    text = json.dumps(ir)
    ours = gc3lib.IR(text).check_slots(1)
    assert ours == reflib.check_slots(text, 1)


@pytest.mark.parametrize("base,k,target", [
    ("ring_ar_8_ch8_inst1", 4, "ring_ar_8_ch8_inst4"),
    ("ring_ar_4_ch4_inst1", 4, "ring_ar_4_ch4_inst4"),
    ("ring_ar_2_ch2_inst1", 4, "ring_ar_2_ch2_inst4"),
])
def test_instances_rewrite_equals_compile_time_parallelize(gc3lib, base, k, target):
    """SURVEY.md Finding 5: the runtime `instances` rewrite reproduces parallelize(k) exactly."""
    ours = json.loads(gc3lib.IR(read_ir(base)).replicate(k).serialize())
    ref = json.loads(read_ir(target))
    ours.pop("name"), ref.pop("name")
    assert ours == ref


def test_instances_rewrite_rejects_mixed_counts(gc3lib):
    """The rewrite is only defined for ops of one count: on the two-step AllToAll (count-1 and
    coalesced count-4 ops on the same scratch chunks) it would make unordered ops share spans."""
    with pytest.raises(gc3lib.NcclError):
        gc3lib.IR(read_ir("twostep_a2a_2x4")).replicate(2)
    assert gc3lib.IR(read_ir("twostep_a2a_1x8")).replicate(2).validate(1, 8) == []
