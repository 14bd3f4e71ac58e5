"""Race detection of the functional simulator (oracle gc3o_races; vector
clocks over block steps, comm edges and semaphore edges, conflicts at (rank, buffer, index) slot
granularity).  SPEC's examples: compiled programs are race-free; a hand-built IR writing one slot
from two unordered blocks reports the pair."""
import json

import pytest

from conftest import golden_names, ir_path
from oracle.oracle import FlatIR


def _op(step, opcode, sb, so, db, do, deps=(), count=1):
    return {"step": step, "opcode": opcode, "src_buf": sb, "src_off": so, "dst_buf": db, "dst_off": do, "count": count,
            "has_dep": False, "deps": [{"tb": t, "step": s} for t, s in deps]}


def _ir(gpus, nchunks=(2, 2, 0), inplace=False):
    return {"name": "hand", "collective": "custom", "protocol": "simple", "inplace": inplace,
            "nchunks": {"input": nchunks[0], "output": nchunks[1], "scratch": nchunks[2]},
            "size_range": {"min_bytes": 0, "max_bytes": 1 << 40},
            "gpus": [{"rank": r, "threadblocks": tbs} for r, tbs in enumerate(gpus)]}


def _tb(i, ops, send=-1, recv=-1, ch=0):
    return {"id": i, "send_peer": send, "recv_peer": recv, "channel": ch, "ops": ops}


@pytest.mark.parametrize("name", golden_names(include_unfused=True, include_ll=True))
def test_compiled_programs_are_race_free(name):
    assert FlatIR(json.load(open(ir_path(name)))).races() == []


def test_two_unordered_writers_of_one_slot_race():
    ir = _ir([[_tb(0, [_op(0, "copy", "input", 0, "output", 0)]), _tb(1, [_op(0, "copy", "input", 1, "output", 0)])]])
    races = FlatIR(ir).races()
    assert len(races) == 1
    r = races[0]
    assert (r["rank"], r["buf"], r["index"], r["kind"]) == (0, "output", 0, "write/write")
    assert {r["a"], r["b"]} == {(0, 0), (1, 0)}


def test_a_dep_orders_the_writers():
    ir = _ir([[_tb(0, [_op(0, "copy", "input", 0, "output", 0)]),
               _tb(1, [_op(0, "copy", "input", 1, "output", 0, deps=[(0, 0)])])]])
    assert FlatIR(ir).races() == []


def test_read_write_race_and_in_place_aliasing():
    # tb0 reads input 0 (send), tb1 overwrites output 0 == input 0 (in place): unordered
    ir = _ir([[_tb(0, [_op(0, "send", "input", 0, "input", 0)], send=1),
               _tb(1, [_op(0, "copy", "input", 1, "output", 0)])],
              [_tb(0, [_op(0, "recv", "input", 0, "input", 0)], recv=0)]], inplace=True)
    races = FlatIR(ir).races()
    assert [(r["rank"], r["buf"], r["index"], r["kind"]) for r in races] == [(0, "input", 0, "read/write")]
    ir["inplace"] = False  # out of place: output 0 is a different slot
    assert FlatIR(ir).races() == []


def test_message_edge_orders_accesses_across_thread_blocks():
    # rank 1: tb0 receives into output 0, then sends it back; tb1 copies output 0 after its own
    # receive of rank 0's second message, which rank 0 sends only after receiving the echo: ordered
    # through two message edges and rank 0's program order
    ir = _ir([[_tb(0, [_op(0, "send", "input", 0, "output", 0), _op(1, "recv", "input", 0, "output", 1),
                       _op(2, "send", "input", 1, "output", 1)], send=1, recv=1)],
              [_tb(0, [_op(0, "recv", "input", 0, "output", 0), _op(1, "send", "output", 0, "output", 1)], send=0, recv=0),
               _tb(1, [_op(0, "recv", "input", 0, "input", 1), _op(1, "copy", "input", 1, "output", 0)], recv=0, ch=1)]])
    # the second message travels on channel 0 as well (rank 0 has one tb): re-route tb1's receive
    ir["gpus"][0]["threadblocks"].append(_tb(1, [_op(0, "send", "input", 1, "input", 1, deps=[(0, 1)])], send=1, ch=1))
    ir["gpus"][0]["threadblocks"][0]["ops"].pop()
    assert FlatIR(ir).races() == []
    # without the dep on the echo the copy can overwrite output 0 before rank 1's send reads it
    ir["gpus"][0]["threadblocks"][1]["ops"][0]["deps"] = []
    races = FlatIR(ir).races()
    assert {(r["rank"], r["buf"], r["index"]) for r in races} == {(1, "output", 0)}


def test_deadlocking_program_is_an_error():
    ir = _ir([[_tb(0, [_op(0, "copy", "input", 0, "output", 0, deps=[(1, 0)])]),
               _tb(1, [_op(0, "copy", "input", 1, "output", 1, deps=[(0, 0)])])]])
    with pytest.raises(ValueError, match="deadlock"):
        FlatIR(ir).races()
