"""The C-ABI boundary: libgc3.so loads without a GPU and exports every entry point include/gc3.h
declares (no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import REPO, read_ir


def declared_functions():
    text = open(os.path.join(REPO, "include", "gc3.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\s*\*?\s+((?:nccl|gc3)\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_nccl_subset():
    names = declared_functions()
    for f in ["ncclGetVersion", "ncclGetUniqueId", "ncclCommInitRank", "ncclCommInitAll", "ncclCommDestroy",
              "ncclCommAbort", "ncclGetErrorString", "ncclGetLastError", "ncclCommGetAsyncError", "ncclCommCount",
              "ncclCommCuDevice", "ncclCommUserRank", "ncclAllReduce", "ncclReduceScatter", "ncclAllGather",
              "ncclAlltoAll", "ncclAllToAll", "ncclGroupStart", "ncclGroupEnd", "gc3RegisterIR",
              "gc3SetProtocolOverride", "gc3QueryPlan", "gc3SetConfig", "gc3IrParse", "gc3IrSerialize",
              "gc3IrValidate", "gc3IrCheckSlots", "gc3IrReplicate", "gc3IrFree"]:
        assert f in names, f


def test_library_exports_every_declared_symbol(gc3lib):
    out = subprocess.run(["nm", "-D", "--defined-only", gc3lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (\w+)$", out, flags=re.M))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    # nothing else leaks: internal symbols are hidden (-fvisibility=hidden)
    leaked = [s for s in exported if not s.startswith(("nccl", "gc3"))]
    assert not leaked, leaked[:10]


def test_version_and_error_strings(gc3lib):
    L = gc3lib.lib()
    v = ctypes.c_int()
    assert L.ncclGetVersion(ctypes.byref(v)) == 0 and v.value == 22809
    assert L.ncclGetErrorString(0) == b"no error"
    assert b"invalid argument" in L.ncclGetErrorString(4)
    assert L.ncclGetErrorString(99) == b"unknown result code"


def test_unique_ids_are_distinct(gc3lib):
    a, b = gc3lib.get_unique_id(), gc3lib.get_unique_id()
    assert a[:4] == b"GC3\0" and a != b and len(a) == 128


def test_invalid_arguments_return_errors(gc3lib):
    L = gc3lib.lib()
    assert L.ncclCommCount(None, None) == 4
    assert L.ncclGroupEnd() == 5  # without ncclGroupStart
    assert L.ncclAllReduce(None, None, 1, 7, 0, None, None) == 4


def test_bootstrap_single_rank(gc3lib):
    uid = gc3lib.get_unique_id()
    assert gc3lib.bootstrap_exchange(uid, 0, 1, b"hello") == [b"hello"]


def test_arena_layout_shapes(gc3lib):
    ir = gc3lib.IR(read_ir("twostep_a2a_2x4"))
    lay = ir.arena_layout(0, 4, 2, 1 << 16)
    # rank 0 receives on 4 thread blocks; the coalesced connection carries count-4 messages
    assert lay["n_in"] == 4 and sorted(lay["slot_stride"]) == [1 << 16] * 3 + [4 << 16]
    assert lay["fifo_off"][0] == 0 and lay["bytes"] % 256 == 0


def test_direct_message_analysis(gc3lib):
    """AllToAll / AllGather receives land in spans no earlier op touches: all direct. Ring
    AllReduce / ReduceScatter reducing receives combine with a live span: never direct; the
    AllReduce broadcast receives (rcs / recv) overwrite spans whose earlier uses all happen before
    the matching send: direct."""
    import json
    for name, direct_ops in [("twostep_a2a_1x8", {"recv"}), ("ring_ag_8", {"recv", "rcs"}),
                             ("ring_ar_8_ch1", {"recv", "rcs"}), ("ring_rs_8", set()),
                             ("hier_ar_2x4_par1", {"recv", "rcs"})]:
        irj = json.loads(read_ir(name))
        flags = gc3lib.IR(read_ir(name)).direct_messages()
        recvs = [(r, t, s, o["opcode"]) for r, g in enumerate(irj["gpus"]) for t, tb in enumerate(g["threadblocks"])
                 for s, o in enumerate(tb["ops"]) if o["opcode"] in ("recv", "rcs", "rrc", "rrcs", "rrs")]
        for r, t, s, op in recvs:
            assert bool(flags[r][t][s] & 1) == (op in direct_ops), (name, r, t, s, op)
    # two-step: the scratch staging recv is direct, and so is the final coalesced receive
    f = gc3lib.IR(read_ir("twostep_a2a_2x4")).direct_messages()
    assert sum(x & 1 for g in f for tb in g for x in tb) == 56
