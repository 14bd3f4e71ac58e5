"""GPU parity of the line protocols: LL (16-byte lines, 8 payload bytes) and
LL128 (128-byte lines of 15 payload words + a 64-bit flag), bit for bit against the CPU oracle, and
the protocol hygiene of the FIFOs: every protocol has its own slots, so one connection can carry
Simple, LL and LL128 messages in any order (including payloads that look like flags)."""
import json

import numpy as np
import pytest

from conftest import read_ir
from test_gpu_parity import _check, _setup

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,count", [
    ("ring_ar_8_ch1", 8 * 4096), ("ring_ar_8_ch1", 8 * 15 * 37), ("ring_ar_8_ch8_inst4", 32 * 4096),
    ("ring_ar_8_inst4_auto", 32 * 1000), ("hier_ar_2x4_par1", 8 * 4096), ("hier_ar_2x4_par2", 16 * 512),
    ("allpairs_ar_8", 8 * 778), ("ring_ar_4_ch1", 4 * 3000), ("ring_ar_2_ch1", 2 * 64),
    ("ring_ar_8_ch8_inst1.unfused", 8 * 1024), ("ring_ag_8", 4096), ("ring_rs_8", 4096), ("ring_rs_4", 1000),
    ("twostep_a2a_2x4", 2048), ("twostep_a2a_1x8", 1000),
])
def test_ll128_families(name, count):
    _check(name, count, proto="ll128")


@pytest.mark.parametrize("dtype,op", [("bfloat16", "sum"), ("float16", "sum"), ("int32", "sum"), ("float64", "sum"),
                                      ("int64", "prod"), ("float32", "max"), ("bfloat16", "min"), ("uint8", "sum"),
                                      ("int8", "max"), ("uint32", "prod")])
def test_ll128_dtypes(dtype, op):
    _check("hier_ar_2x4_par1", 8 * 2048, dtype, op, proto="ll128")


@pytest.mark.parametrize("lanes,tile_bytes", [(1, 0), (3, 0), (16, 0), (4, 1040), (7, 120), (2, 8), (5, 968)])
def test_ll128_lanes_and_tiles(lanes, tile_bytes):
    """Tiles that end inside a line (ragged last line of a segment), one-word tiles, many lanes."""
    _check("hier_ar_2x4_par1", 8 * 5000, proto="ll128", lanes=lanes, tile_bytes=tile_bytes)
    _check("ring_ar_8_ch1", 8 * 4000, proto="ll128", lanes=lanes, tile_bytes=tile_bytes)
    _check("twostep_a2a_2x4", 3000, proto="ll128", lanes=lanes, tile_bytes=tile_bytes)


@pytest.mark.parametrize("name,count,dtype", [("ring_ar_8_ch1", 8 * 1000 + 2, "float32"), ("hier_ar_2x4_par1", 8 * 4096 + 4, "bfloat16"),
                                              ("ring_rs_8", 778, "float32"), ("twostep_a2a_1x8", 1002, "float32")])
def test_ll128_ragged_counts(name, count, dtype):
    _check(name, count, dtype, proto="ll128")


def test_ll128_larger_messages():
    """Multi-tile messages through full slots (several lines per thread group in flight)."""
    _check("ring_ar_8_ch1", 8 * (1 << 18), proto="ll128")
    _check("ring_ar_8_ch8_inst4", 32 * (1 << 15), proto="ll128", dtype="bfloat16")


def test_protocols_interleaved_on_one_connection():
    """One communicator, one IR, the protocol switched between launches (Simple -> LL -> LL128 ->
    Simple ...) with adversarial payloads: int32 data equal to the message sequence numbers the line
    protocols use as flags. A slot shared between protocols would let a line receiver accept a stale
    Simple payload as a posted line; per-protocol slots make every launch bit-exact."""
    from gpu_util import oracle_collective, run_collective, to_np_bits
    comms, irj = _setup("ring_ar_8_ch1", lanes=1)
    try:
        R = 8
        for it, proto in enumerate(["simple", "ll", "ll128", "simple", "ll128", "ll", "simple", "ll", "ll128"] * 2):
            for c in comms:
                c.set_protocol(0, proto)
            count = 8 * (256 + 64 * (it % 5))
            # every value a small counter: in the range of the FIFO sequence numbers
            inputs = [torch.full((count,), it + 1, dtype=torch.int32, device="cuda") + (torch.arange(count, device="cuda", dtype=torch.int32) % 7)
                      for r in range(R)]
            expected = oracle_collective(irj, "allreduce", [x.clone() for x in inputs], count, "int32")
            outs = run_collective(comms, "allreduce", inputs, count, "int32")
            torch.cuda.synchronize()
            assert comms[0].async_error()[0] == 0
            for r in range(R):
                assert np.array_equal(to_np_bits(outs[r], "int32"), expected[r]), (it, proto, r)
    finally:
        for c in comms:
            c.destroy()


def test_size_based_protocol_choice():
    """ll_max_bytes / ll128_max_bytes: a Simple IR runs LL up to the first threshold, LL128 up to the
    second and Simple above; all bit-exact."""
    comms, irj = _setup("ring_ar_8_ch8_inst4", ll_max_bytes=64 << 10, ll128_max_bytes=4 << 20)
    try:
        assert comms[0].query_plan("allreduce", 32 * 256, "float32")["protocol"] == 1     # 32 KiB per rank
        assert comms[0].query_plan("allreduce", 32 * 8192, "float32")["protocol"] == 2    # 1 MiB per rank
        assert comms[0].query_plan("allreduce", 32 * 65536, "float32")["protocol"] == 0   # 8 MiB per rank
    finally:
        for c in comms:
            c.destroy()
    for count in (32 * 256, 32 * 8192, 32 * 65536):
        _check("ring_ar_8_ch8_inst4", count, ll_max_bytes=64 << 10, ll128_max_bytes=4 << 20)


def test_ll128_fifo_only_and_instances():
    _check("twostep_a2a_2x4", 2048, proto="ll128", direct=0)
    _check("ring_ar_8_ch8_inst1", 32 * 512, instances=4, proto="ll128")


def test_ll128_tagged_ir():
    """An IR whose protocol tag is ll128 runs LL128 without an override (ir.hpp:21-66)."""
    from paper_2201_11840_b200 import gc3
    from gpu_util import make_input, oracle_collective, run_collective, to_np_bits
    irj = json.loads(read_ir("ring_ar_8_ch1"))
    irj["protocol"] = "ll128"
    irj["name"] = "ring_ar_8_ch1_ll128"
    comms = gc3.init_all([0] * 8)
    try:
        for c in comms:
            c.register_ir(json.dumps(irj))
        count = 8 * 3000
        assert comms[0].query_plan("allreduce", count, "float32")["protocol"] == 2
        inputs = [make_input(count, "float32", 90 + r) for r in range(8)]
        expected = oracle_collective(irj, "allreduce", [x.clone() for x in inputs], count, "float32")
        outs = run_collective(comms, "allreduce", inputs, count, "float32")
        torch.cuda.synchronize()
        assert comms[0].async_error()[0] == 0
        for r in range(8):
            assert np.array_equal(to_np_bits(outs[r], "float32"), expected[r])
    finally:
        for c in comms:
            c.destroy()
