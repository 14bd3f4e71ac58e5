"""Full-size checks at BASELINE.json's sizes through size-independent properties (the oracle is
too slow at 8 x 64 MiB): AllToAll / AllGather are exact permutations of the inputs; AllReduce /
ReduceScatter of integer data (wrapping sum: association-free) equal the torch sum exactly."""
import json

import pytest

from conftest import ir_path, read_ir

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _comms(name, **cfg):
    from paper_2201_11840_b200 import gc3
    R = len(json.loads(read_ir(name))["gpus"])
    comms = gc3.init_all([0] * R)
    for c in comms:
        for k, v in cfg.items():
            c.set_config(k, v)
        c.register_ir(ir_path(name))
    return comms


@pytest.mark.parametrize("name", ["twostep_a2a_2x4", "twostep_a2a_1x8"])
@pytest.mark.parametrize("tma", [1, 0])
def test_alltoall_64MiB_is_the_transposition(name, tma):
    from paper_2201_11840_b200 import gc3
    comms = _comms(name, tma=tma)
    R, count = 8, (64 << 20) // 4 // 8
    try:
        g = torch.Generator(device="cuda").manual_seed(1)
        ins = [torch.randint(-2 ** 31, 2 ** 31 - 1, (R * count,), device="cuda", dtype=torch.int32, generator=g) for _ in range(R)]
        outs = [torch.empty_like(x) for x in ins]
        for _ in range(2):  # twice: persistent FIFO counters and epochs across launches
            with gc3.group():
                for c, x, y in zip(comms, ins, outs):
                    c.all_to_all(x, y, count, "float32")
            torch.cuda.synchronize()
            assert comms[0].async_error()[0] == 0
            for d in range(R):
                for s in range(R):
                    assert torch.equal(outs[d][s * count:(s + 1) * count], ins[s][d * count:(d + 1) * count]), (d, s)
            for y in outs:
                y.zero_()
    finally:
        for c in comms:
            c.destroy()


def test_allgather_64MiB_is_the_concatenation():
    from paper_2201_11840_b200 import gc3
    comms = _comms("ring_ag_8")
    R, count = 8, (64 << 20) // 4 // 8
    try:
        ins = [torch.full((count,), r + 1, device="cuda", dtype=torch.int32) * torch.arange(count, device="cuda", dtype=torch.int32)
               for r in range(R)]
        outs = [torch.empty(R * count, device="cuda", dtype=torch.int32) for _ in range(R)]
        with gc3.group():
            for c, x, y in zip(comms, ins, outs):
                c.all_gather(x, y, count, "float32")
        torch.cuda.synchronize()
        want = torch.cat(ins)
        for y in outs:
            assert torch.equal(y, want)
    finally:
        for c in comms:
            c.destroy()


@pytest.mark.parametrize("name,mib", [("ring_ar_8_ch8_inst4", 64), ("hier_ar_2x4_par1", 256), ("ring_ar_8_ch1", 4)])
def test_allreduce_int_full_size_equals_sum(name, mib):
    from paper_2201_11840_b200 import gc3
    comms = _comms(name)
    R, count = 8, (mib << 20) // 4
    try:
        g = torch.Generator(device="cuda").manual_seed(2)
        ins = [torch.randint(-2 ** 20, 2 ** 20, (count,), device="cuda", dtype=torch.int32, generator=g) for _ in range(R)]
        want = torch.stack(ins).sum(0, dtype=torch.int64).to(torch.int32)
        with gc3.group():
            for c, x in zip(comms, ins):
                c.all_reduce(x, x, count, "int32", "sum")
        torch.cuda.synchronize()
        assert comms[0].async_error()[0] == 0
        for x in ins:
            assert torch.equal(x, want)
    finally:
        for c in comms:
            c.destroy()


# ---------------------------------------------------------------------------------------------
# Bit-exact parity with the CPU oracle at BASELINE.json's own sizes and dtypes (the planner picks
# different tiles, lane multipliers and bulk / L2 paths there than at the small parity sizes).

def _oracle_full(name, coll, count, dtype, proto=None, seed=3, **cfg):
    import numpy as np
    from gpu_util import input_len, oracle_collective, run_collective, to_np_bits
    comms = _comms(name, **cfg)
    R = len(comms)
    try:
        if proto is not None:
            for c in comms:
                c.set_protocol(0, proto)
        g = torch.Generator(device="cuda").manual_seed(seed)
        n = input_len(coll, count, R)
        inputs = [torch.randn(n, device="cuda", generator=g, dtype=torch.float32).to(getattr(torch, dtype)) for _ in range(R)]
        host = [x.cpu() for x in inputs]
        want_proto = {None: None, "simple": 0, "ll": 1, "ll128": 2}[proto]
        if want_proto is not None:
            assert comms[0].query_plan(coll, count, dtype)["protocol"] == want_proto
        outs = run_collective(comms, coll, inputs, count, dtype, "sum")
        torch.cuda.synchronize()
        assert comms[0].async_error()[0] == 0
        got = [to_np_bits(o, dtype) for o in outs]
        del outs, inputs
        from oracle.oracle import collective
        odt = {"bfloat16": 9, "float16": 6}.get(dtype, dtype)
        want = collective(json.loads(read_ir(name)), coll, [to_np_bits(x, dtype) for x in host], count, odt, "sum", mode="threaded")
        for r in range(R):
            if not np.array_equal(got[r], want[r]):
                bad = np.nonzero(got[r] != want[r])[0]
                raise AssertionError(f"{name} {proto} rank {r}: {bad.size} mismatches, first at {bad[:8]}")
    finally:
        for c in comms:
            c.destroy()


def test_c3_hier_allreduce_bf16_256MiB_vs_oracle():
    """C3: hierarchical 2x4 AllReduce with rrcs fusion, bf16, 256 MiB per rank."""
    _oracle_full("hier_ar_2x4_par1", "allreduce", (256 << 20) // 2, "bfloat16")


@pytest.mark.parametrize("proto", ["simple", "ll", "ll128"])
@pytest.mark.parametrize("name", ["ring_ar_8_ch8_inst4", "ring_ar_8_inst4_auto"])
def test_c4_ring_allreduce_f32_64MiB_vs_oracle(name, proto):
    """C4: ring AllReduce instances=4 / channels=8 (and auto channels), f32, 64 MiB per rank, per protocol."""
    _oracle_full(name, "allreduce", (64 << 20) // 4, "float32", proto)


def test_c5_ring_reducescatter_f32_64MiB_vs_oracle():
    """C5-RS: ring ReduceScatter over 8 ranks, f32, 64 MiB per rank (recvcount = 2 Mi elements)."""
    _oracle_full("ring_rs_8", "reducescatter", (64 << 20) // 4 // 8, "float32")


@pytest.mark.parametrize("proto", ["simple", "ll", "ll128"])
def test_c1_ring_allreduce_f32_4MiB_vs_oracle(proto):
    """C1: ring AllReduce, 1 channel, f32, 4 MiB per rank, per protocol."""
    _oracle_full("ring_ar_8_ch1", "allreduce", (4 << 20) // 4, "float32", proto)


def test_c5_ring_allgather_f32_64MiB_vs_oracle():
    _oracle_full("ring_ag_8", "allgather", (64 << 20) // 4 // 8, "float32")


def test_c2_twostep_alltoall_f32_64MiB_vs_oracle():
    _oracle_full("twostep_a2a_2x4", "alltoall", (64 << 20) // 4 // 8, "float32")
