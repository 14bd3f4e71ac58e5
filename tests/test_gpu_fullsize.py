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
