"""Seeded fuzz over the runtime's knobs (registration-time and launch-time), on several program
families: whatever combination of transports, lanes, unit sizes, tile sizes, bulk-engine paths,
work-queue mode, grouping and protocol the planner accepts, the result is bit-exact vs the oracle.
Combinations the planner rejects (e.g. co-residency) must fail cleanly, never hang or corrupt."""
import json
import random

import numpy as np
import pytest

from conftest import ir_path, read_ir

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REG = {"direct": [0, 1, 2, 3], "balance": [0, 1, 2], "l2hint": [0, 1, 3], "source": [0, 1], "slots": [2, 3]}
LAUNCH = {"unit_warps": [0, 1, 2, 4, 8], "lanes": [0, 0, 1, 3, 8], "tile_bytes": [0, 0, 4096, 16384, 65536],
          "tma": [0, 1, 3, 11], "tma_min": [0, 32768], "wq": [0, 1, 2], "group": [0, 1, 2], "taper": [0, 1],
          "wq_items": [1, 4], "wq_lag": [0, 1, 3]}
RAN, REFUSED = [], []
CASES = [("ring_ar_8_ch8_inst1", "allreduce", 8 * 70001, "float32"), ("hier_ar_2x4_par1", "allreduce", 8 * 65536, "bfloat16"),
         ("twostep_a2a_2x4", "alltoall", 40000, "float32"), ("ring_rs_8", "reducescatter", 33333, "int32"),
         ("ring_ag_4", "allgather", 50000, "float16"), ("allpairs_ar_8", "allreduce", 8 * 20000, "float32")]


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("seed", range(16))
def test_config_fuzz(case, seed):
    from paper_2201_11840_b200 import gc3
    from gpu_util import input_len, make_input, oracle_collective, run_collective, to_np_bits
    name, coll, count, dtype = CASES[case]
    rnd = random.Random(1000 * case + seed)
    reg = {k: rnd.choice(v) for k, v in REG.items()}
    launch = {k: rnd.choice(v) for k, v in LAUNCH.items()}
    proto = rnd.choice([None, None, "ll"])
    irj = json.loads(read_ir(name))
    R = len(irj["gpus"])
    comms = gc3.init_all([0] * R)
    try:
        for c in comms:
            for k, v in reg.items():
                c.set_config(k, v)
            i = c.register_ir(ir_path(name))
            if proto:
                c.set_protocol(i, proto)
            for k, v in launch.items():
                c.set_config(k, v)
        inputs = [make_input(input_len(coll, count, R), dtype, 7 * seed + r) for r in range(R)]
        expected = oracle_collective(irj, coll, [x.clone() for x in inputs], count, dtype)
        try:
            outs = run_collective(comms, coll, inputs, count, dtype)
        except gc3.NcclError as e:  # an infeasible combination is refused up front
            assert "co-resident" in str(e) or "invalid usage" in str(e), (reg, launch, proto, str(e))
            REFUSED.append((case, seed))
            return
        RAN.append((case, seed))
        torch.cuda.synchronize()
        err = comms[0].async_error()
        assert err[0] == 0, (reg, launch, proto, err)
        for r in range(R):
            got, exp = to_np_bits(outs[r], dtype), expected[r]
            ut = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[exp.dtype.itemsize]
            assert np.array_equal(got.view(ut), exp.view(ut)), (r, reg, launch, proto)
    finally:
        for c in comms:
            c.destroy()


def test_zz_most_combinations_run():
    """(runs after the fuzz cases in the same session) the fuzz is not vacuous"""
    if not RAN and not REFUSED:
        pytest.skip("fuzz cases not run in this session")
    assert len(RAN) >= 2 * len(REFUSED), (len(RAN), len(REFUSED))
