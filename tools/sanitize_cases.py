#!/usr/bin/env python3
"""Small collectives for compute-sanitizer (tools/sanitize.sh): C1 (ring AllReduce), C2 (two-step
AlltoAll, work queue), C3 (hierarchical AllReduce, bf16), dataflow mode, LL and LL128 — each
through the C ABI on 8 loopback ranks of cuda:0 and checked bit-exact against the oracle.

    python tools/sanitize_cases.py [case ...]
"""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

CASES = {
    "c1": ("ring_ar_8_ch1", "allreduce", 8 * 4096, "float32", {}),
    "c2": ("twostep_a2a_2x4", "alltoall", 4096, "float32", {}),
    "c3": ("hier_ar_2x4_par1", "allreduce", 8 * 8192, "bfloat16", {}),
    "c4df": ("ring_ar_8_ch8_inst4", "allreduce", 32 * 4096, "float32", {"df": 2, "df_min_tile": 4096}),
    "c1ll": ("ring_ar_8_ch1", "allreduce", 8 * 4096, "float32", {"proto": "ll"}),
    "c1ll128": ("ring_ar_8_ch1", "allreduce", 8 * 4096, "float32", {"proto": "ll128"}),
    "c5rs_tma": ("ring_rs_8", "reducescatter", 16384, "float32", {"tma_min": 1024}),
}


def run(name):
    import numpy as np
    import torch
    from paper_2201_11840_b200 import gc3
    from gpu_util import input_len, make_input, oracle_collective, run_collective, to_np_bits
    ir, coll, count, dtype, cfg = CASES[name]
    path = os.path.join(REPO, "tests", "golden", "ir", ir + ".ir.json")
    irj = json.load(open(path))
    R = len(irj["gpus"])
    comms = gc3.init_all([0] * R)
    try:
        for c in comms:
            for k, v in cfg.items():
                if k != "proto":
                    c.set_config(k, v)
            i = c.register_ir(path)
            if "proto" in cfg:
                c.set_protocol(i, cfg["proto"])
        ins = [make_input(input_len(coll, count, R), dtype, 7 + r) for r in range(R)]
        exp = oracle_collective(irj, coll, [x.clone() for x in ins], count, dtype)
        outs = run_collective(comms, coll, ins, count, dtype)
        torch.cuda.synchronize()
        assert comms[0].async_error()[0] == 0
        for r in range(R):
            assert np.array_equal(to_np_bits(outs[r], dtype), exp[r]), (name, r)
    finally:
        for c in comms:
            c.destroy()
    print(f"{name}: ok")


if __name__ == "__main__":
    for n in sys.argv[1:] or list(CASES):
        run(n)
