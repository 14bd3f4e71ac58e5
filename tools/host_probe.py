#!/usr/bin/env python3
"""Host enqueue cost vs device time per step (is a config host-bound?).

    python tools/host_probe.py --config c1
Prints host µs per step (enqueue only), event µs per step back to back, and event µs per step when
the steps are queued behind a long device sleep (pure device time).
"""
import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    import torch
    import bench
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--steps", type=int, default=50)
    a = ap.parse_args()
    cfg = dict(bench.CONFIGS[a.config])
    args = argparse.Namespace(lanes=0, tile_bytes=0, instances=1, bytes=0)
    torch.cuda.set_device(0)
    R = 8
    comms = bench.setup_comms(cfg, args, R, 0, 1, 0, None)
    count = bench.per_rank_count(cfg, cfg["bytes"], R)
    n_in = bench.input_elems(cfg["coll"], count, R)
    tdt = getattr(torch, cfg["dtype"])
    ins = [torch.randn(n_in, device="cuda").to(tdt) for _ in range(R)]
    outs = [torch.empty(R * count if cfg["coll"] in ("allgather", "alltoall") else count, device="cuda", dtype=tdt)
            for _ in range(R)]
    stream = torch.cuda.Stream()
    from paper_2201_11840_b200 import gc3

    def step():
        with gc3.group():
            for c, x, y in zip(comms, ins, outs):
                if cfg["coll"] == "allreduce":
                    c.all_reduce(x, x, count, cfg["dtype"], "sum", stream)
                elif cfg["coll"] == "alltoall":
                    c.all_to_all(x, y, count, cfg["dtype"], stream)
                elif cfg["coll"] == "allgather":
                    c.all_gather(x, y, count, cfg["dtype"], stream)
                else:
                    c.reduce_scatter(x, y, count, cfg["dtype"], "sum", stream)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    out = {"config": a.config}
    t0 = time.perf_counter()
    for _ in range(a.steps):
        step()
    out["host_us_per_step"] = (time.perf_counter() - t0) / a.steps * 1e6
    torch.cuda.synchronize()
    for behind in (False, True):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            if behind:
                torch.cuda._sleep(int(2e9 * a.steps * 200e-6))  # ~200 µs per step of head start
            e0.record(stream)
            for _ in range(a.steps):
                step()
            e1.record(stream)
        torch.cuda.synchronize()
        out["device_us_behind_sleep" if behind else "event_us_back_to_back"] = e0.elapsed_time(e1) / a.steps * 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    main()
