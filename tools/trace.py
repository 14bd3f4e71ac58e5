#!/usr/bin/env python3
"""Runs one config with the in-kernel event log enabled and summarises where time goes.

    python tools/trace.py --config c2 [--bytes N] [--lanes L] [--tile-bytes T] [--json out.json]

Per opcode: mean time waiting for preconditions (deps / FIFO credit / posted message), warp 0's
data time, publish lag (last warp done -> flag), and the block-level busy fraction.
"""
import argparse
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    import torch
    import bench
    from paper_2201_11840_b200 import gc3

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--bytes", type=int, default=0)
    ap.add_argument("--lanes", type=int, default=0)
    ap.add_argument("--tile-bytes", type=int, default=0)
    ap.add_argument("--proto", default=None)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS[args.config])
    if args.proto:
        cfg["proto"] = args.proto
    R = 8
    path = os.path.join(bench.IR_DIR, cfg["ir"] + ".ir.json")
    irj = json.load(open(path))
    comms = gc3.init_all([0] * R)
    for c in comms:
        if args.lanes:
            c.set_config("lanes", args.lanes)
        if args.tile_bytes:
            c.set_config("tile_bytes", args.tile_bytes)
        i = c.register_ir(path)
        if cfg["proto"]:
            c.set_protocol(i, cfg["proto"])
    nbytes = args.bytes or cfg["bytes"]
    count = bench.per_rank_count(cfg, nbytes, R)
    n_in = bench.input_elems(cfg["coll"], count, R)
    tdt = getattr(torch, cfg["dtype"])
    ins = [torch.randn(n_in, device="cuda").to(tdt) for _ in range(R)]
    outs = [torch.empty(R * count if cfg["coll"] in ("allgather", "alltoall") else count, device="cuda", dtype=tdt) for _ in range(R)]

    def step():
        with gc3.group():
            for c, x, y in zip(comms, ins, outs):
                if cfg["coll"] == "allreduce":
                    c.all_reduce(x, x, count, cfg["dtype"])
                elif cfg["coll"] == "alltoall":
                    c.all_to_all(x, y, count, cfg["dtype"])
                elif cfg["coll"] == "allgather":
                    c.all_gather(x, y, count, cfg["dtype"])
                else:
                    c.reduce_scatter(x, y, count, cfg["dtype"])

    for _ in range(3):
        step()
    for c in comms:
        c.set_config("trace", 1)
    step()
    torch.cuda.synchronize()
    tr, lanes = comms[0].trace()
    plan = comms[0].query_plan(cfg["coll"], count, cfg["dtype"])
    # unit -> (rank, tb) in launch order: thread block i runs lanes x mult_i units
    mult = gc3.IR(open(path).read()).lane_multipliers()
    blocks = []
    for g in irj["gpus"]:
        for t, tb in enumerate(g["threadblocks"]):
            blocks += [(g["rank"], tb)] * mult[g["rank"]][t]
    valid = tr[:, :, 3] > 0
    t0 = tr[:, :, 0][valid].min()
    t_end = tr[:, :, 3][valid].max()
    span = (t_end - t0) / 1e3
    stats = {}
    busy = []
    if tr.shape[0] != len(blocks) * lanes:  # balance off (uniform lanes): one unit group per thread block
        blocks = [(g["rank"], tb) for g in irj["gpus"] for tb in g["threadblocks"]]
    for b in range(tr.shape[0]):
        if blocks is None:
            break
        rank, tb = blocks[b // lanes]
        nops = len(tb["ops"])
        ev = tr[b]
        n = int((ev[:, 3] > 0).sum())
        if n == 0:
            continue
        first, last = ev[0, 0], ev[:n, 3].max()
        data = 0.0
        for q in range(n):
            op = tb["ops"][q % nops]["opcode"]
            w = (ev[q, 1] - ev[q, 0]) / 1e3
            d = (ev[q, 2] - ev[q, 1]) / 1e3
            p = (ev[q, 3] - ev[q, 2]) / 1e3 if ev[q, 3] >= ev[q, 2] else 0.0
            s = stats.setdefault(op, {"n": 0, "wait": 0.0, "data": 0.0, "publish": 0.0})
            s["n"] += 1
            s["wait"] += w
            s["data"] += d
            s["publish"] += p
            data += d
        busy.append(data / max((last - first) / 1e3, 1e-9))
    # per thread block: when its units finish (median / max)
    per_tb = []
    if blocks is not None:
        groups = {}
        for i, (rank, tb) in enumerate(blocks):
            groups.setdefault((rank, tb["id"]), []).extend(range(i * lanes, (i + 1) * lanes))
        for (rank, tid), units in groups.items():
            ends = [(tr[b, :int((tr[b, :, 3] > 0).sum()), 3].max() - t0) / 1e3 for b in units
                    if b < tr.shape[0] and (tr[b, :, 3] > 0).any()]
            if ends:
                per_tb.append({"rank": rank, "tb": tid, "units": len(units), "end_med_us": float(np.median(ends)),
                               "end_max_us": float(max(ends))})
    out = {"config": args.config, "plan": plan, "span_us": span, "blocks": int(tr.shape[0]), "per_tb": per_tb,
           "mean_block_data_fraction": float(np.mean(busy)) if busy else None,
           "per_opcode_us": {k: {"n": v["n"], "wait": v["wait"] / v["n"], "data": v["data"] / v["n"],
                                 "publish": v["publish"] / v["n"]} for k, v in stats.items()}}
    print(json.dumps(out, indent=1))
    if args.json:
        np.save(args.json.replace(".json", ".npy"), tr)
        json.dump(out, open(args.json, "w"), indent=1)
    for c in comms:
        c.destroy()


if __name__ == "__main__":
    main()
