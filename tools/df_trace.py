#!/usr/bin/env python3
"""Event log of one dataflow launch (interp_df_kernel) and where its time goes.

    GC3_DF=2 python tools/df_trace.py --config c4 [--bytes N] [--tile-bytes T]

Every (node, tile) item records four %globaltimer stamps: its queue position claimed, the item
ready (resolved), its data moved, its successors published. Reported: the launch span, the
units' busy fraction (ready -> published summed over items / units x span), the mean claim wait,
move and publish times, the number of items moving over time (deciles of the span) and the
achieved algorithmic bandwidth.
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
    ap.add_argument("--config", default="c4")
    ap.add_argument("--bytes", type=int, default=0)
    ap.add_argument("--tile-bytes", type=int, default=0)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS[args.config])
    R = bench.ir_ranks(cfg)
    comms = gc3.init_all([0] * R)
    for c in comms:
        if args.tile_bytes:
            c.set_config("tile_bytes", args.tile_bytes)
        c.register_ir(os.path.join(bench.IR_DIR, cfg["ir"] + ".ir.json"))
        if cfg["proto"]:
            c.set_protocol(0, cfg["proto"])
    S = args.bytes or cfg["bytes"]
    count = bench.per_rank_count(cfg, S, R)
    n_in = bench.input_elems(cfg["coll"], count, R)
    tdt = getattr(torch, cfg["dtype"])
    ins = [torch.randn(n_in, device="cuda").to(tdt) for _ in comms]
    outs = [torch.empty(R * count if cfg["coll"] in ("allgather", "alltoall") else count, device="cuda", dtype=tdt) for _ in comms]

    def step():
        with gc3.group():
            for c, x, y in zip(comms, ins, outs):
                if cfg["coll"] == "allreduce":
                    c.all_reduce(x, x, count, cfg["dtype"], "sum")
                elif cfg["coll"] == "alltoall":
                    c.all_to_all(x, y, count, cfg["dtype"])
                elif cfg["coll"] == "allgather":
                    c.all_gather(x, y, count, cfg["dtype"])
                else:
                    c.reduce_scatter(x, y, count, cfg["dtype"], "sum")
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    plan = comms[0].query_plan(cfg["coll"], count, cfg["dtype"])
    if plan["mode"] != 2:
        raise SystemExit(f"not a dataflow launch (mode {plan['mode']}); set GC3_DF=2")
    for c in comms:
        c.set_config("trace", 1)
    step()
    torch.cuda.synchronize()
    tr, _ = comms[0].trace()
    tr = tr.reshape(-1, 4).astype(np.int64)
    tr = tr[tr[:, 3] > 0]
    t0 = tr[:, 0].min()
    tr = tr - t0
    span = tr[:, 3].max()
    units = plan["grid"] * (512 // 32 // plan["unit_warps"])
    wait = tr[:, 1] - tr[:, 0]
    move = tr[:, 2] - tr[:, 1]
    pub = tr[:, 3] - tr[:, 2]
    busy = (tr[:, 3] - tr[:, 1]).sum() / (units * span)
    dec = []
    for k in range(10):
        a, b = span * k / 10, span * (k + 1) / 10
        ov = np.clip(np.minimum(tr[:, 2], b) - np.maximum(tr[:, 1], a), 0, None).sum() / (b - a)
        dec.append(round(float(ov), 1))
    out = {"config": args.config, "bytes": S, "items": int(len(tr)), "units": units, "tile": plan["tile_elems"] * bench.ESIZE[cfg["dtype"]],
           "span_us": round(span / 1e3, 1), "busy_frac": round(float(busy), 3),
           "wait_us_mean": round(float(wait.mean()) / 1e3, 2), "wait_us_p90": round(float(np.percentile(wait, 90)) / 1e3, 2),
           "move_us_mean": round(float(move.mean()) / 1e3, 2), "move_us_p90": round(float(np.percentile(move, 90)) / 1e3, 2),
           "publish_us_mean": round(float(pub.mean()) / 1e3, 2),
           "moving_items_by_decile": dec,
           "algorithmic_gbs": round(plan["hbm_bytes"] / span, 1)}
    print(json.dumps(out))
    if args.json:
        with open(args.json, "w") as f:
            json.dump({"summary": out, "trace": tr.tolist()}, f)
    for c in comms:
        c.destroy()


if __name__ == "__main__":
    main()
