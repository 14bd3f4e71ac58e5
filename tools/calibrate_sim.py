#!/usr/bin/env python3
"""Calibrates the timed simulator (csrc/timed.cpp) for loopback on one B200 against measured
kernel times, and reports the per-point error.

    python tools/calibrate_sim.py [--out profiles/r02_sim_calibration.md]

Measured points: the seven BASELINE configurations (bench.py --quick, device time), Simple protocol;
with --sweep the C4 message-size sweep is reported as a held-out set. Each point is simulated the way
the runtime executed it: static lanes (every thread block as `lanes` units, lane l taking tiles
l, l + lanes, ...) or, for launches on the whole grid with lanes 1, the dataflow executor
(`workers` = grid x 4 units taking ready (op, tile) items), tiles of the measured tile size, every
rank on GPU 0, local traffic sharing one device-memory resource (hbm_gbps), alpha per message, a
fixed cost per op and tile, a fixed launch cost.
The fit minimises the largest |log(predicted / measured)| over the points (grid over alpha and the
device-memory rate, the additive launch cost scanned per grid point).
"""
import argparse
import json
import math
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

IR_DIR = os.path.join(REPO, "tests", "golden", "ir")
CONFIG_POINTS = os.path.join(REPO, "profiles", "r02z_quick.jsonl")
SWEEP = os.path.join(REPO, "profiles", "r02z_sweep_c4.jsonl")
IRS = {"c1": ("ring_ar_8_ch1", "allreduce"), "c2": ("twostep_a2a_2x4", "alltoall"), "c2d": ("twostep_a2a_1x8", "alltoall"),
       "c3": ("hier_ar_2x4_par1", "allreduce"), "c4": ("ring_ar_8_ch8_inst4", "allreduce"), "c5ag": ("ring_ag_8", "allgather"),
       "c5rs": ("ring_rs_8", "reducescatter")}


def points(with_sweep=False):
    pts = []
    with open(CONFIG_POINTS) as f:
        for line in f:
            d = json.loads(line)
            if d.get("proto", "simple") != "simple" or d["config"] not in IRS:
                continue
            ir, coll = IRS[d["config"]]
            # dataflow / work-queue launches (lanes 1 on the whole grid): every unit takes ready items
            workers = d["grid"] * (16 // d.get("uw", 4)) if d["lanes"] == 1 and d["grid"] >= 148 else 0
            pts.append(dict(name=d["config"], ir=ir, coll=coll, bytes=d["bytes"], us=d["ms"] * 1e3, lanes=d["lanes"],
                            grid=d["grid"], tile=d["tile"], uw=d.get("uw", 4), group=d.get("group", 1), workers=workers))
    if not with_sweep:
        return pts
    with open(SWEEP) as f:
        for line in f:
            d = json.loads(line)
            if d.get("proto") != "simple" or not d.get("ok", True):
                continue
            pts.append(dict(name=f"c4@{d['bytes']}", ir=d["ir"], coll="allreduce", bytes=d["bytes"], us=d["us"],
                            lanes=d["lanes"], grid=None, tile=d["tile"], uw=4, group=d.get("group")))
    return pts


def chunk_bytes(irj, coll, nbytes):
    R = len(irj["gpus"])
    if coll == "allgather":
        return nbytes // irj["nchunks"]["output"]
    return nbytes // irj["nchunks"]["input"] if R else 0


class Sim:
    def __init__(self):
        from paper_2201_11840_b200 import gc3
        self.gc3 = gc3
        self.cache = {}

    def prepare(self, p):
        key = (p["ir"], p["coll"], p["bytes"], p["lanes"], p["grid"], p["tile"])
        if key in self.cache:
            return self.cache[key]
        text = open(os.path.join(IR_DIR, p["ir"] + ".ir.json")).read()
        irj = json.loads(text)
        R = len(irj["gpus"])
        ntbs = sum(len(g["threadblocks"]) for g in irj["gpus"])
        # parallel instances of the program in the launch: its lanes (work-queue / dataflow launches
        # report lanes = 1 and spread units over thread blocks: units / thread blocks)
        L = p["lanes"]
        if p["grid"] and L == 1:
            L = max(1, p["grid"] * (16 // p["uw"]) // ntbs)
        L = max(1, min(L, 64))
        cb = chunk_bytes(irj, p["coll"], p["bytes"])
        ir = self.gc3.IR(text)
        tile = min(p["tile"], cb)
        G = p.get("group")
        if G is None:  # the runtime's choice: chains run op-major groups, the largest deadlock-free G <= 64
            chain = any(o["opcode"] in ("rcs", "rrcs", "rrs") for g in irj["gpus"] for tb in g["threadblocks"] for o in tb["ops"])
            per_lane = -(-(-(-cb // tile)) // L)
            G = min(64, max(1, per_lane)) if chain else 1
            while G > 1 and not ir.simulate(cb, tile, lanes=L, group=G, rank_gpu=[0] * R)["completed"]:
                G //= 2
        p["group"] = G
        out = (ir, cb, tile, R, L)
        self.cache[key] = out
        return out

    def predict(self, p, prm):
        ir, cb, tile, R, L = self.prepare(p)
        r = ir.simulate(cb, tile, lanes=L, group=p["group"], workers=p.get("workers", 0), rank_gpu=[0] * R, alpha_us=[prm["alpha"], 2.0, 8.0], gbps=[1e9, 770.0, 50.0],
                        gamma_gbps=1e9, copy_gbps=1e9, hbm_gbps=prm["hbm"], launch_us=prm["launch"], op_us=prm.get("op", 0.0),
                        msg_read_passes=1)
        return r["makespan_us"]


def fit(sim, pts):
    """Grid over (alpha, device memory rate); the launch cost is additive, so for each grid point the
    best launch is a 1-D scan over the zero-launch predictions."""
    best = None
    for alpha in [0.5 * k for k in range(0, 9)]:
        for op in [0.5 * k for k in range(0, 7)]:
            for hbm in [500 * k for k in range(8, 19)]:
                q = {"alpha": alpha, "hbm": float(hbm), "launch": 0.0, "op": op}
                base = [sim.predict(p, q) for p in pts]
                for launch in [0.5 * k for k in range(0, 81)]:
                    worst = max(abs(math.log((b + launch) / p["us"])) for b, p in zip(base, pts))
                    if best is None or worst < best[0]:
                        best = (worst, dict(q, launch=launch))
    return best[1], best[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--sweep", action="store_true", help="also report the C4 size sweep (held out, not fitted)")
    args = ap.parse_args()
    sim = Sim()
    pts = points()
    prm, worst = fit(sim, pts)
    rows = []
    for p in pts + (points(True)[len(pts):] if args.sweep else []):
        pred = sim.predict(p, prm)
        rows.append((p["name"], p["bytes"], p["us"], pred, pred / p["us"] - 1))
    lines = ["# Timed simulator calibration (loopback, one B200)", "",
             f"`tools/calibrate_sim.py`: measured device times (bench.py --quick, Simple; `profiles/{os.path.basename(CONFIG_POINTS)}`)",
             "vs the simulator running the IR the way the launch ran it -- static lanes (c1, c5ag: lanes x thread",
             "blocks) or the dataflow / work-queue executor (c2, c2d, c3, c4, c5rs: `workers` = grid x 4 units",
             "taking ready (op, tile) items) -- at the measured tile size, all ranks on GPU 0 and one",
             "processor-shared device-memory resource. Fitted on the seven BASELINE configurations only",
             "(repeated rows are the second quick pass of the same run).", "",
             f"Fitted: alpha = {prm['alpha']} us per message, {prm['op']} us per op and tile, device memory = {prm['hbm']} GB/s, "
             f"launch = {prm['launch']} us; reducing receives read their message (+1 pass); "
             f"worst |error| = {100 * (math.exp(worst) - 1):.1f} %.", "",
             "| point | bytes / rank | measured us | predicted us | error |", "|---|---|---|---|---|"]
    for name, b, us, pred, err in rows:
        lines.append(f"| {name} | {b} | {us:.1f} | {pred:.1f} | {100 * err:+.1f} % |")
    if args.sweep:
        held = [abs(r[4]) for r in rows[len(pts):]]
        big = [abs(r[4]) for r in rows[len(pts):] if r[1] >= (64 << 20)]
        lines += ["", f"Held out (not fitted): the C4 size sweep rows `c4@bytes` (`profiles/{os.path.basename(SWEEP)}`) are",
                  "simulated with static lanes as recorded; the sweep does not record which executor or grid the",
                  f"runtime picked per size. Worst held-out error {100 * max(held):.0f} % overall, {100 * max(big or [0]):.0f} % from 64 MiB",
                  "per rank up: the fitted fixed launch cost absorbs per-launch work of the large configurations and",
                  "overstates the small-message floor, so the model extrapolates in size only above a few MiB."]
    text = "\n".join(lines) + "\n"
    print(text)
    if args.out:
        with open(args.out, "w") as f:
            f.write(text)
    print(json.dumps(prm))


if __name__ == "__main__":
    main()
