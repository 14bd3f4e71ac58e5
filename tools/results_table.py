#!/usr/bin/env python3
"""Markdown tables for BASELINE.md §5 from the box's JSON lines.

    python tools/results_table.py gpurun_out/<tag>/quick.jsonl [gpurun_out/<tag>/sweep_c4.jsonl]
"""
import json
import sys

CFG = {"c1": ("ring_ar_8_ch1", "AllReduce", "f32"), "c2": ("twostep_a2a_2x4", "AlltoAll", "f32"),
       "c2d": ("twostep_a2a_1x8", "AlltoAll", "f32"), "c3": ("hier_ar_2x4_par1", "AllReduce", "bf16"),
       "c4": ("ring_ar_8_ch8_inst4", "AllReduce", "f32"), "c5ag": ("ring_ag_8", "AllGather", "f32"),
       "c5rs": ("ring_rs_8", "ReduceScatter", "f32")}


def lines(path):
    for ln in open(path):
        ln = ln.strip()
        if ln.startswith("{"):
            try:
                yield json.loads(ln)
            except ValueError:
                pass


def main():
    print("| Config | IR | Collective | Dtype | Proto | Bytes/rank | Time (µs) | busBW/rank (GB/s) | "
          "aggregate busBW (GB/s) | HBM roofline frac (of measured) |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for d in lines(sys.argv[1]):
        ir, coll, dt = CFG.get(d["config"], ("?", "?", "?"))
        R = 8
        print(f"| {d['config']} | `{ir}` | {coll} | {dt} | {d['proto']} | {d['bytes']} | {d['ms'] * 1e3:.1f} | "
              f"{d['agg_busbw'] / R:.1f} | {d['agg_busbw']:.1f} | {d['hbm_frac']:.3f} |")
    if len(sys.argv) > 2:
        rows = {}
        for d in lines(sys.argv[2]):
            rows.setdefault(d["bytes"], {})[d["proto"]] = d
        protos = sorted({p for r in rows.values() for p in r})
        print()
        print("| Bytes/rank | " + " | ".join(f"{p} µs | {p} busBW/rank GB/s | {p} HBM frac" for p in protos) + " |")
        print("|---|" + "---|---|---|" * len(protos))
        for b in sorted(rows):
            cells = []
            for p in protos:
                d = rows[b].get(p)
                cells += [f"{d['us']:.1f}", f"{d['busbw_gbs']:.1f}", f"{d['hbm_frac']:.3f}"] if d else ["", "", ""]
            print(f"| {b} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()
