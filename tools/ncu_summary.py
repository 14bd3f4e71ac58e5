#!/usr/bin/env python3
"""Summarise ncu artefacts from gpurun_out/ into committed profiles/ files.

    python tools/ncu_summary.py <tag> <config> <ir> <bytes_per_rank> [--world 1] [--out DIR]
    python tools/ncu_summary.py --merge gpurun_out/<tag>/profiles     # box-side summaries -> profiles/

Reads gpurun_out/<tag>/launches_<config>.csv (the `--metrics gpu__time_duration.sum` launch list)
and gpurun_out/<tag>/prof_<config>.ncu-rep (one `--set full` capture of the interpreter), writes
profiles/<tag>_<config>.md and merges the per-launch DRAM traffic into profiles/ncu_summary.json
(keyed "<ir>:<bytes_per_rank>:<world>", read by bench.py for `roofline.traffic`).
"""
import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__shared_mem_per_block_dynamic"]
UNIT_SCALE = {"us": 1e3, "ns": 1, "ms": 1e6, "Kbyte/block": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}


def launches(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    out = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"]) * UNIT_SCALE.get(r["Metric Unit"], 1)
        out.append((r["Kernel Name"], r["Grid Size"], r["Block Size"], ns))
    return out


def raw(rep):
    text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k, u, v in zip(hdr, units, r):
            if k in KEYS or k == "Kernel Name":
                try:
                    d[k] = float(v.replace(",", "")) * UNIT_SCALE.get(u, 1)
                except ValueError:
                    d[k] = v
        res.append(d)
    return res


def stall_reasons(rep, top=10):
    """Kernel-wide warp-stall reasons (smsp__pcsamp_warps_issue_stalled_* sample counts, raw page)."""
    text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    if len(rows) < 3:
        return []
    hdr, vals = rows[0], rows[2]
    out = []
    for k, v in zip(hdr, vals):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                out.append((float(v.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(x[0] for x in out) or 1
    return [(n / tot, k) for n, k in sorted(out, reverse=True)[:top]]


def stalls(rep, top=8):
    """Top SASS instructions by warp-stall samples."""
    text = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    while rows and (not rows[0] or rows[0][0] != "Address"):
        rows = rows[1:]
    if not rows:
        return []
    hdr = rows[0]
    try:
        isrc, isamp = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
        iline = hdr.index("Address")
    except ValueError:
        return []
    lines = []
    for r in rows[1:]:
        try:
            lines.append((int(float(r[isamp])), r[iline], r[isrc].strip()[:100]))
        except (ValueError, IndexError):
            pass
    tot = sum(x[0] for x in lines) or 1
    return [(s / tot, ln, src) for s, ln, src in sorted(lines, reverse=True)[:top]]


def merge(src):
    dst = os.path.join(REPO, "profiles")
    os.makedirs(dst, exist_ok=True)
    for f in os.listdir(src):
        if f.endswith(".md"):
            with open(os.path.join(src, f)) as a, open(os.path.join(dst, f), "w") as b:
                b.write(a.read())
    sj = os.path.join(src, "ncu_summary.json")
    if os.path.exists(sj):
        p = os.path.join(dst, "ncu_summary.json")
        allr = json.load(open(p)) if os.path.exists(p) else {}
        allr.update(json.load(open(sj)))
        with open(p, "w") as f:
            json.dump(allr, f, indent=1, sort_keys=True)


def main():
    if sys.argv[1] == "--merge":
        return merge(sys.argv[2])
    tag, cfg, ir, nbytes = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
    outdir = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else os.path.join(REPO, "profiles")
    world = int(sys.argv[sys.argv.index("--world") + 1]) if "--world" in sys.argv else 1
    src = os.path.join(REPO, "gpurun_out", tag)
    md = [f"# ncu summary — {tag}, config {cfg} ({ir}, {nbytes} B per rank, {world} GPU)", ""]
    lpath = os.path.join(src, f"launches_{cfg}.csv")
    if os.path.exists(lpath):
        ls = launches(lpath)
        tot = sum(x[3] for x in ls) or 1
        mine = [x for x in ls if "interp" in x[0]]
        md += ["## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`; cold-cache, serialised)", "",
               "| # | kernel | grid | block | µs | share |", "|---|---|---|---|---|---|"]
        for i, (k, g, b, ns) in enumerate(ls):
            md.append(f"| {i} | `{k[:70]}` | {g} | {b} | {ns / 1e3:.1f} | {ns / tot:.1%} |")
        if mine:
            md += ["", f"Interpreter launches: {len(mine)}, mean {sum(x[3] for x in mine) / len(mine) / 1e3:.1f} µs, "
                   f"{sum(x[3] for x in mine) / tot:.1%} of all device time in the captured window "
                   "(the rest is the bench's input generation)."]
    rep = os.path.join(src, f"prof_{cfg}.ncu-rep")
    rec = None
    if os.path.exists(rep):
        for d in raw(rep):
            if "interp" not in str(d.get("Kernel Name", "")):
                continue
            rd, wr = d.get("dram__bytes_read.sum", 0), d.get("dram__bytes_write.sum", 0)
            t = d.get("gpu__time_duration.sum", 0)
            rec = {"dram_bytes": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr), "ncu_time_ns": t,
                   "capture": f"profiles/{tag}_{cfg}.md"}
            md += ["", "## `ncu --set full` capture of the interpreter", "", "| metric | value |", "|---|---|"]
            md += [f"| {k} | {d[k]:,.2f} |" if isinstance(d[k], float) else f"| {k} | {d[k]} |" for k in KEYS if k in d]
            md += [f"| DRAM read+write per launch | {rd + wr:,.0f} B |", f"| DRAM GB/s under ncu | {(rd + wr) / t:,.1f} |"]
            break
        st = stalls(rep)
        if st:
            md += ["", "## Top stall instructions (warp-stall samples, SASS)", "", "| share | address | instruction |", "|---|---|---|"]
            md += [f"| {s:.1%} | {ln} | `{src_.replace('|', '/')}` |" for s, ln, src_ in st]
        sr = stall_reasons(rep)
        if sr:
            md += ["", "## Warp-stall reasons (kernel-wide samples)", "", "| share | reason |", "|---|---|"]
            md += [f"| {s_:.1%} | {k} |" for s_, k in sr]
    os.makedirs(outdir, exist_ok=True)
    with open(os.path.join(outdir, f"{tag}_{cfg}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    if rec:
        p = os.path.join(outdir, "ncu_summary.json")
        allr = json.load(open(p)) if os.path.exists(p) else {}
        allr[f"{ir}:{nbytes}:{world}"] = rec
        with open(p, "w") as f:
            json.dump(allr, f, indent=1, sort_keys=True)
    print("\n".join(md))


if __name__ == "__main__":
    main()
