#!/usr/bin/env python3
"""Benchmark of the GC3-IR interpreter path (BASELINE.json metric: collective bus GB/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl gc3|reference]

A "step" is one grouped collective over all IR ranks on one batch of synthetic data.  At N=1 the
8 IR ranks run as loopback ranks on cuda:0 (one cooperative launch per step); under torchrun with
N>1 the same 8-rank program is spread over the N GPUs (8/N ranks per GPU, CUDA IPC FIFOs over
NVLink), so the total work is fixed ("scaling": "strong").

`value` is the whole-job aggregate bus bandwidth: the nccl-tests busBW of one rank
(S/t * (R-1)/R for AllToAll/AllGather/ReduceScatter, S/t * 2(R-1)/R for AllReduce, S = per-rank
buffer) summed over the R ranks.  Per-rank busBW and algBW are reported alongside.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
IR_DIR = os.path.join(REPO, "tests", "golden", "ir")
METRIC = "AllReduce/AllToAll bus GB/s vs msg size at 2/4/8×B200; % NVLink peak"

# BASELINE.json configs
CONFIGS = {
    "c1": dict(ir="ring_ar_8_ch1", coll="allreduce", dtype="float32", bytes=4 << 20, proto=None,
               desc="Ring AllReduce GC3-IR, 8 ranks, 1 channel, fp32 4 MB buffer"),
    "c2": dict(ir="twostep_a2a_2x4", coll="alltoall", dtype="float32", bytes=64 << 20, proto=None,
               desc="Two-step AllToAll GC3-IR, 8 ranks, fp32 64 MB per rank, instances=1"),
    "c2d": dict(ir="twostep_a2a_1x8", coll="alltoall", dtype="float32", bytes=64 << 20, proto=None,
                desc="Direct (1x8) AllToAll GC3-IR, 8 ranks, fp32 64 MB per rank"),
    "c3": dict(ir="hier_ar_2x4_par1", coll="allreduce", dtype="bfloat16", bytes=256 << 20, proto=None,
               desc="Hierarchical (2x4 split) AllReduce with rrcs fusion, bf16 256 MB"),
    "c4": dict(ir="ring_ar_8_ch8_inst4", coll="allreduce", dtype="float32", bytes=64 << 20, proto="simple",
               desc="Ring AllReduce instances=4/channels=8"),
    "c5ag": dict(ir="ring_ag_8", coll="allgather", dtype="float32", bytes=64 << 20, proto=None,
                 desc="Ring AllGather GC3-IR, 8 ranks"),
    "c5rs": dict(ir="ring_rs_8", coll="reducescatter", dtype="float32", bytes=64 << 20, proto=None,
                 desc="Ring ReduceScatter GC3-IR, 8 ranks"),
    # C5 at 2 and 4 ranks (sweep / quick only; the 8-rank bench line stays the default contract)
    "c5ag4": dict(ir="ring_ag_4", coll="allgather", dtype="float32", bytes=64 << 20, proto=None, desc="Ring AllGather, 4 ranks"),
    "c5ag2": dict(ir="ring_ag_2", coll="allgather", dtype="float32", bytes=64 << 20, proto=None, desc="Ring AllGather, 2 ranks"),
    "c5rs4": dict(ir="ring_rs_4", coll="reducescatter", dtype="float32", bytes=64 << 20, proto=None, desc="Ring ReduceScatter, 4 ranks"),
    "c5rs2": dict(ir="ring_rs_2", coll="reducescatter", dtype="float32", bytes=64 << 20, proto=None, desc="Ring ReduceScatter, 2 ranks"),
}


def ir_ranks(cfg):
    with open(os.path.join(IR_DIR, cfg["ir"] + ".ir.json")) as f:
        return len(json.load(f)["gpus"])
ESIZE = {"float32": 4, "bfloat16": 2, "float16": 2, "int32": 4}


def bus_factor(coll, R):
    return 2.0 * (R - 1) / R if coll == "allreduce" else (R - 1) / R


def per_rank_count(cfg, nbytes, R):
    """NCCL `count` argument for a per-rank buffer of nbytes (AllGather: total output)."""
    e = ESIZE[cfg["dtype"]]
    if cfg["coll"] == "allreduce":
        return nbytes // e
    return nbytes // e // R  # alltoall / reducescatter count per peer; allgather sendcount


def input_elems(coll, count, R):
    return count if coll in ("allreduce", "allgather") else R * count


def load_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index):
        self.index, self.proc, self.lines = index, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for n, v in zip(names, p[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ------------------------------------------------------------------------------------------- gc3
def setup_comms(cfg, args, R, rank, world, local_rank, dist):
    from paper_2201_11840_b200 import gc3
    path = os.path.join(IR_DIR, cfg["ir"] + ".ir.json")
    if world == 1:
        comms = gc3.init_all([0] * R)
    else:
        per = R // world
        uid = [gc3.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comms = []
        with gc3.group():
            for k in range(per):
                comms.append(gc3.init_rank(R, uid[0], rank * per + k))
    for c in comms:
        if args.lanes:
            c.set_config("lanes", args.lanes)
        if args.tile_bytes:
            c.set_config("tile_bytes", args.tile_bytes)
        i = c.register_ir(path, args.instances)
        if cfg["proto"]:
            c.set_protocol(i, cfg["proto"])
    return comms


def run_gc3(args, cfg):
    import torch
    rank, world, local_rank = dist_env()
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    torch.cuda.set_device(local_rank)
    R = 8
    if R % world:
        raise SystemExit(f"--gpus {world} must divide the 8 IR ranks")
    comms = setup_comms(cfg, args, R, rank, world, local_rank, dist)
    nbytes = args.bytes or cfg["bytes"]
    count = per_rank_count(cfg, nbytes, R)
    n_in = input_elems(cfg["coll"], count, R)
    tdt = getattr(torch, cfg["dtype"])
    stream = torch.cuda.Stream()
    g = torch.Generator(device="cuda")
    ins, outs = [], []
    for c in comms:
        g.manual_seed(0x6C33 + c.rank)
        ins.append(torch.randn(n_in, device="cuda", generator=g, dtype=torch.float32).to(tdt))
        out_n = R * count if cfg["coll"] in ("allgather", "alltoall") else count
        outs.append(torch.empty(out_n, device="cuda", dtype=tdt))

    def step():
        from paper_2201_11840_b200 import gc3
        with gc3.group():
            for c, x, y in zip(comms, ins, outs):
                if cfg["coll"] == "allreduce":
                    c.all_reduce(x, x, count, cfg["dtype"], "sum", stream)  # in place, like nccl-tests -c 0
                elif cfg["coll"] == "alltoall":
                    c.all_to_all(x, y, count, cfg["dtype"], stream)
                elif cfg["coll"] == "allgather":
                    c.all_gather(x, y, count, cfg["dtype"], stream)
                else:
                    c.reduce_scatter(x, y, count, cfg["dtype"], "sum", stream)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    plan = comms[0].query_plan(cfg["coll"], count, cfg["dtype"])
    for _ in range(args.warmup):
        step()
    barrier()
    err = comms[0].async_error()
    if err[0]:
        raise SystemExit(f"warm-up failed: {err[1]}")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local_rank) as clocks:
        barrier()
        with torch.cuda.stream(stream):
            ev[0].record(stream)
            for k in range(args.steps):
                step()
                ev[k + 1].record(stream)
        barrier()
    per_step = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    ms = sum(per_step) / args.steps
    if dist:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    err = comms[0].async_error()
    if err[0]:
        raise SystemExit(f"timed run failed: {err[1]}")

    # e2e through the C ABI with host buffers: H2D of every rank's input, collective, D2H of the result
    if args.quick:
        e2e_ms, h2d, d2h = float("nan"), 0, 0
    else:
        e2e_ms, h2d, d2h = e2e_run(args, cfg, comms, ins, outs, count, stream, step, barrier, dist)
    bf = bus_factor(cfg["coll"], R)
    S = nbytes
    busbw = S / (ms * 1e-3) * bf / 1e9
    result = {
        "metric": METRIC, "value": round(busbw * R, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": {"float32": "f32", "bfloat16": "bf16"}.get(cfg["dtype"], cfg["dtype"]),
        "data": "synthetic (seeded N(0,1), seed 0x6C33+rank)",
        "config": {"workload": cfg["desc"], "ir": cfg["ir"], "collective": cfg["coll"], "ranks": R,
                   "bytes_per_rank": S, "count": count,
                   "placement": "loopback: 8 IR ranks on 1 GPU" if world == 1 else f"{R // world} IR ranks per GPU",
                   "protocol": "ll" if plan["protocol"] else "simple", "lanes": plan["lanes"], "grid": plan["grid"],
                   "tile_bytes": plan["tile_elems"] * ESIZE[cfg["dtype"]], "slots": plan["slots"],
                   "l2": f"inputs larger than L2 ({R * S >> 20} MiB per step)" if R * S > (126 << 20) else "L2-resident inputs",
                   "value_definition": "sum over the R ranks of nccl-tests busBW"},
        "busbw_per_rank_gbs": round(busbw, 2),
        "algbw_per_rank_gbs": round(S / (ms * 1e-3) / 1e9, 2),
        "impl": "gc3",
    }
    peaks, kind = load_peaks()
    hbm_ms = ms  # the launch is the only kernel of the step (no pre-copies for this call shape)
    achieved = plan["hbm_bytes"] / (hbm_ms * 1e-3) / 1e9 if world == 1 else None
    result["roofline"] = {
        "bound": "hbm", "achieved": round(achieved, 1) if achieved else None, "peak": peaks["hbm_gbs"],
        "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4) if achieved else None,
        "traffic": load_traffic(cfg, S, world), "peak_kind": kind,
        "algorithmic_bytes_per_launch": plan["hbm_bytes"],
        "note": "algorithmic bytes = local reads+writes of user/scratch buffers per op (send 1R, recv 1W, "
                "copy 1R1W, rrc 1R1W, rcs 1W, rrcs 1R1W, rrs 1R, reduce 2R1W) x count x chunk bytes, all ranks of the launch",
    }
    if world > 1:
        wire = plan["wire_bytes"] / (ms * 1e-3) / 1e9
        result["nvlink"] = {"achieved_wire_gbs": round(wire, 1), "peak": 770.0, "nominal": 900.0,
                            "frac_of_measured": round(wire / 770.0, 4)}
    result["e2e"] = {"value": round(S / (e2e_ms * 1e-3) * bf / 1e9 * R, 2), "unit": "GB/s",
                     "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 4)}
    result["clocks"] = clocks.summary()
    result["gpu_launches"] = args.steps * world
    if args.quick and rank == 0:
        print(json.dumps({"config": args.config, "bytes": S, "ms": round(ms, 4), "agg_busbw": result["value"],
                          "hbm_frac": result["roofline"]["frac"], "lanes": plan["lanes"], "grid": plan["grid"],
                          "tile": result["config"]["tile_bytes"], "proto": result["config"]["protocol"],
                          "uw": plan["unit_warps"], "group": plan["group"], "ntiles": plan["ntiles"]}), flush=True)
        for c in comms:
            c.destroy()
        return
    if rank == 0 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(cfg, S, R, budget_s=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(result), flush=True)
    for c in comms:
        c.destroy()
    if dist:
        dist.destroy_process_group()


def e2e_run(args, cfg, comms, ins, outs, count, stream, step, barrier, dist):
    """End to end through the C ABI with host buffers: every step uploads every rank's input from
    pinned host memory, runs the collective and downloads every rank's result into pinned host
    memory.  Device buffers are double-buffered and the copies run on their own streams, so step
    k's download overlaps step k+1's upload (PCIe is full duplex); each step's collective waits for
    its own upload and its download waits for the collective."""
    import torch
    host_in = [x.cpu().pin_memory() for x in ins]
    inplace = cfg["coll"] == "allreduce"
    host_out = [torch.empty_like(y if not inplace else x, device="cpu").pin_memory() for x, y in zip(ins, outs)]
    h2d = sum(x.numel() * x.element_size() for x in host_in)
    d2h = sum(y.numel() * y.element_size() for y in host_out)
    sets = [(ins, outs), ([torch.empty_like(x) for x in ins], [torch.empty_like(y) for y in outs])]
    # copy streams per direction (GC3_E2E_STREAMS; one saturates the PCIe link in each direction)
    ns = int(os.environ.get("GC3_E2E_STREAMS", "1"))  # measured: 1 stream 38.9, 2: 37.3, 4: 32.0 GB/s
    s_ins, s_outs = [torch.cuda.Stream() for _ in range(ns)], [torch.cuda.Stream() for _ in range(ns)]
    s_in, s_out = s_ins[0], s_outs[0]
    steps = max(1, min(args.steps, 8))
    done = [torch.cuda.Event(), torch.cuda.Event()]      # collective of the set finished
    drained = [torch.cuda.Event(), torch.cuda.Event()]   # download of the set finished
    for e in drained:
        e.record(s_out)

    def one(k):
        xs, ys = sets[k % 2]
        res = xs if inplace else ys
        for si in s_ins:
            si.wait_event(drained[k % 2])                # the set's previous result is on the host
        for i, (h, d) in enumerate(zip(host_in, xs)):
            with torch.cuda.stream(s_ins[i % ns]):
                d.copy_(h, non_blocking=True)
        for si in s_ins:
            up = torch.cuda.Event()
            up.record(si)
            stream.wait_event(up)
        run_step(xs, ys)
        done[k % 2].record(stream)
        for so in s_outs:
            so.wait_event(done[k % 2])
        for i, (d, h) in enumerate(zip(res, host_out)):
            with torch.cuda.stream(s_outs[i % ns]):
                h.copy_(d, non_blocking=True)
        for so in s_outs[1:]:
            ev = torch.cuda.Event()
            ev.record(so)
            s_out.wait_event(ev)
        drained[k % 2].record(s_out)

    def run_step(xs, ys):
        from paper_2201_11840_b200 import gc3
        with gc3.group():
            for c, x, y in zip(comms, xs, ys):
                if cfg["coll"] == "allreduce":
                    c.all_reduce(x, x, count, cfg["dtype"], "sum", stream)
                elif cfg["coll"] == "alltoall":
                    c.all_to_all(x, y, count, cfg["dtype"], stream)
                elif cfg["coll"] == "allgather":
                    c.all_gather(x, y, count, cfg["dtype"], stream)
                else:
                    c.reduce_scatter(x, y, count, cfg["dtype"], "sum", stream)

    one(0)
    one(1)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_in)
    for si in s_ins[1:]:
        si.wait_event(e0)
    for k in range(steps):
        one(k)
    e1.record(s_out)
    barrier()
    ms = e0.elapsed_time(e1) / steps
    if dist:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms, h2d, d2h


def load_traffic(cfg, S, world):
    """dram read+write bytes per launch from the committed ncu capture of this workload, if any."""
    path = os.path.join(REPO, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        rec = d.get(f"{cfg['ir']}:{S}:{world}")
        return rec["dram_bytes"] if rec else None
    except (OSError, KeyError, ValueError):
        return None


# ------------------------------------------------------------------------------------------- CPU
def cpu_run(cfg, S, R, budget_s, threads=True):
    """The CPU oracle (restated reference interpreter) on the same IR; returns (GB/s agg, sample, cores)."""
    import numpy as np
    from oracle.oracle import FlatIR
    ir = FlatIR(os.path.join(IR_DIR, cfg["ir"] + ".ir.json"))
    e = ESIZE[cfg["dtype"]]
    count = per_rank_count(cfg, S, R)
    nin, nout, nsc = ir.nchunks
    ce = count // nin if cfg["coll"] in ("allreduce", "allgather") else count // (nin // R)
    np_dt = {"float32": np.float32, "bfloat16": np.uint16}[cfg["dtype"]]
    rng = np.random.default_rng(0)
    bufs = []
    for r in range(R):
        inp = rng.standard_normal(nin * ce).astype(np.float32)
        if np_dt is np.uint16:
            inp = (inp.view(np.uint32) >> 16).astype(np.uint16)
        out = inp if ir.inplace else np.zeros(nout * ce, dtype=np_dt)
        sc = np.zeros(max(nsc, 1) * ce, dtype=np_dt)
        bufs.append([inp, out, sc])
    ntbs = sum(len(g["threadblocks"]) for g in ir.json["gpus"])
    times, t_start = [], time.time()
    mode = "threaded" if threads else "deterministic"
    dt = {"float32": 7, "bfloat16": 9}[cfg["dtype"]]
    tile = max(1, (256 << 10) // e // max(1, max(o["count"] for g in ir.json["gpus"] for t in g["threadblocks"] for o in t["ops"])))
    while True:
        t0 = time.perf_counter()
        rc, err = ir.run(bufs, ce, dt, "sum", mode=mode, slots=2, tile_elems=tile)
        times.append(time.perf_counter() - t0)
        if rc != 0:
            raise RuntimeError(err)
        if time.time() - t_start > budget_s or len(times) >= 20:
            break
    t = sum(times) / len(times)
    agg = S / t * bus_factor(cfg["coll"], R) / 1e9 * R
    cores = min(ntbs, os.cpu_count() or 1) if threads else 1
    sample = f"{len(times)} full runs of {cfg['ir']} ({R} ranks x {S >> 20} MiB), oracle {mode} mode, {ntbs} threads"
    return agg, sample, cores, t


def cpu_baseline(cfg, S, R, budget_s=10.0):
    agg, sample, cores, _ = cpu_run(cfg, S, R, budget_s)
    return {"value": round(agg, 3), "unit": "GB/s", "cores": cores, "kind": "port", "sample": sample,
            "host_cpu": host_cpu()}


def host_cpu():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical cpus)"
    except OSError:
        pass
    return f"{os.cpu_count()} logical cpus"


def run_sweep(args, cfg):
    """Message-size sweep (BASELINE config C4: 1 KiB - 1 GiB, Simple vs LL): one JSON line per
    (protocol, size) with the device time of one collective (CUDA events, mean of the timed steps,
    inputs re-used: small sizes are L2-resident), algBW / busBW per rank and the HBM roofline
    fraction of the launch's algorithmic bytes."""
    import torch
    from paper_2201_11840_b200 import gc3
    torch.cuda.set_device(0)
    R = ir_ranks(cfg)
    comms = setup_comms(dict(cfg, proto=None), args, R, 0, 1, 0, None)
    peaks, _ = load_peaks()
    stream = torch.cuda.Stream()
    lo, hi = args.sweep_min, args.sweep_max
    sizes = []
    b = lo
    while b <= hi:
        sizes.append(b)
        b *= 2
    tdt = getattr(torch, cfg["dtype"])
    for proto in args.sweep_protos.split(","):
        for c in comms:
            c.set_protocol(0, proto)
        for nbytes in sizes:
            count = per_rank_count(cfg, nbytes, R)
            n_in = input_elems(cfg["coll"], count, R)
            ins = [torch.randn(n_in, device="cuda").to(tdt) for _ in comms]
            outs = [torch.empty(R * count if cfg["coll"] in ("allgather", "alltoall") else count, device="cuda", dtype=tdt)
                    for _ in comms]

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
            steps = max(3, min(args.steps, int(2e9 // max(nbytes * R, 1))))
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            err = comms[0].async_error()
            plan = comms[0].query_plan(cfg["coll"], count, cfg["dtype"])
            print(json.dumps({"config": args.config, "ir": cfg["ir"], "ranks": R, "proto": proto, "bytes": nbytes, "us": round(ms * 1e3, 2),
                              "algbw_gbs": round(nbytes / (ms * 1e-3) / 1e9, 2),
                              "busbw_gbs": round(nbytes / (ms * 1e-3) / 1e9 * bus_factor(cfg["coll"], R), 2),
                              "hbm_frac": round(plan["hbm_bytes"] / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 4),
                              "lanes": plan["lanes"], "tile": plan["tile_elems"] * ESIZE[cfg["dtype"]], "ok": err[0] == 0}),
                  flush=True)
            del ins, outs
    for c in comms:
        c.destroy()


def run_reference(args, cfg):
    """The reference arm: the reference's interpreter semantics on the host cores (oracle port;
    the reference ships no runtime)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    S = args.bytes or cfg["bytes"]
    R = 8
    times = []
    for _ in range(args.warmup):
        cpu_run(cfg, S, R, budget_s=0.0)
    for _ in range(args.steps):
        agg, sample, cores, t = cpu_run(cfg, S, R, budget_s=0.0)
        times.append(t)
    t = sum(times) / len(times)
    agg = S / t * bus_factor(cfg["coll"], R) / 1e9 * R
    out = {
        "metric": METRIC, "value": round(agg, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": {"float32": "f32", "bfloat16": "bf16"}.get(cfg["dtype"]), "data": "synthetic",
        "config": {"workload": cfg["desc"], "ir": cfg["ir"], "collective": cfg["coll"], "ranks": R,
                   "bytes_per_rank": S},
        "impl": "reference",
        "cpu_baseline": {"value": round(agg, 3), "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": f"each step: {sample}", "host_cpu": host_cpu()},
        "e2e": {"value": round(agg, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="gc3", choices=["gc3", "reference"])
    ap.add_argument("--bytes", type=int, default=0, help="override the per-rank buffer size")
    ap.add_argument("--proto", default=None, choices=[None, "simple", "ll"])
    ap.add_argument("--lanes", type=int, default=0)
    ap.add_argument("--tile-bytes", type=int, default=0)
    ap.add_argument("--instances", type=int, default=1)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="kernel timing only: one compact JSON line")
    ap.add_argument("--sweep", action="store_true", help="message-size sweep (one JSON line per protocol and size)")
    ap.add_argument("--sweep-min", type=int, default=1 << 10)
    ap.add_argument("--sweep-max", type=int, default=1 << 30)
    ap.add_argument("--sweep-protos", default="simple,ll")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = dict(CONFIGS[args.config])
    if args.proto:
        cfg["proto"] = args.proto
    if args.sweep:
        run_sweep(args, cfg)
    elif args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_gc3(args, cfg)


if __name__ == "__main__":
    main()
