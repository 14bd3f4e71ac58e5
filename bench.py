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
    "c1ap": dict(ir="allpairs_ar_8", coll="allreduce", dtype="float32", bytes=4 << 20, proto=None,
                 desc="All-pairs AllReduce GC3-IR, 8 ranks, fp32 4 MB buffer (small-message alternative to C1)"),
    "c4auto": dict(ir="ring_ar_8_inst4_auto", coll="allreduce", dtype="float32", bytes=64 << 20, proto="simple",
                   desc="Ring AllReduce instances=4, automatic channels"),
    "c4i1": dict(ir="ring_ar_8_ch8_inst1", coll="allreduce", dtype="float32", bytes=64 << 20, proto=None,
                 desc="Ring AllReduce channels=8, instances=1 (sweep / quick only)"),
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


PROTO_NAMES = {0: "simple", 1: "ll", 2: "ll128"}
NVLINK_PEER_GBS = 770.0  # measured peer copy per direction per GPU (B200_PROFILING.md; 900 nominal)


def workload_config(cfg, S, R, world):
    """The `config` object of the JSON line: identical in both arms (gc3 and reference)."""
    return {"workload": cfg["desc"], "ir": cfg["ir"], "collective": cfg["coll"], "dtype": cfg["dtype"], "ranks": R,
            "bytes_per_rank": S, "count": per_rank_count(cfg, S, R),
            "placement": "loopback: 8 IR ranks on 1 GPU" if world == 1 else f"{R // world} IR ranks per GPU",
            "l2": f"inputs larger than L2 ({R * S >> 20} MiB per step)" if R * S > (126 << 20) else "L2-resident inputs",
            "value_definition": "sum over the R ranks of nccl-tests busBW"}


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
        if getattr(args, "builtin", False):
            continue  # no registration: every call runs the runtime's built-in program for its size
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
    verified = verify_outputs(cfg, comms, count, stream, dist)
    result = {
        "metric": METRIC, "value": round(busbw * R, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": {"float32": "f32", "bfloat16": "bf16"}.get(cfg["dtype"], cfg["dtype"]),
        "data": "synthetic (seeded N(0,1), seed 0x6C33+rank)",
        "config": workload_config(cfg, S, R, world),
        "plan": {"protocol": PROTO_NAMES.get(plan["protocol"], plan["protocol"]), "lanes": plan["lanes"], "grid": plan["grid"],
                 "tile_bytes": plan["tile_elems"] * ESIZE[cfg["dtype"]], "slots": plan["slots"]},
        "busbw_per_rank_gbs": round(busbw, 2),
        "algbw_per_rank_gbs": round(S / (ms * 1e-3) / 1e9, 2),
        "verified": verified,
        "impl": "gc3",
    }
    peaks, kind = load_peaks()
    if world == 1:
        # loopback: every message is HBM traffic; the launch is the only kernel of the step
        achieved = plan["hbm_bytes"] / (ms * 1e-3) / 1e9
        result["roofline"] = {
            "bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": load_traffic(cfg, S, world), "peak_kind": kind,
            "algorithmic_bytes_per_launch": plan["hbm_bytes"],
            "note": "algorithmic bytes = local reads+writes of user/scratch buffers per op (send 1R, recv 1W, "
                    "copy 1R1W, rrc 1R1W, rcs 1W, rrcs 1R1W, rrs 1R, reduce 2R1W) x count x chunk bytes, all ranks of the launch",
        }
    else:
        # across GPUs: the bytes that must cross NVLink (max over ranks of bytes sent or received) per
        # launch over the measured peer-copy bandwidth
        wire = plan["wire_bytes"] / (ms * 1e-3) / 1e9
        result["roofline"] = {
            "bound": "nvlink", "achieved": round(wire, 1), "peak": NVLINK_PEER_GBS, "unit": "GB/s",
            "frac": round(wire / NVLINK_PEER_GBS, 4), "traffic": None, "peak_kind": "measured peer copy (B200_PROFILING.md)",
            "algorithmic_bytes_per_launch": plan["wire_bytes"],
            "note": "wire bytes = max over ranks of chunks sent or received x chunk bytes; 900 GB/s nominal",
        }
    result["e2e"] = {"value": round(S / (e2e_ms * 1e-3) * bf / 1e9 * R, 2), "unit": "GB/s",
                     "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 4)}
    result["clocks"] = clocks.summary()
    result["gpu_launches"] = args.steps * world
    if args.quick and rank == 0:
        print(json.dumps({"config": args.config, "bytes": S, "ms": round(ms, 4), "agg_busbw": result["value"],
                          "hbm_frac": result["roofline"]["frac"], "lanes": plan["lanes"], "grid": plan["grid"],
                          "tile": result["plan"]["tile_bytes"], "proto": result["plan"]["protocol"], "verified": verified,
                          "uw": plan["unit_warps"], "group": plan["group"], "ntiles": plan["ntiles"]}), flush=True)
        for c in comms:
            c.destroy()
        return
    if world == 1 and not args.no_more:
        for c in comms:
            c.destroy()
        comms = []
        result["more"] = [more_config(name, args) for name in args.more.split(",") if name]
    if rank == 0 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(cfg, S, R, budget_s=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(result), flush=True)
    for c in comms:
        c.destroy()
    if dist:
        dist.destroy_process_group()


def verify_outputs(cfg, comms, count, stream=None, dist=None, seed=0x5EED, ir_json=None):
    """Parity gate of a timed configuration: one more collective on fresh seeded inputs, checked
    exactly. AllToAll / AllGather outputs must be the exact permutation of the inputs; reductions
    must equal the CPU oracle's result (oracle/, used here only as the checker) bit for bit.
    Returns True, or raises."""
    import json as _json
    import numpy as np
    import torch
    from paper_2201_11840_b200 import gc3
    R = comms[0].nranks
    coll, dt = cfg["coll"], cfg["dtype"]
    tdt = getattr(torch, dt)
    n_in = input_elems(coll, count, R)

    def host_input(r):
        g = torch.Generator(device="cpu").manual_seed(seed + r)
        return torch.randn(n_in, generator=g, dtype=torch.float32).to(tdt)

    hins = {c.rank: host_input(c.rank) for c in comms}
    ins = {r: x.cuda() for r, x in hins.items()}
    outs = {}
    with gc3.group():
        for c in comms:
            x = ins[c.rank]
            if coll == "allreduce":
                outs[c.rank] = torch.empty(count, device="cuda", dtype=tdt)
                c.all_reduce(x, outs[c.rank], count, dt, "sum", stream)
            elif coll == "alltoall":
                outs[c.rank] = torch.empty(R * count, device="cuda", dtype=tdt)
                c.all_to_all(x, outs[c.rank], count, dt, stream)
            elif coll == "allgather":
                outs[c.rank] = torch.empty(R * count, device="cuda", dtype=tdt)
                c.all_gather(x, outs[c.rank], count, dt, stream)
            else:
                outs[c.rank] = torch.empty(count, device="cuda", dtype=tdt)
                c.reduce_scatter(x, outs[c.rank], count, dt, "sum", stream)
    torch.cuda.synchronize()
    err = comms[0].async_error()
    if err[0]:
        raise SystemExit(f"verification run failed: {err[1]}")
    if coll in ("alltoall", "allgather"):
        allin = [hins[r] if r in hins else host_input(r) for r in range(R)]
        for d, y in outs.items():
            y = y.cpu()
            for s_ in range(R):
                want = allin[s_][d * count:(d + 1) * count] if coll == "alltoall" else allin[s_]
                if not torch.equal(y[s_ * count:(s_ + 1) * count].view(torch.int16 if tdt != torch.float32 else torch.int32),
                                   want.view(torch.int16 if tdt != torch.float32 else torch.int32)):
                    raise SystemExit(f"verification failed: rank {d} block {s_} differs")
        return True
    from oracle.oracle import collective

    def bits(t):
        t = t.contiguous()
        return t.view(torch.int16).numpy().view(np.uint16) if t.element_size() == 2 else t.view(torch.int32).numpy().view(np.uint32)

    if ir_json is not None:  # the program the runtime ran (e.g. a built-in), given by the caller
        irj = ir_json
    else:
        with open(os.path.join(IR_DIR, cfg["ir"] + ".ir.json")) as f:
            irj = _json.load(f)
    odt = {"bfloat16": 9, "float16": 6}.get(dt, dt)
    want = collective(irj, coll, [bits(hins[r] if r in hins else host_input(r)) for r in range(R)], count, odt, "sum",
                      mode="threaded")
    for r, y in outs.items():
        if not np.array_equal(bits(y.cpu()), want[r]):
            raise SystemExit(f"verification failed: rank {r} differs from the oracle")
    return True


def more_config(name, args):
    """Device time of another BASELINE configuration (the AllReduce half of the metric), verified
    like the headline: {config, ms, aggregate busBW, HBM roofline fraction}."""
    import torch
    from paper_2201_11840_b200 import gc3
    cfg = CONFIGS[name]
    R = ir_ranks(cfg)
    comms = setup_comms(dict(cfg), args, R, 0, 1, 0, None)
    try:
        S = cfg["bytes"]
        count = per_rank_count(cfg, S, R)
        tdt = getattr(torch, cfg["dtype"])
        n_in = input_elems(cfg["coll"], count, R)
        g = torch.Generator(device="cuda")
        ins = []
        for c in comms:
            g.manual_seed(0x6C33 + c.rank)
            ins.append(torch.randn(n_in, device="cuda", generator=g, dtype=torch.float32).to(tdt))
        outs = [torch.empty(R * count if cfg["coll"] in ("allgather", "alltoall") else count, device="cuda", dtype=tdt)
                for _ in comms]
        stream = torch.cuda.Stream()

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
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        steps = max(5, min(args.steps, 20))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        err = comms[0].async_error()
        if err[0]:
            raise SystemExit(f"{name} failed: {err[1]}")
        plan = comms[0].query_plan(cfg["coll"], count, cfg["dtype"])
        del ins, outs
        verified = verify_outputs(cfg, comms, count, stream)
        peaks, _ = load_peaks()
        busbw = S / (ms * 1e-3) * bus_factor(cfg["coll"], R) / 1e9
        return {"config": name, "ir": cfg["ir"], "collective": cfg["coll"], "dtype": cfg["dtype"], "bytes_per_rank": S,
                "protocol": PROTO_NAMES.get(plan["protocol"]), "ms_per_step": round(ms, 5), "value": round(busbw * R, 2),
                "unit": "GB/s", "hbm_frac": round(plan["hbm_bytes"] / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 4),
                "verified": verified}
    finally:
        for c in comms:
            c.destroy()


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
class CpuWorkload:
    """The CPU oracle (restated reference interpreter) on the same IR and sizes: buffers allocated
    and first-touched once (no page faults inside the timed runs), inputs restored before every
    run outside the timed region (the in-place reductions would otherwise feed their own output)."""

    def __init__(self, cfg, S, R, threads=True):
        import numpy as np
        from oracle.oracle import FlatIR
        self.cfg, self.S, self.R, self.threads = cfg, S, R, threads
        self.ir = ir = FlatIR(os.path.join(IR_DIR, cfg["ir"] + ".ir.json"))
        e = ESIZE[cfg["dtype"]]
        count = per_rank_count(cfg, S, R)
        nin, nout, nsc = ir.nchunks
        self.ce = count // nin if cfg["coll"] in ("allreduce", "allgather") else count // (nin // R)
        np_dt = {"float32": np.float32, "bfloat16": np.uint16}[cfg["dtype"]]
        rng = np.random.default_rng(0)
        self.bufs, self.pristine = [], []
        for r in range(R):
            inp = rng.standard_normal(nin * self.ce).astype(np.float32)
            if np_dt is np.uint16:
                inp = (inp.view(np.uint32) >> 16).astype(np.uint16)
            out = inp if ir.inplace else np.zeros(nout * self.ce, dtype=np_dt)
            sc = np.zeros(max(nsc, 1) * self.ce, dtype=np_dt)
            self.bufs.append([inp, out, sc])
            self.pristine.append(inp.copy())
        self.ntbs = sum(len(g["threadblocks"]) for g in ir.json["gpus"])
        self.mode = "threaded" if threads else "deterministic"
        self.dt = {"float32": 7, "bfloat16": 9}[cfg["dtype"]]
        maxc = max(o["count"] for g in ir.json["gpus"] for t in g["threadblocks"] for o in t["ops"])
        self.tile = max(1, (256 << 10) // e // max(1, maxc))
        self.cores = min(self.ntbs, os.cpu_count() or 1) if threads else 1

    def run(self):
        """One full run of the IR over all ranks; returns seconds (inputs restored first, untimed)."""
        import numpy as np
        for b, p in zip(self.bufs, self.pristine):
            np.copyto(b[0], p)
        t0 = time.perf_counter()
        rc, err = self.ir.run(self.bufs, self.ce, self.dt, "sum", mode=self.mode, slots=2, tile_elems=self.tile)
        t = time.perf_counter() - t0
        if rc != 0:
            raise RuntimeError(err)
        return t

    def gbs(self, t):
        return self.S / t * bus_factor(self.cfg["coll"], self.R) / 1e9 * self.R

    def sample(self, n):
        return (f"{n} full runs of {self.cfg['ir']} ({self.R} ranks x {self.S >> 20} MiB, buffers allocated and touched once), "
                f"oracle {self.mode} mode, {self.ntbs} threads")


def cpu_baseline(cfg, S, R, budget_s=10.0):
    w = CpuWorkload(cfg, S, R)
    w.run()  # warm: page-in, thread creation paths
    times, t_start = [], time.time()
    while time.time() - t_start < budget_s and len(times) < 20:
        times.append(w.run())
    t = sum(times) / len(times)
    return {"value": round(w.gbs(t), 3), "unit": "GB/s", "cores": w.cores, "kind": "port", "sample": w.sample(len(times)),
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


def verify_int_sum(cfg, comms, nbytes, stream):
    """Parity property for reductions too large for the oracle: int32 data (wrapping sum: the
    association does not matter) must equal the torch sum exactly."""
    import torch
    from paper_2201_11840_b200 import gc3
    R = comms[0].nranks
    icfg = dict(cfg, dtype="int32")
    count = per_rank_count(icfg, nbytes, R)
    n_in = input_elems(cfg["coll"], count, R)
    g = torch.Generator(device="cuda").manual_seed(7)
    ins = [torch.randint(-2 ** 20, 2 ** 20, (n_in,), device="cuda", dtype=torch.int32, generator=g) for _ in comms]
    want = torch.stack(ins).sum(0, dtype=torch.int64).to(torch.int32)
    outs = [torch.empty(count, device="cuda", dtype=torch.int32) for _ in comms]
    with gc3.group():
        for c, x, y in zip(comms, ins, outs):
            if cfg["coll"] == "allreduce":
                c.all_reduce(x, y, count, "int32", "sum", stream)
            else:
                c.reduce_scatter(x, y, count, "int32", "sum", stream)
    torch.cuda.synchronize()
    if comms[0].async_error()[0]:
        raise SystemExit("verification run failed")
    for c, y in zip(comms, outs):
        w = want if cfg["coll"] == "allreduce" else want[c.rank * count:(c.rank + 1) * count]
        if not torch.equal(y, w):
            raise SystemExit(f"verification failed: rank {c.rank} int32 sum differs")
    return True


def run_sweep(args, cfg):
    """Message-size sweep (BASELINE configs C4 / C5: 1 KiB - 1 GiB per protocol): one JSON line per
    (protocol, size) with the device time of one collective (CUDA events, mean of the timed steps,
    inputs re-used: small sizes are L2-resident), algBW / busBW per rank and the HBM roofline
    fraction of the launch's algorithmic bytes. Every point is verified before it is printed:
    permutations exactly, reductions against the oracle up to 64 MiB per rank and by an exact int32
    sum above."""
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
    for proto in (["builtin"] if args.builtin else args.sweep_protos.split(",")):
        for c in comms:
            if not args.builtin:
                c.set_protocol(0, proto)
        for nbytes in sizes:
            count = per_rank_count(cfg, nbytes, R)
            n_in = input_elems(cfg["coll"], count, R)
            irj = None
            if args.builtin:  # the built-in program this size runs (size tiers), for the parity gate
                sel = count * ESIZE[cfg["dtype"]] * (1 if cfg["coll"] == "allreduce" else R)
                irj = json.loads(gc3.IR.builtin(cfg["coll"], R, sel).serialize())
            if cfg["coll"] in ("alltoall", "allgather") or nbytes <= (64 << 20):
                verified = verify_outputs(cfg, comms, count, stream, ir_json=irj)
            else:
                verified = verify_int_sum(cfg, comms, nbytes, stream)
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
            graph_us = graph_time_us(step, stream) if args.graph and nbytes <= args.graph_max else None
            err = comms[0].async_error()
            plan = comms[0].query_plan(cfg["coll"], count, cfg["dtype"])
            print(json.dumps({"config": args.config, "ir": plan["name"] if args.builtin else cfg["ir"], "ranks": R, "proto": proto,
                              "bytes": nbytes, "us": round(ms * 1e3, 2),
                              "graph_us": graph_us,
                              "algbw_gbs": round(nbytes / (ms * 1e-3) / 1e9, 2),
                              "busbw_gbs": round(nbytes / (ms * 1e-3) / 1e9 * bus_factor(cfg["coll"], R), 2),
                              "hbm_frac": round(plan["hbm_bytes"] / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 4),
                              "ran": PROTO_NAMES.get(plan["protocol"]), "lanes": plan["lanes"],
                              "tile": plan["tile_elems"] * ESIZE[cfg["dtype"]], "ok": err[0] == 0, "verified": verified}),
                  flush=True)
            del ins, outs
    for c in comms:
        c.destroy()


def graph_time_us(step, stream, reps=20):
    """Per-collective device time with `reps` collectives captured in one CUDA graph (launch cost
    amortised: the small-message floor without host enqueue overhead)."""
    import torch
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        step()  # warm on the capture stream
        stream.synchronize()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(reps):
                step()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    with torch.cuda.stream(stream):
        for _ in range(5):
            g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) * 1e3 / (5 * reps), 2)


def run_reference(args, cfg):
    """The reference arm: the reference's interpreter semantics on the host cores (oracle port;
    the reference ships no runtime), with warm buffers like the gc3 arm's
    cpu_baseline: W untimed runs, then K timed runs of the whole workload."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    S = args.bytes or cfg["bytes"]
    R = ir_ranks(cfg)
    w = CpuWorkload(cfg, S, R)
    for _ in range(args.warmup):
        w.run()
    times = [w.run() for _ in range(args.steps)]
    t = sum(times) / len(times)
    agg = w.gbs(t)
    out = {
        "metric": METRIC, "value": round(agg, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": {"float32": "f32", "bfloat16": "bf16"}.get(cfg["dtype"]),
        "data": "synthetic (seeded N(0,1))",
        "config": workload_config(cfg, S, R, world),
        "impl": "reference",
        "cpu_baseline": {"value": round(agg, 3), "unit": "GB/s", "cores": w.cores, "kind": "port",
                         "sample": f"each step: {w.sample(1)}", "host_cpu": host_cpu()},
        "e2e": {"value": round(agg, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def enforce_world(args):
    """--gpus N means N processes, one per GPU: under torchrun WORLD_SIZE must be N; without it the
    bench re-executes itself under torch.distributed.run. Never a silent loopback fallback."""
    rank, world, _ = dist_env()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if "WORLD_SIZE" in os.environ:
        if world != args.gpus:
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    elif args.gpus > 1:
        if args.impl == "gc3":
            import torch
            n = torch.cuda.device_count()
            if n < args.gpus:
                raise SystemExit(f"--gpus {args.gpus}: only {n} GPU(s) visible")
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        os.execvp(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
                                   "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:])
    if args.impl == "gc3" and world > 1:
        import torch
        if torch.cuda.device_count() < world:
            raise SystemExit(f"WORLD_SIZE={world} but only {torch.cuda.device_count()} GPU(s) visible")
        if 8 % world:
            raise SystemExit(f"--gpus {world} must divide the 8 IR ranks")


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
    ap.add_argument("--more", default="c3,c4", help="other configurations timed (device only) and verified at N=1")
    ap.add_argument("--no-more", action="store_true")
    ap.add_argument("--quick", action="store_true", help="kernel timing only: one compact JSON line")
    ap.add_argument("--sweep", action="store_true", help="message-size sweep (one JSON line per protocol and size)")
    ap.add_argument("--sweep-min", type=int, default=1 << 10)
    ap.add_argument("--sweep-max", type=int, default=1 << 30)
    ap.add_argument("--sweep-protos", default="simple,ll,ll128")
    ap.add_argument("--graph", action="store_true", help="sweep: also time collectives captured in a CUDA graph")
    ap.add_argument("--builtin", action="store_true",
                    help="sweep: register nothing, every size runs the runtime's built-in program (size tiers)")
    ap.add_argument("--graph-max", type=int, default=8 << 20)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if not args.sweep:
        enforce_world(args)
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
