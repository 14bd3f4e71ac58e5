"""N>1 host logic on CPU: two processes (torch.distributed, gloo) run the pieces of the
multi-process path that need no GPU — unique-id distribution, the /dev/shm bootstrap all-gather
that carries device records and CUDA IPC handles, and the per-rank arena layouts every process
computes for every peer (they must agree bit for bit, or a sender would write into the wrong FIFO).
Also: the planner's tile-group deadlock check against an independent simulation."""
import json
import os
import socket

import pytest

from conftest import golden_names, read_ir


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, names, out_q):
    import torch.distributed as dist
    from paper_2201_11840_b200 import gc3
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = [gc3.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        recs = gc3.bootstrap_exchange(uid[0], rank, world, f"rank{rank}:pid{os.getpid():010d}".encode())
        layouts = {}
        for name in names:
            ir = gc3.IR(read_ir(name))
            R = len(json.loads(read_ir(name))["gpus"])
            layouts[name] = [ir.arena_layout(r, 3, 2, 1 << 14) for r in range(R)]
        gathered = [None] * world
        dist.all_gather_object(gathered, layouts)
        out_q.put((rank, [r.decode() for r in recs], gathered[0] == gathered[1], os.getpid()))
    finally:
        dist.destroy_process_group()


def test_two_process_bootstrap_and_layouts(gc3lib):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    names = ["twostep_a2a_2x4", "hier_ar_2x4_par1", "ring_ar_8_ch8_inst4"]
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, names, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pids = {r: pid for r, _, _, pid in results}
    for rank, recs, same, _ in results:
        assert same, "arena layouts differ between processes"
        assert recs == [f"rank{r}:pid{pids[r]:010d}" for r in range(2)]


# -- independent restatement of the lane order used by the kernel (interp.cuh) ---------------
def simulate_order(irj, tiles, G, slots):
    """Greedy maximal run of every thread block's (group of G tiles, op-major) order with FIFO
    depth `slots`, atomic fused ops and deps keyed by (step, tile). True if it completes."""
    def order(nops):
        seq = []
        for g0 in range(0, tiles, G):
            gs = min(G, tiles - g0)
            for s in range(nops):
                for j in range(gs):
                    seq.append((s, g0 + j))
        return seq

    tbs = [(g["rank"], t, tb) for g in irj["gpus"] for t, tb in enumerate(g["threadblocks"])]
    seqs = {(r, t): order(len(tb["ops"])) for r, t, tb in tbs}
    done = {(r, t): set() for r, t, _ in tbs}
    pos = {(r, t): 0 for r, t, _ in tbs}
    idx = {(g["rank"], tb["id"]): t for g in irj["gpus"] for t, tb in enumerate(g["threadblocks"])}
    sent, used = {}, {}
    recvs = ("recv", "rrc", "rcs", "rrcs", "rrs")
    sends = ("send", "rcs", "rrcs", "rrs")
    progress = True
    while progress:
        progress = False
        for r, t, tb in tbs:
            while pos[(r, t)] < len(seqs[(r, t)]):
                s, tile = seqs[(r, t)][pos[(r, t)]]
                op = tb["ops"][s]
                ok = all((d["step"], tile) in done[(r, idx[(r, d["tb"])])] for d in op["deps"])
                cin = (tb["recv_peer"], r, tb["channel"])
                cout = (r, tb["send_peer"], tb["channel"])
                if ok and op["opcode"] in recvs and sent.get(cin, 0) <= used.get(cin, 0):
                    ok = False
                if ok and op["opcode"] in sends and sent.get(cout, 0) - used.get(cout, 0) >= slots:
                    ok = False
                if not ok:
                    break
                if op["opcode"] in recvs:
                    used[cin] = used.get(cin, 0) + 1
                if op["opcode"] in sends:
                    sent[cout] = sent.get(cout, 0) + 1
                done[(r, t)].add((s, tile))
                pos[(r, t)] += 1
                progress = True
    return all(pos[k] == len(seqs[k]) for k in pos)


@pytest.mark.parametrize("name", [n for n in golden_names() if not n.startswith("allpairs_ar_8")])
def test_order_check_matches_independent_simulation(gc3lib, name):
    irj = json.loads(read_ir(name))
    ir = gc3lib.IR(read_ir(name))
    for tiles, G, slots in [(1, 1, 1), (1, 1, 2), (4, 1, 2), (4, 2, 2), (4, 4, 2), (4, 4, 8), (5, 2, 3)]:
        assert ir.order_deadlock_free(tiles, G, slots) == simulate_order(irj, tiles, G, slots), (tiles, G, slots)


def test_tile_major_order_agrees_with_oracle_deadlocks(gc3lib):
    """G = 1 is the paper's tile-major loop: the planner check agrees with the oracle's
    randomized simulation (SURVEY.md Finding 1: s=1 deadlocks, s=2 does not)."""
    from test_oracle import S1_DEADLOCK, run_numeric
    for name in golden_names():
        ir = gc3lib.IR(read_ir(name))
        assert ir.order_deadlock_free(2, 1, 2), name
        rc, _, _ = run_numeric(name, "random", seed=1, slots=1, tile=12)  # 2 tiles of 12 elements
        assert ir.order_deadlock_free(2, 1, 1) == (rc == 0), name
        if name in S1_DEADLOCK:
            assert rc == 1
