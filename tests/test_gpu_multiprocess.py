"""The multi-process path on one B200: two processes host four ranks each (ncclCommInitRank inside
a group, /dev/shm bootstrap, CUDA IPC arenas). Messages between the processes travel the way the
N-GPU runs move them: direct writes into and pulled reads from the peer process's registered user
buffers (per-call buffer exchange, remote=1, the default) or the receiver-resident FIFOs (remote=0,
and every LL message); bulk copies stay on because both processes drive the same GPU. Results must
be bit-exact vs the oracle, and the plan must show the transports it claims."""
import json
import os
import socket

import numpy as np
import pytest

from conftest import ir_path, read_ir

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(proc, nproc, port, name, coll, count, dtype, proto, q, remote=1, force_sys=0):
    import torch.distributed as dist
    from paper_2201_11840_b200 import gc3
    from gpu_util import input_len, make_input, oracle_collective, run_collective, to_np_bits
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=proc, world_size=nproc)
    try:
        torch.cuda.set_device(0)
        irj = json.loads(read_ir(name))
        R = len(irj["gpus"])
        per = R // nproc
        uid = [gc3.get_unique_id() if proc == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        with gc3.group():
            comms = [gc3.init_rank(R, uid[0], proc * per + k) for k in range(per)]
        for c in comms:
            c.set_config("remote", remote)
            c.set_config("force_sys", force_sys)
            c.set_config("tma_min", 4096)  # these small calls take the bulk-copy paths too
            i = c.register_ir(ir_path(name))
            if proto:
                c.set_protocol(i, proto)
        inputs = [make_input(input_len(coll, count, R), dtype, 90 + r) for r in range(R)]
        expected = oracle_collective(irj, coll, [x.clone() for x in inputs], count, dtype)
        mine = [inputs[proc * per + k] for k in range(per)]
        ok, why = True, []
        for it in range(2):
            outs = run_collective(comms, coll, [x.clone() for x in mine], count, dtype, nranks=R, first_rank=proc * per)
            torch.cuda.synchronize()
            err = comms[0].async_error()
            if err[0] != 0:
                ok = False
                why.append(f"it {it}: async error {err}")
            for k in range(per):
                r = proc * per + k
                got, exp = to_np_bits(outs[k], dtype), expected[r]
                if not np.array_equal(got, exp):
                    ok = False
                    bad = np.nonzero(got != exp)[0]
                    why.append(f"it {it} rank {r}: {bad.size} mismatches, first {bad[:6].tolist()}")
            dist.barrier()
        info = comms[0].query_plan(coll, count, dtype)
        for c in comms:
            c.destroy()
        q.put((proc, ok, "; ".join(why), info))
    except Exception as e:  # reported to the parent
        q.put((proc, False, repr(e), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,coll,count,dtype,proto", [
    ("ring_ar_8_ch1", "allreduce", 8 * 40000, "float32", None),
    ("twostep_a2a_2x4", "alltoall", 30000, "bfloat16", None),
    ("ring_rs_8", "reducescatter", 20000, "int32", None),
    ("hier_ar_2x4_par1", "allreduce", 8 * 30000, "bfloat16", None),
    ("ring_ag_8", "allgather", 25000, "float32", None),
    # LL lines across processes, and a ragged count (padded chunks)
    ("ring_ar_8_ch1", "allreduce", 8 * 5000, "float32", "ll"),
    ("twostep_a2a_2x4", "alltoall", 7000, "float16", "ll"),
    ("ring_ar_8_ch1", "allreduce", 8 * 40000 + 13, "float32", None)])
@pytest.mark.parametrize("remote", [1, 0])
def test_two_processes_share_a_gpu(name, coll, count, dtype, proto, remote):
    results = _run(name, coll, count, dtype, proto, remote)
    for proc, ok, err, info in results:
        assert ok, (proc, err)
        assert info["local_ranks"] == 4 and info["sys_scope"] == 0, info  # one GPU: .gpu scope everywhere
        if proto is None:
            assert info["tma_stages"] > 0, info  # bulk copies across the process boundary too
            # direct / pulled messages across the process boundary exactly when remote transports are on
            assert (info["remote_messages"] > 0) == bool(remote), info


def _run(name, coll, count, dtype, proto, remote, force_sys=0):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(p, 2, port, name, coll, count, dtype, proto, q, remote, force_sys)) for p in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    return results


@pytest.mark.parametrize("name,coll,count,dtype,proto", [
    ("ring_ar_8_ch1", "allreduce", 8 * 40000, "float32", None),
    ("hier_ar_2x4_par1", "allreduce", 8 * 30000, "bfloat16", None),
    ("twostep_a2a_2x4", "alltoall", 30000, "float32", None),
    ("ring_rs_8", "reducescatter", 20000, "int32", "ll128")])
def test_two_processes_with_cross_gpu_code_path(name, coll, count, dtype, proto):
    """The N-GPU code path on one GPU (config force_sys): thread blocks with a connection to the
    other process use .sys-scope fences, flags and lines and the register path (no bulk copies),
    while direct / pulled messages still cross the process boundary; bit-exact vs the oracle."""
    for proc, ok, err, info in _run(name, coll, count, dtype, proto, 1, force_sys=1):
        assert ok, (proc, err)
        assert info["sys_scope"] == 1, info
        if proto is None:
            assert info["remote_messages"] > 0, info
