"""Helpers for the GPU parity tests: run a collective through libgc3.so (loopback ranks on one
GPU) and through the CPU oracle on the same inputs, and compare bit for bit."""
import json

import numpy as np
import torch

from oracle.oracle import collective

TORCH_DT = {"float32": torch.float32, "bfloat16": torch.bfloat16, "float16": torch.float16, "int32": torch.int32,
            "float64": torch.float64, "int64": torch.int64, "uint8": torch.uint8, "int8": torch.int8,
            "uint32": torch.uint32, "uint64": torch.uint64}
NP_VIEW = {"float32": np.uint32, "bfloat16": np.uint16, "float16": np.uint16, "int32": np.uint32, "float64": np.uint64,
           "int64": np.uint64, "uint8": np.uint8, "int8": np.uint8, "uint32": np.uint32, "uint64": np.uint64}


def make_input(n, dtype, seed, device="cuda"):
    """Seeded synthetic data: floats N(0,1) (RNE-rounded for 16-bit types), ints uniform."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    if dtype in ("float32", "float64", "float16", "bfloat16"):
        t = torch.randn(n, generator=g, dtype=torch.float32).to(TORCH_DT[dtype])
    elif dtype in ("int32", "int64", "int8"):
        lo, hi = (-(2 ** 20), 2 ** 20) if dtype != "int8" else (-128, 128)
        t = torch.randint(lo, hi, (n,), generator=g, dtype=torch.int64).to(TORCH_DT[dtype])
    else:
        hi = {"uint8": 256, "uint32": 2 ** 31, "uint64": 2 ** 40}[dtype]
        t = torch.randint(0, hi, (n,), generator=g, dtype=torch.int64).to(TORCH_DT[dtype])
    return t.to(device)


def to_np_bits(t, dtype):
    t = t.detach().cpu().contiguous()
    if t.dtype in (torch.bfloat16, torch.float16):
        return t.view(torch.int16).numpy().view(np.uint16).copy()
    if t.dtype == torch.uint32:
        return t.view(torch.int32).numpy().view(np.uint32).copy()
    if t.dtype == torch.uint64:
        return t.view(torch.int64).numpy().view(np.uint64).copy()
    return t.numpy().copy()


def oracle_collective(ir_json, coll, inputs, count, dtype, op="sum"):
    """Expected recvbuffs (numpy, raw bits) of every rank from the CPU oracle."""
    odt = {"bfloat16": 9, "float16": 6}.get(dtype, dtype)
    return collective(json.loads(ir_json) if isinstance(ir_json, str) else ir_json, coll,
                      [to_np_bits(x, dtype) for x in inputs], count, odt, op)


def run_collective(comms, coll, inputs, count, dtype, op="sum", inplace=False, stream=None, nranks=None, first_rank=0):
    """Issues one grouped collective over the comms (ranks first_rank.. of an nranks-rank clique,
    all of it by default); returns the recv tensors."""
    from paper_2201_11840_b200 import gc3
    R = nranks or len(comms)
    tdt = TORCH_DT[dtype]
    outs = []
    with gc3.group():
        for k, c in enumerate(comms):
            r = first_rank + k
            x = inputs[k]
            if coll == "allreduce":
                recv = x if inplace else torch.empty(count, dtype=tdt, device=x.device)
                c.all_reduce(x, recv, count, dtype, op, stream)
            elif coll == "allgather":
                if inplace:
                    recv = torch.zeros(R * count, dtype=tdt, device=x.device)
                    recv[r * count:(r + 1) * count].copy_(x)
                    send = recv[r * count:(r + 1) * count]
                else:
                    recv, send = torch.empty(R * count, dtype=tdt, device=x.device), x
                c.all_gather(send, recv, count, dtype, stream)
            elif coll == "reducescatter":
                recv = x[r * count:(r + 1) * count] if inplace else torch.empty(count, dtype=tdt, device=x.device)
                c.reduce_scatter(x, recv, count, dtype, op, stream)
            elif coll == "alltoall":
                recv = torch.empty(R * count, dtype=tdt, device=x.device)
                c.all_to_all(x, recv, count, dtype, stream)
            outs.append(recv)
    return outs


def input_len(coll, count, R):
    return count if coll in ("allreduce", "allgather") else R * count
