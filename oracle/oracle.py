"""Python binding of the CPU oracle (gc3_oracle.c).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may import
this module, and only as the checker or the timed CPU baseline.  The IR is flattened here with
Python's json module, independently of the product's C++ loader.
"""
import ctypes
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")

OPCODES = {"send": 0, "recv": 1, "copy": 2, "reduce": 3, "rrc": 4, "rcs": 5, "rrcs": 6, "rrs": 7, "nop": 8}
BUFS = {"input": 0, "output": 1, "scratch": 2}
DTYPES = {  # ncclDataType_t -> numpy
    0: np.int8, 1: np.uint8, 2: np.int32, 3: np.uint32, 4: np.int64, 5: np.uint64,
    6: np.float16, 7: np.float32, 8: np.float64, 9: np.uint16,  # bf16 carried as raw uint16
}
NCCL_DTYPE = {"int8": 0, "uint8": 1, "int32": 2, "uint32": 3, "int64": 4, "uint64": 5,
              "float16": 6, "float32": 7, "float64": 8, "bfloat16": 9}
REDOPS = {"sum": 0, "prod": 1, "max": 2, "min": 3}
MODES = {"deterministic": 0, "random": 1, "threaded": 2}
MAX_DEPS = 8


class Op(ctypes.Structure):
    _fields_ = [("opcode", ctypes.c_int32), ("src_buf", ctypes.c_int32), ("src_off", ctypes.c_int32),
                ("dst_buf", ctypes.c_int32), ("dst_off", ctypes.c_int32), ("count", ctypes.c_int32),
                ("has_dep", ctypes.c_int32), ("ndeps", ctypes.c_int32),
                ("dep_tb", ctypes.c_int32 * MAX_DEPS), ("dep_step", ctypes.c_int32 * MAX_DEPS)]


class Tb(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("send_peer", ctypes.c_int32), ("recv_peer", ctypes.c_int32),
                ("channel", ctypes.c_int32), ("first_op", ctypes.c_int32), ("nops", ctypes.c_int32)]


class Program(ctypes.Structure):
    _fields_ = [("nranks", ctypes.c_int32), ("ntbs", ctypes.c_int32), ("tbs", ctypes.POINTER(Tb)),
                ("ops", ctypes.POINTER(Op)), ("nchunks", ctypes.c_int32 * 3), ("inplace", ctypes.c_int32)]


class Race(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int32) for k in ("rank", "buf", "index", "kind", "tb_a", "step_a", "tb_b", "step_b")]


RACE_KINDS = ("write/write", "write/read", "read/write")

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            import subprocess
            subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-o", LIB,
                                   os.path.join(HERE, "gc3_oracle.c")])
        _lib = ctypes.CDLL(LIB)
        _lib.gc3o_run.argtypes = [ctypes.POINTER(Program), ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t,
                                  ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
                                  ctypes.c_size_t, ctypes.c_char_p, ctypes.c_size_t]
        _lib.gc3o_run.restype = ctypes.c_int
        _lib.gc3o_reduce.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int]
        _lib.gc3o_reduce.restype = ctypes.c_int
        _lib.gc3o_races.argtypes = [ctypes.POINTER(Program), ctypes.POINTER(Race), ctypes.c_int, ctypes.c_char_p,
                                    ctypes.c_size_t]
        _lib.gc3o_races.restype = ctypes.c_int
    return _lib


class FlatIR:
    """An IR flattened into the oracle's C structures (independent of the product loader)."""

    def __init__(self, ir):
        if isinstance(ir, str):
            ir = json.loads(open(ir).read() if not ir.lstrip().startswith("{") else ir)
        self.json = ir
        self.nranks = len(ir["gpus"])
        self.nchunks = (ir["nchunks"]["input"], ir["nchunks"]["output"], ir["nchunks"]["scratch"])
        self.inplace = bool(ir["inplace"])
        tbs, ops = [], []
        for g in ir["gpus"]:
            ids = {tb["id"]: k for k, tb in enumerate(g["threadblocks"])}
            for tb in g["threadblocks"]:
                first = len(ops)
                for o in tb["ops"]:
                    op = Op(OPCODES[o["opcode"]], BUFS[o["src_buf"]], o["src_off"], BUFS[o["dst_buf"]],
                            o["dst_off"], o["count"], int(o["has_dep"]), len(o["deps"]))
                    if len(o["deps"]) > MAX_DEPS:
                        raise ValueError("too many deps for the oracle")
                    for k, d in enumerate(o["deps"]):
                        op.dep_tb[k] = ids[d["tb"]]
                        op.dep_step[k] = d["step"]
                    ops.append(op)
                tbs.append(Tb(g["rank"], tb["send_peer"], tb["recv_peer"], tb["channel"], first, len(tb["ops"])))
        self._tbs = (Tb * max(1, len(tbs)))(*tbs)
        self._ops = (Op * max(1, len(ops)))(*ops)
        self.prog = Program(self.nranks, len(tbs), self._tbs, self._ops, (ctypes.c_int32 * 3)(*self.nchunks),
                            int(self.inplace))

    def run(self, bufs, chunk_elems, dtype, redop="sum", mode="deterministic", seed=0, slots=2, tile_elems=0):
        """bufs: per rank [input, output, scratch] numpy arrays (output may be input when in place).
        Executes in place; returns (rc, error message)."""
        arr = (ctypes.c_void_p * (3 * self.nranks))()
        keep = []
        for r in range(self.nranks):
            for b in range(3):
                a = bufs[r][b]
                if a is None:
                    a = np.zeros(1, dtype=np.uint8)
                assert a.flags["C_CONTIGUOUS"]
                keep.append(a)
                arr[3 * r + b] = a.ctypes.data
        dt = NCCL_DTYPE[dtype] if isinstance(dtype, str) else dtype
        op = REDOPS[redop] if isinstance(redop, str) else redop
        err = ctypes.create_string_buffer(512)
        rc = lib().gc3o_run(ctypes.byref(self.prog), arr, chunk_elems, dt, op, MODES[mode], seed, slots, tile_elems,
                            err, 512)
        return rc, err.value.decode()

    def races(self, max_pairs=64):
        """Vector-clock race detection (gc3o_races): a list of dicts naming each conflicting pair of
        accesses to one (rank, buffer, chunk) slot, unordered by happens-before. Raises ValueError
        for a malformed or deadlocking program."""
        out = (Race * max_pairs)()
        err = ctypes.create_string_buffer(512)
        n = lib().gc3o_races(ctypes.byref(self.prog), out, max_pairs, err, 512)
        if n < 0:
            raise ValueError(err.value.decode())
        names = {v: k for k, v in BUFS.items()}
        res = []
        for r in out[:min(n, max_pairs)]:
            res.append({"rank": r.rank, "buf": names[r.buf], "index": r.index, "kind": RACE_KINDS[r.kind],
                        "a": (r.tb_a, r.step_a), "b": (r.tb_b, r.step_b)})
        return res if n <= max_pairs else res + [{"truncated": n}]


def reduce_arrays(a, b, dtype, redop="sum"):
    """a = a (op) b with the oracle arithmetic (returns a new array)."""
    out = np.array(a, copy=True)
    dt = NCCL_DTYPE[dtype] if isinstance(dtype, str) else dtype
    rc = lib().gc3o_reduce(out.ctypes.data, np.ascontiguousarray(b).ctypes.data, out.size, dt,
                           REDOPS[redop] if isinstance(redop, str) else redop)
    assert rc == 0
    return out


def collective(ir, coll, arrays, count, dtype, redop="sum", **run_kw):
    """NCCL-level oracle: the recvbuff of every rank after `coll` over `count` (NCCL's count
    argument) with the IR, from per-rank sendbuff arrays (numpy, raw bits).

    Buffer mapping: AllReduce / ReduceScatter run the in-place IR on the send
    data (ReduceScatter returns the rank's owned block); AllGather and AlltoAll map IR input/output
    to sendbuff/recvbuff.  A rank block (AllReduce: count; AllGather: sendcount; ReduceScatter:
    recvcount; AlltoAll: count per peer) is cut into the IR's c chunks per block of
    ce = ceil(count / c) elements; when c does not divide count the last chunks are clipped:
    element p of a block is element p % ce of chunk p // ce (each block padded to c * ce here;
    ops map chunk position x to position x, so padding never mixes into real elements).
    """
    if not isinstance(ir, FlatIR):
        ir = FlatIR(ir)
    R, (nin, nout, nsc) = ir.nranks, ir.nchunks
    c = nin if coll in ("allreduce", "allgather") else nin // R
    ce = -(-count // c) if count else 0
    pb = c * ce
    nblk = 1 if coll in ("allreduce", "allgather") else R

    def pad(a):
        out = np.zeros(nblk * pb, dtype=a.dtype)
        for b in range(nblk):
            out[b * pb:b * pb + count] = a[b * count:(b + 1) * count]
        return out

    def unpad(a, blocks):
        return np.concatenate([a[b * pb:b * pb + count] for b in range(blocks)]) if blocks else a[:0]

    bufs = []
    for r in range(R):
        inp = pad(np.ascontiguousarray(arrays[r]))
        out = inp if ir.inplace else np.zeros(max(nout, 1) * ce, dtype=inp.dtype)
        sc = np.zeros(max(nsc, 1) * ce, dtype=inp.dtype)
        bufs.append([inp, out, sc])
    if count:
        rc, err = ir.run(bufs, ce, dtype, redop, **run_kw)
        if rc != 0:
            raise RuntimeError(err)
    if coll == "reducescatter":
        return [bufs[r][0][r * pb:r * pb + count].copy() for r in range(R)]
    if coll == "allreduce":
        return [unpad(bufs[r][0], 1) for r in range(R)]
    return [unpad(bufs[r][1], R) for r in range(R)]
