"""ctypes bindings of libgc3.so (include/gc3.h).

Mirrors the NCCL entry points the GC3 paper's runtime exposes plus the GC3
extensions, with NCCL's argument meaning and error behaviour: every call returns ncclResult_t and
a non-zero result raises NcclError carrying ncclGetLastError().
"""
import contextlib
import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GC3_LIB_PATH", os.path.join(PKG, "libgc3.so"))

# ncclDataType_t (nccl.h:278-290) keyed by torch dtype name
NCCL_DTYPES = {
    "int8": 0, "uint8": 1, "int32": 2, "uint32": 3, "int64": 4, "uint64": 5,
    "float16": 6, "float32": 7, "float64": 8, "bfloat16": 9,
}
REDOPS = {"sum": 0, "prod": 1, "max": 2, "min": 3}
COLLS = {"allreduce": 0, "allgather": 1, "reducescatter": 2, "alltoall": 3}


def coll_id(name):
    return COLLS[name]


class NcclError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"ncclResult {code}: {msg}")
        self.code = code


class SimConfig(ctypes.Structure):
    _fields_ = [("nranks_gpu", ctypes.c_int), ("rank_gpu", ctypes.POINTER(ctypes.c_int)), ("gpus_per_node", ctypes.c_int),
                ("alpha_us", ctypes.c_double * 3), ("gbps", ctypes.c_double * 3), ("gamma_gbps", ctypes.c_double),
                ("copy_gbps", ctypes.c_double), ("protocol", ctypes.c_int), ("slots", ctypes.c_int),
                ("chunk_bytes", ctypes.c_int64), ("tile_bytes", ctypes.c_int64), ("launch_us", ctypes.c_double),
                ("hbm_gbps", ctypes.c_double), ("lanes", ctypes.c_int), ("group", ctypes.c_int),
                ("op_us", ctypes.c_double), ("msg_read_passes", ctypes.c_int), ("workers", ctypes.c_int)]


class SimReport(ctypes.Structure):
    _fields_ = [("completed", ctypes.c_int), ("makespan_us", ctypes.c_double), ("util", ctypes.c_double * 3),
                ("messages", ctypes.c_int64), ("tiles", ctypes.c_int64), ("deadlock", ctypes.c_char * 256)]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("ir_id", ctypes.c_int), ("protocol", ctypes.c_int), ("lanes", ctypes.c_int), ("grid", ctypes.c_int),
        ("local_ranks", ctypes.c_int), ("slots", ctypes.c_int),
        ("chunk_elems", ctypes.c_int64), ("tile_elems", ctypes.c_int64), ("ntiles", ctypes.c_int64),
        ("slot_bytes", ctypes.c_int64), ("wire_bytes", ctypes.c_int64), ("hbm_bytes", ctypes.c_int64),
        ("name", ctypes.c_char * 64), ("unit_warps", ctypes.c_int), ("group", ctypes.c_int),
        ("mode", ctypes.c_int), ("mail_messages", ctypes.c_int), ("remote_messages", ctypes.c_int),
        ("sys_scope", ctypes.c_int), ("tma_stages", ctypes.c_int),
    ]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["name"] = self.name.decode()
        return d


class UniqueId(ctypes.Structure):
    _fields_ = [("internal", ctypes.c_char * 128)]


_lib = None


def lib():
    """Loads libgc3.so (never a fallback: a missing library is an error)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2201_11840_b200.build`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i, sz, cp = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_char_p
    sigs = {
        "ncclGetVersion": [ctypes.POINTER(i)],
        "ncclGetUniqueId": [ctypes.POINTER(UniqueId)],
        "ncclCommInitRank": [ctypes.POINTER(vp), i, UniqueId, i],
        "ncclCommInitAll": [ctypes.POINTER(vp), i, ctypes.POINTER(i)],
        "ncclCommDestroy": [vp],
        "ncclCommAbort": [vp],
        "ncclCommGetAsyncError": [vp, ctypes.POINTER(i)],
        "ncclCommCount": [vp, ctypes.POINTER(i)],
        "ncclCommCuDevice": [vp, ctypes.POINTER(i)],
        "ncclCommUserRank": [vp, ctypes.POINTER(i)],
        "ncclAllReduce": [vp, vp, sz, i, i, vp, vp],
        "ncclReduceScatter": [vp, vp, sz, i, i, vp, vp],
        "ncclAllGather": [vp, vp, sz, i, vp, vp],
        "ncclAlltoAll": [vp, vp, sz, i, vp, vp],
        "ncclAllToAll": [vp, vp, sz, i, vp, vp],
        "ncclGroupStart": [],
        "ncclGroupEnd": [],
        "gc3RegisterIR": [vp, cp, i, ctypes.POINTER(i)],
        "gc3SetProtocolOverride": [vp, i, i],
        "gc3QueryPlan": [vp, i, sz, i, ctypes.POINTER(PlanInfo)],
        "gc3SetConfig": [vp, cp, ctypes.c_int64],
        "gc3GetTrace": [vp, ctypes.c_void_p, sz, ctypes.POINTER(i), ctypes.POINTER(i), ctypes.POINTER(i)],
        "gc3IrParse": [cp, ctypes.POINTER(vp), ctypes.POINTER(vp)],
        "gc3IrSerialize": [vp, ctypes.POINTER(vp)],
        "gc3IrParseXml": [cp, i, ctypes.POINTER(vp), ctypes.POINTER(vp)],
        "gc3IrToXml": [vp, ctypes.POINTER(vp)],
        "gc3IrLaneMultipliers": [vp, ctypes.POINTER(vp)],
        "gc3IrSourceReads": [vp, ctypes.POINTER(i), ctypes.POINTER(vp)],
        "gc3IrResultWrites": [vp, ctypes.POINTER(i), ctypes.POINTER(vp)],
        "gc3IrBuiltin": [cp, i, ctypes.POINTER(vp)],
        "gc3IrGenerate": [cp, cp, i, i, i, ctypes.POINTER(vp)],
        "gc3IrBuiltinSized": [cp, i, ctypes.c_uint64, ctypes.POINTER(vp)],
        "gc3IrPredict": [vp, ctypes.c_int64, i, i, ctypes.POINTER(ctypes.c_double)],
        "gc3SimDefaults": [ctypes.POINTER(SimConfig)],
        "gc3IrSimulate": [vp, ctypes.POINTER(SimConfig), ctypes.POINTER(SimReport)],
        "gc3IrSweep": [vp, ctypes.POINTER(SimConfig), ctypes.POINTER(ctypes.c_int64), i, ctypes.c_int64, ctypes.POINTER(vp)],
        "gc3IrValidate": [vp, i, i, i, i, ctypes.POINTER(vp)],
        "gc3IrCheckSlots": [vp, i, ctypes.POINTER(vp)],
        "gc3IrReplicate": [vp, i, ctypes.POINTER(vp)],
        "gc3IrFree": [vp],
        "gc3IrArenaLayout": [vp, i, i, i, ctypes.c_int64, ctypes.POINTER(vp)],
        "gc3IrDirectMessages": [vp, ctypes.POINTER(vp)],
        "gc3IrOrderCheck": [vp, ctypes.c_int64, i, i, ctypes.POINTER(i)],
        "gc3BootstrapExchange": [ctypes.POINTER(UniqueId), i, i, vp, sz, vp, i],
    }
    for name, args in sigs.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.ncclGetErrorString.argtypes = [i]
    L.ncclGetErrorString.restype = cp
    L.ncclGetLastError.argtypes = [vp]
    L.ncclGetLastError.restype = cp
    L.gc3Free.argtypes = [vp]
    L.gc3Free.restype = None
    _lib = L
    return L


def check(rc, comm=None):
    if rc != 0:
        L = lib()
        raise NcclError(rc, f"{L.ncclGetErrorString(rc).decode()}: {L.ncclGetLastError(comm).decode()}")


def _take(p):
    s = ctypes.string_at(p).decode() if p else ""
    if p:
        lib().gc3Free(p)
    return s


# ---------------------------------------------------------------------------- IR library
class IR:
    """Host-only handle on a parsed GC3-IR (reference ir.hpp semantics)."""

    def __init__(self, text):
        L = lib()
        h, err = ctypes.c_void_p(), ctypes.c_void_p()
        rc = L.gc3IrParse(text.encode() if isinstance(text, str) else text, ctypes.byref(h), ctypes.byref(err))
        if rc != 0:
            path, _, msg = _take(err.value).partition("\t")
            e = NcclError(rc, f"schema: {path}: {msg}")
            e.path, e.message = path, msg
            raise e
        self._h = h

    @classmethod
    def builtin(cls, collective, nranks, nbytes=None):
        """The runtime's built-in program for `collective` on nranks ranks; with nbytes (per-rank
        buffer bytes) the one a call of that size runs (AllReduce size tiers)."""
        h = ctypes.c_void_p()
        if nbytes is None:
            check(lib().gc3IrBuiltin(collective.encode(), nranks, ctypes.byref(h)))
        else:
            check(lib().gc3IrBuiltinSized(collective.encode(), nranks, nbytes, ctypes.byref(h)))
        return cls._wrap(h)

    @classmethod
    def generate(cls, algo, collective, nranks, channels=1, instances=1):
        """A program generated at communicator time: algo "ring" / "allpairs" / "direct" with
        `channels` rings and `instances` instances (gc3IrGenerate)."""
        h = ctypes.c_void_p()
        check(lib().gc3IrGenerate(algo.encode(), collective.encode(), nranks, channels, instances, ctypes.byref(h)))
        return cls._wrap(h)

    @classmethod
    def from_xml(cls, text, fold_nops=True):
        """An MSCCL algorithm XML file's text as a program (msccl_xml.hpp)."""
        h, err = ctypes.c_void_p(), ctypes.c_void_p()
        rc = lib().gc3IrParseXml(text.encode() if isinstance(text, str) else text, int(fold_nops), ctypes.byref(h),
                                 ctypes.byref(err))
        if rc != 0:
            raise NcclError(rc, _take(err.value))
        return cls._wrap(h)

    def to_xml(self):
        out = ctypes.c_void_p()
        check(lib().gc3IrToXml(self._h, ctypes.byref(out)))
        return _take(out.value)

    @classmethod
    def _wrap(cls, h):
        obj = cls.__new__(cls)
        obj._h = h
        return obj

    def serialize(self):
        out = ctypes.c_void_p()
        check(lib().gc3IrSerialize(self._h, ctypes.byref(out)))
        return _take(out.value)

    def validate(self, nodes, gpus_per_node, max_threadblocks=0, max_channels=0):
        out = ctypes.c_void_p()
        check(lib().gc3IrValidate(self._h, nodes, gpus_per_node, max_threadblocks, max_channels, ctypes.byref(out)))
        return [x for x in _take(out.value).split("\n") if x]

    def check_slots(self, slots):
        out = ctypes.c_void_p()
        check(lib().gc3IrCheckSlots(self._h, slots, ctypes.byref(out)))
        return [x for x in _take(out.value).split("\n") if x]

    def replicate(self, instances):
        out = ctypes.c_void_p()
        check(lib().gc3IrReplicate(self._h, instances, ctypes.byref(out)))
        return IR._wrap(out)

    def arena_layout(self, rank, lanes, slots, slot_unit):
        import json
        out = ctypes.c_void_p()
        check(lib().gc3IrArenaLayout(self._h, rank, lanes, slots, slot_unit, ctypes.byref(out)))
        return json.loads(_take(out.value))

    def direct_messages(self):
        import json
        out = ctypes.c_void_p()
        check(lib().gc3IrDirectMessages(self._h, ctypes.byref(out)))
        return json.loads(_take(out.value))

    def source_reads(self):
        """(complete, flags[rank][tb][step]) of the const-source analysis."""
        import json
        out, comp = ctypes.c_void_p(), ctypes.c_int()
        check(lib().gc3IrSourceReads(self._h, ctypes.byref(comp), ctypes.byref(out)))
        return bool(comp.value), json.loads(_take(out.value))

    def result_writes(self):
        """(complete, flags[rank][tb][step]) of the ReduceScatter result-buffer analysis."""
        import json
        out, comp = ctypes.c_void_p(), ctypes.c_int()
        check(lib().gc3IrResultWrites(self._h, ctypes.byref(comp), ctypes.byref(out)))
        return bool(comp.value), json.loads(_take(out.value))

    def predict_us(self, chunk_bytes, protocol="simple", lanes=1):
        """Timed-model prediction of one launch (microseconds)."""
        out = ctypes.c_double()
        check(lib().gc3IrPredict(self._h, chunk_bytes, {"simple": 0, "ll": 1}.get(protocol, protocol), lanes,
                                 ctypes.byref(out)))
        return out.value

    @staticmethod
    def _sim_config(rank_gpu=None, protocol="simple", **kw):
        cfg = SimConfig()
        check(lib().gc3SimDefaults(ctypes.byref(cfg)))
        keep = None
        if rank_gpu is not None:
            keep = (ctypes.c_int * len(rank_gpu))(*rank_gpu)
            cfg.nranks_gpu, cfg.rank_gpu = len(rank_gpu), keep
        cfg.protocol = {"simple": 0, "ll": 1, "ll128": 2}.get(protocol, protocol)
        names = {f[0] for f in SimConfig._fields_}
        for k, v in kw.items():
            if k not in names:
                raise TypeError(f"unknown simulator parameter {k!r}")
            if k in ("alpha_us", "gbps"):
                for j, x in enumerate(v):
                    getattr(cfg, k)[j] = x
            else:
                setattr(cfg, k, v)
        return cfg, keep

    def simulate(self, chunk_bytes, tile_bytes=0, **kw):
        """Timed simulation (gc3IrSimulate): dict with completed, makespan_us, util (per link class),
        messages, tiles, deadlock. kw: rank_gpu, protocol, alpha_us, gbps, gamma_gbps, copy_gbps,
        slots, gpus_per_node, launch_us, hbm_gbps, op_us, msg_read_passes, lanes, group, workers
        (> 0: the dataflow executor with that many units)."""
        cfg, keep = self._sim_config(chunk_bytes=chunk_bytes, tile_bytes=tile_bytes, **kw)
        rep = SimReport()
        check(lib().gc3IrSimulate(self._h, ctypes.byref(cfg), ctypes.byref(rep)))
        del keep
        return {"completed": bool(rep.completed), "makespan_us": rep.makespan_us, "util": list(rep.util),
                "messages": rep.messages, "tiles": rep.tiles, "deadlock": rep.deadlock.decode()}

    def sweep(self, sizes, tile_bytes=0, **kw):
        """CSV rows size_bytes,makespan_us,util_intra,util_inter, one timed run per size (gc3IrSweep)."""
        cfg, keep = self._sim_config(**kw)
        arr = (ctypes.c_int64 * max(1, len(sizes)))(*sizes)
        out = ctypes.c_void_p()
        check(lib().gc3IrSweep(self._h, ctypes.byref(cfg), arr, len(sizes), tile_bytes, ctypes.byref(out)))
        del keep
        return _take(out.value)

    def lane_multipliers(self):
        import json
        out = ctypes.c_void_p()
        check(lib().gc3IrLaneMultipliers(self._h, ctypes.byref(out)))
        return json.loads(_take(out.value))

    def order_deadlock_free(self, tiles, group, slots):
        ok = ctypes.c_int()
        check(lib().gc3IrOrderCheck(self._h, tiles, group, slots, ctypes.byref(ok)))
        return bool(ok.value)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.gc3IrFree(self._h)
            self._h = None


# ---------------------------------------------------------------------------- communicators
def _ptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _stream(s):
    if s is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return s if isinstance(s, int) else s.cuda_stream


class Comm:
    """One rank (ncclComm_t)."""

    def __init__(self, handle):
        self.h = ctypes.c_void_p(handle)
        n, r, d = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        L = lib()
        check(L.ncclCommCount(self.h, ctypes.byref(n)))
        check(L.ncclCommUserRank(self.h, ctypes.byref(r)))
        check(L.ncclCommCuDevice(self.h, ctypes.byref(d)))
        self.nranks, self.rank, self.device = n.value, r.value, d.value

    def register_ir(self, path_or_json, instances=1):
        out = ctypes.c_int()
        check(lib().gc3RegisterIR(self.h, path_or_json.encode(), instances, ctypes.byref(out)), self.h)
        return out.value

    def set_protocol(self, ir_id, proto):
        check(lib().gc3SetProtocolOverride(self.h, ir_id, {None: -1, "simple": 0, "ll": 1, "ll128": 2}.get(proto, proto)), self.h)

    def set_config(self, key, value):
        check(lib().gc3SetConfig(self.h, key.encode(), int(value)), self.h)

    def query_plan(self, coll, count, dtype):
        info = PlanInfo()
        check(lib().gc3QueryPlan(self.h, COLLS[coll], count, NCCL_DTYPES[dtype], ctypes.byref(info)), self.h)
        return info.as_dict()

    def trace(self):
        """Event log of the last traced launch: (numpy [grid, ops, 4] uint64 ns, lanes)."""
        import numpy as np
        g, o, ln = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        check(lib().gc3GetTrace(self.h, None, 0, ctypes.byref(g), ctypes.byref(o), ctypes.byref(ln)), self.h)
        buf = np.zeros(g.value * o.value * 4, dtype=np.uint64)
        check(lib().gc3GetTrace(self.h, buf.ctypes.data, buf.size, ctypes.byref(g), ctypes.byref(o), ctypes.byref(ln)), self.h)
        return buf.reshape(g.value, o.value, 4), ln.value

    def async_error(self):
        e = ctypes.c_int()
        check(lib().ncclCommGetAsyncError(self.h, ctypes.byref(e)))
        return e.value, lib().ncclGetLastError(self.h).decode()

    # collectives: buffers are torch tensors (or raw device pointers), dtype a torch dtype name
    def all_reduce(self, send, recv, count, dtype, op="sum", stream=None):
        check(lib().ncclAllReduce(_ptr(send), _ptr(recv), count, NCCL_DTYPES[dtype], REDOPS[op], self.h, _stream(stream)), self.h)

    def reduce_scatter(self, send, recv, recvcount, dtype, op="sum", stream=None):
        check(lib().ncclReduceScatter(_ptr(send), _ptr(recv), recvcount, NCCL_DTYPES[dtype], REDOPS[op], self.h, _stream(stream)), self.h)

    def all_gather(self, send, recv, sendcount, dtype, stream=None):
        check(lib().ncclAllGather(_ptr(send), _ptr(recv), sendcount, NCCL_DTYPES[dtype], self.h, _stream(stream)), self.h)

    def all_to_all(self, send, recv, count, dtype, stream=None):
        check(lib().ncclAlltoAll(_ptr(send), _ptr(recv), count, NCCL_DTYPES[dtype], self.h, _stream(stream)), self.h)

    def destroy(self):
        if self.h:
            check(lib().ncclCommDestroy(self.h))
            self.h = None

    def abort(self):
        """ncclCommAbort: raises the device abort flag (spinning blocks exit) and frees the comm."""
        if self.h:
            check(lib().ncclCommAbort(self.h))
            self.h = None


@contextlib.contextmanager
def group():
    L = lib()
    check(L.ncclGroupStart())
    try:
        yield
    finally:
        check(L.ncclGroupEnd())


def init_all(devices):
    """ncclCommInitAll; repeating a device creates loopback ranks that share it."""
    n = len(devices)
    arr = (ctypes.c_void_p * n)()
    devs = (ctypes.c_int * n)(*devices)
    check(lib().ncclCommInitAll(arr, n, devs))
    return [Comm(arr[k]) for k in range(n)]


def get_unique_id():
    uid = UniqueId()
    check(lib().ncclGetUniqueId(ctypes.byref(uid)))
    return ctypes.string_at(ctypes.addressof(uid), 128)  # .internal would stop at the first NUL


def bootstrap_exchange(uid_bytes, rank, nranks, payload, timeout_ms=60000):
    """All-gather of equal-size byte records between the ranks of one node (gc3BootstrapExchange)."""
    uid = UniqueId()
    ctypes.memmove(ctypes.addressof(uid), uid_bytes, 128)  # attribute assignment stops at a NUL
    out = ctypes.create_string_buffer(len(payload) * nranks)
    check(lib().gc3BootstrapExchange(ctypes.byref(uid), rank, nranks, payload, len(payload), out, timeout_ms))
    return [out.raw[r * len(payload):(r + 1) * len(payload)] for r in range(nranks)]


def init_rank(nranks, uid_bytes, rank):
    uid = UniqueId()
    ctypes.memmove(ctypes.addressof(uid), uid_bytes, 128)  # attribute assignment stops at a NUL
    h = ctypes.c_void_p()
    check(lib().ncclCommInitRank(ctypes.byref(h), nranks, uid, rank))
    return Comm(h.value)
