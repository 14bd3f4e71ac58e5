"""GPU parity: the sm_100a interpreter (through the C ABI) vs the CPU oracle, bit for bit.

All R ranks of an IR run as loopback ranks on cuda:0 (ncclCommInitAll with a repeated device),
so cross-rank FIFO / flag / semaphore logic is exercised inside one cooperative launch.
"""
import json

import numpy as np
import pytest

from conftest import ir_path, read_ir

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

COLL_OF = {"allreduce": "allreduce", "allgather": "allgather", "reducescatter": "reducescatter", "alltoall": "alltoall"}


def _setup(name, instances=1, proto=None, **cfg):
    from paper_2201_11840_b200 import gc3
    text = read_ir(name)
    R = len(json.loads(text)["gpus"])
    comms = gc3.init_all([0] * R)
    for c in comms:
        for k, v in cfg.items():
            c.set_config(k, v)
    ids = [c.register_ir(ir_path(name), instances) for c in comms]
    if proto is not None:
        for c, i in zip(comms, ids):
            c.set_protocol(i, proto)
    ir_json = comms[0] and gc3.IR(text).replicate(instances).serialize() if instances > 1 else text
    return comms, json.loads(ir_json)


def _check(name, count, dtype="float32", op="sum", instances=1, proto=None, inplace=False, seed=0, **cfg):
    from gpu_util import input_len, make_input, oracle_collective, run_collective, to_np_bits
    comms, irj = _setup(name, instances, proto, **cfg)
    try:
        coll = irj["collective"]
        R = len(comms)
        inputs = [make_input(input_len(coll, count, R), dtype, seed * 100 + r) for r in range(R)]
        expected = oracle_collective(irj, coll, [x.clone() for x in inputs], count, dtype, op)
        outs = run_collective(comms, coll, inputs, count, dtype, op, inplace=inplace)
        torch.cuda.synchronize()
        for c in comms:
            err, msg = c.async_error()
            assert err == 0, msg
        for r in range(R):
            got = to_np_bits(outs[r], dtype)
            exp = expected[r]
            if not np.array_equal(got.view(exp.dtype) if got.dtype != exp.dtype else got, exp):
                bad = np.nonzero(got.view(exp.dtype) != exp)[0] if got.size == exp.size else []
                raise AssertionError(f"rank {r}: {len(bad)} mismatches, first at {bad[:8]}")
    finally:
        for c in comms:
            c.destroy()


@pytest.mark.parametrize("name,count", [
    ("ring_ar_8_ch1", 8 * 1024), ("ring_ar_8_ch1", 1 << 20), ("ring_ar_8_ch8_inst4", 32 * 4096),
    ("ring_ar_8_inst4_auto", 32 * 1000), ("hier_ar_2x4_par1", 8 * 4096), ("hier_ar_2x4_par2", 16 * 512),
    ("allpairs_ar_8", 8 * 777), ("ring_ar_4_ch1", 4 * 3000), ("ring_ar_2_ch1", 2 * 64),
    ("ring_ar_8_ch8_inst1.unfused", 8 * 1024), ("hier_ar_2x4_par1.unfused", 8 * 2048),
])
def test_allreduce_f32(name, count):
    _check(name, count)


@pytest.mark.parametrize("dtype,op", [("bfloat16", "sum"), ("float16", "sum"), ("int32", "sum"), ("float64", "sum"),
                                      ("int64", "prod"), ("float32", "max"), ("bfloat16", "min"), ("uint8", "sum"),
                                      ("int8", "max"), ("uint32", "prod")])
def test_allreduce_dtypes(dtype, op):
    _check("hier_ar_2x4_par1", 8 * 2048, dtype, op)


@pytest.mark.parametrize("name,count", [("ring_ag_8", 4096), ("ring_ag_4", 1000), ("ring_ag_2", 7)])
def test_allgather(name, count):
    _check(name, count)
    _check(name, count, inplace=True, dtype="bfloat16")


@pytest.mark.parametrize("name,count", [("ring_rs_8", 4096), ("ring_rs_4", 999), ("ring_rs_2", 16)])
def test_reducescatter(name, count):
    _check(name, count)
    _check(name, count, inplace=True, dtype="bfloat16")


@pytest.mark.parametrize("name,count", [("twostep_a2a_2x4", 4096), ("twostep_a2a_1x8", 1024), ("twostep_a2a_2x2", 333),
                                        ("twostep_a2a_1x2", 5)])
def test_alltoall(name, count):
    _check(name, count)


def test_allreduce_out_of_place_and_in_place():
    _check("ring_ar_8_ch1", 8 * 2000, inplace=False)
    _check("ring_ar_8_ch1", 8 * 2000, inplace=True)


@pytest.mark.parametrize("name,count", [("ring_ar_8_ch1", 8 * 4096), ("hier_ar_2x4_par1", 8 * 4096),
                                        ("twostep_a2a_2x4", 2048), ("ring_rs_8", 1024), ("ring_ag_8", 1024)])
def test_ll_protocol(name, count):
    _check(name, count, proto="ll")
    _check(name, count, proto="ll", dtype="bfloat16")


@pytest.mark.parametrize("lanes,tile_bytes", [(1, 0), (3, 0), (16, 0), (4, 1040), (7, 48)])
def test_lanes_and_tiles(lanes, tile_bytes):
    _check("hier_ar_2x4_par1", 8 * 5000, lanes=lanes, tile_bytes=tile_bytes)
    _check("twostep_a2a_2x4", 3000, lanes=lanes, tile_bytes=tile_bytes)


def test_instances_runtime_rewrite():
    _check("ring_ar_8_ch8_inst1", 32 * 512, instances=4)


def test_repeated_launches_keep_fifo_counters_consistent():
    from gpu_util import make_input, oracle_collective, run_collective, to_np_bits
    comms, irj = _setup("ring_ar_8_ch1")
    try:
        for it, count in enumerate([8 * 100, 8 * 4096, 8, 8 * 12345]):
            inputs = [make_input(count, "float32", 10 * it + r) for r in range(8)]
            expected = oracle_collective(irj, "allreduce", [x.clone() for x in inputs], count, "float32")
            outs = run_collective(comms, "allreduce", inputs, count, "float32")
            torch.cuda.synchronize()
            for r in range(8):
                assert np.array_equal(to_np_bits(outs[r], "float32"), expected[r])
    finally:
        for c in comms:
            c.destroy()


def test_watchdog_reports_deadlock_instead_of_hanging():
    """SURVEY Finding 1 on hardware: s=1 deadlocks ring_ar_8_ch1; the watchdog must report it."""
    from gpu_util import make_input, run_collective
    comms, irj = _setup("ring_ar_8_ch1", slots=1, timeout_ms=1500, lanes=1)
    try:
        inputs = [make_input(8 * 65536, "float32", r) for r in range(8)]
        for c in comms:
            c.set_config("tile_bytes", 4096)
        run_collective(comms, "allreduce", inputs, 8 * 65536, "float32")
        torch.cuda.synchronize()
        err, msg = comms[0].async_error()
        assert err != 0 and "watchdog" in msg
    finally:
        for c in comms:
            c.destroy()


def test_size_range_selection_and_no_fallback():
    from paper_2201_11840_b200 import gc3
    text = json.loads(read_ir("ring_ar_8_ch1"))
    small = dict(text, name="small", size_range={"min_bytes": 0, "max_bytes": 4096})
    big = dict(text, name="big", size_range={"min_bytes": 4097, "max_bytes": 1 << 40})
    comms = gc3.init_all([0] * 8)
    try:
        for c in comms:
            c.set_config("builtin", 0)  # no built-in programs: an unmatched call is an error
            c.register_ir(json.dumps(small))
            c.register_ir(json.dumps(big))
        assert comms[0].query_plan("allreduce", 1024, "float32")["name"] == "small"
        assert comms[0].query_plan("allreduce", 8192, "float32")["name"] == "big"
        assert comms[0].query_plan("allgather", 8192, "float32")["ir_id"] == -1
        with pytest.raises(gc3.NcclError):
            with gc3.group():
                for c in comms:
                    x = torch.zeros(64, device="cuda")
                    c.all_gather(x, torch.zeros(512, device="cuda"), 64, "float32")
    finally:
        for c in comms:
            c.destroy()


@pytest.mark.parametrize("name,count", [("twostep_a2a_2x4", 2048), ("ring_ag_8", 1024), ("ring_ar_8_ch1", 8 * 1024)])
def test_fifo_only_path(name, count):
    """direct=0 forces every message through the receiver FIFO (the multi-process path)."""
    _check(name, count, direct=0)
    _check(name, count, direct=0, proto="ll")


@pytest.mark.parametrize("name,count", [("twostep_a2a_2x4", 4096), ("ring_ag_8", 2048), ("twostep_a2a_1x8", 1000)])
def test_direct_path_ll(name, count):
    _check(name, count, proto="ll")
    _check(name, count, proto="ll", dtype="bfloat16")


@pytest.mark.parametrize("name,count", [("twostep_a2a_2x4", 5000), ("hier_ar_2x4_par1", 8 * 6000)])
@pytest.mark.parametrize("balance", [0, 1])
def test_lane_multipliers(name, count, balance):
    """Per-component lane counts (balance=1) and uniform lanes (balance=0) give the same bits."""
    _check(name, count, balance=balance, tile_bytes=1024)
    _check(name, count, balance=balance, group=1, lanes=3, tile_bytes=2048)


@pytest.mark.parametrize("name,count,dtype,instances", [
    ("ring_ar_8_ch1", 8 * 1000 + 3, "float32", 1), ("ring_ar_8_ch1", 5, "float32", 1),
    ("hier_ar_2x4_par1", 8 * 4096 + 7, "bfloat16", 1), ("ring_ar_8_ch8_inst4", 32 * 100 + 31, "float32", 1),
    ("ring_ag_8", 1001, "float32", 4), ("ring_ag_4", 3, "bfloat16", 2),
    ("ring_rs_8", 777, "float32", 4), ("ring_rs_2", 1, "int32", 3),
    ("twostep_a2a_1x8", 1003, "float32", 3), ("twostep_a2a_1x8", 2, "float16", 4),
])
def test_ragged_counts(name, count, dtype, instances):
    """Counts the IR's chunks do not divide: chunks of ceil(count / c) elements, the last ones
    clipped (the runtime stages through padded work buffers); bit-exact vs the oracle's clipping."""
    _check(name, count, dtype, instances=instances)
    _check(name, count, dtype, instances=instances, proto="ll")


@pytest.mark.parametrize("coll,name", [("allreduce", "ring_ar_8_ch1"), ("allgather", "ring_ag_8"),
                                       ("reducescatter", "ring_rs_8"), ("alltoall", "twostep_a2a_2x4")])
def test_zero_count_is_a_noop(coll, name):
    from gpu_util import run_collective
    comms, irj = _setup(name)
    try:
        outs = run_collective(comms, coll, [torch.zeros(0, device="cuda") for _ in comms], 0, "float32")
        torch.cuda.synchronize()
        assert all(o.numel() == 0 for o in outs)
        assert comms[0].async_error()[0] == 0
    finally:
        for c in comms:
            c.destroy()


@pytest.mark.parametrize("name,count,fold", [("hier_ar_2x4_par1", 8 * 3000, True), ("twostep_a2a_2x4", 2000, False),
                                             ("ring_rs_8", 1000, True)])
def test_msccl_xml_registration(name, count, fold, tmp_path):
    """gc3RegisterIR with an MSCCL algorithm file (csrc/msccl_xml.cpp): same bits as the oracle run
    on the GC3-IR the XML came from (fold=False registers the nop-expanded text)."""
    from paper_2201_11840_b200 import gc3
    from gpu_util import input_len, make_input, oracle_collective, run_collective, to_np_bits
    ir = gc3.IR(read_ir(name))
    xml = ir.to_xml()
    if not fold:  # register the nop-expanded program text (MSCCL's one-dependency encoding kept)
        xml = gc3.IR.from_xml(xml, fold_nops=False).to_xml()
    f = tmp_path / (name + ".xml")
    f.write_text(xml)
    irj = json.loads(read_ir(name))
    R = len(irj["gpus"])
    comms = gc3.init_all([0] * R)
    try:
        for c in comms:
            c.register_ir(str(f))
        coll = irj["collective"]
        inputs = [make_input(input_len(coll, count, R), "float32", 7 + r) for r in range(R)]
        expected = oracle_collective(irj, coll, [x.clone() for x in inputs], count, "float32")
        outs = run_collective(comms, coll, inputs, count, "float32")
        torch.cuda.synchronize()
        assert comms[0].async_error()[0] == 0
        for r in range(R):
            assert np.array_equal(to_np_bits(outs[r], "float32"), expected[r])
    finally:
        for c in comms:
            c.destroy()


@pytest.mark.parametrize("name,count,dtype", [("hier_ar_2x4_par1", 8 * (1 << 20), "float32"),
                                              ("twostep_a2a_2x4", 1 << 20, "bfloat16"),
                                              ("ring_ar_8_ch1", 8 * (1 << 20) + 8 * 12345, "float32"),
                                              ("ring_rs_8", 1 << 20, "int32")])
def test_tapered_tiles(name, count, dtype):
    """Quarter tiles in the first and last round of every lane (tapered geometry) on few lanes,
    where it is active, vs uniform tiles: same bits as the oracle."""
    _check(name, count, dtype, lanes=2, balance=0, taper=1)
    _check(name, count, dtype, lanes=2, balance=0, taper=0)


@pytest.mark.parametrize("name,count,dtype", [("twostep_a2a_2x4", 1 << 18, "float32"), ("ring_ag_8", 1 << 17, "bfloat16"),
                                              ("ring_rs_8", 1 << 17, "int32"), ("twostep_a2a_1x8", 12345, "float16")])
@pytest.mark.parametrize("wq", [0, 2])
def test_work_queue_mode(name, count, dtype, wq):
    """Programs whose messages are all direct or pulled run as a work queue of (thread block, tile)
    items (interp_wq) or on static lanes: same bits either way."""
    _check(name, count, dtype, wq=wq)
    _check(name, count, dtype, wq=wq, wq_items=1)
    _check(name, count, dtype, wq=wq, wq_items=2, wq_lag=2)  # lagged claim order


@pytest.mark.parametrize("coll,count,dtype", [("allreduce", 8 * 1000 + 5, "float32"), ("allgather", 4096, "bfloat16"),
                                              ("reducescatter", 3000, "int32"), ("alltoall", 2048, "float32"),
                                              ("allreduce", 1 << 18, "float32"), ("allreduce", 1 << 20, "float32"),
                                              ("allreduce", 3 << 20, "float32")])
def test_builtin_programs_without_registration(coll, count, dtype):
    """Drop-in use: collectives on communicators with no registered IR run the runtime's built-in
    programs (comm-time generated, op for op the reference compiler's ring / direct algorithms;
    AllReduce per size tier), bit-exact vs the oracle running the same program; a registered IR for
    the collective takes precedence afterwards."""
    from paper_2201_11840_b200 import gc3
    from gpu_util import input_len, make_input, oracle_collective, run_collective, to_np_bits
    R = 8
    comms = gc3.init_all([0] * R)
    try:
        esize = {"float32": 4, "bfloat16": 2, "int32": 4}[dtype]
        sel = count * esize * (1 if coll == "allreduce" else R)  # size_range measure (selection bytes)
        builtin = gc3.IR.builtin(coll, R, sel)
        irj = json.loads(builtin.serialize())
        inputs = [make_input(input_len(coll, count, R), dtype, 3 + r) for r in range(R)]
        expected = oracle_collective(irj, coll, [x.clone() for x in inputs], count, dtype)
        for it in range(2):  # the second call reuses the registered built-in
            outs = run_collective(comms, coll, [x.clone() for x in inputs], count, dtype)
            torch.cuda.synchronize()
            assert comms[0].async_error()[0] == 0
            for r in range(R):
                assert np.array_equal(to_np_bits(outs[r], dtype), expected[r]), (it, r)
        assert comms[0].query_plan(coll, count, dtype)["name"] == irj["name"]
        name = {"allreduce": "hier_ar_2x4_par1", "allgather": "ring_ag_8", "reducescatter": "ring_rs_8",
                "alltoall": "twostep_a2a_2x4"}[coll]
        for c in comms:
            c.register_ir(ir_path(name))
        assert comms[0].query_plan(coll, count, dtype)["name"] == name
    finally:
        for c in comms:
            c.destroy()


@pytest.mark.parametrize("name", ["hier_ar_2x4_par1", "ring_ar_8_ch1"])
@pytest.mark.parametrize("dtype", ["bfloat16", "float16", "int32", "int64", "uint64", "float32"])
def test_large_sums_with_special_values(name, dtype):
    """Sums big enough for the bulk-engine paths (staged reductions, and for 16-bit floats and
    integers the in-place L2 reduction, cp.reduce.async.bulk), with subnormals, infinities, NaNs and
    rounding ties among the inputs: bit-exact vs the oracle."""
    from paper_2201_11840_b200 import gc3
    from gpu_util import TORCH_DT, make_input, oracle_collective, run_collective, to_np_bits
    irj = json.loads(read_ir(name))
    R, count = 8, 8 * 65536
    comms = gc3.init_all([0] * R)
    try:
        for c in comms:
            c.register_ir(ir_path(name))
            c.set_config("tma_min", 0)  # every aligned op through the bulk engine (L2 sums included)
            c.set_config("lanes", 2)    # large tiles
        inputs = []
        for r in range(R):
            x = make_input(count, dtype, 40 + r)
            if dtype in ("bfloat16", "float16", "float32"):
                bits = {"bfloat16": torch.int16, "float16": torch.int16, "float32": torch.int32}[dtype]
                v = x.view(bits)
                v[r::97] = 1                      # smallest subnormal
                v[r + 5::389] = -32767 if dtype != "float32" else -2147483647  # negative subnormal
                v[5000:5400] = torch.arange(1, 401, dtype=bits) * (r + 1)  # all-subnormal sums
                x[r + 11::1009] = float("inf")
                x[r + 13::4099] = float("-inf")
                x[r + 17::8191] = float("nan")
            inputs.append(x)
        expected = oracle_collective(irj, "allreduce", [x.clone() for x in inputs], count, dtype)
        outs = run_collective(comms, "allreduce", inputs, count, dtype, inplace=True)
        torch.cuda.synchronize()
        assert comms[0].async_error()[0] == 0
        for r in range(R):  # compare bit patterns (NaN payloads included)
            got = to_np_bits(outs[r], dtype)
            exp = expected[r]
            ut = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[exp.dtype.itemsize]
            g, e = got.view(ut), exp.view(ut)
            bad = np.nonzero(g != e)[0]
            assert bad.size == 0, (r, bad[:8], g[bad[:4]], e[bad[:4]])
    finally:
        for c in comms:
            c.destroy()


def test_select_by_timed_model():
    """Config "select": among matching IRs the runtime runs the one the timed model predicts fastest
    (runtime.cpp predict_us), and the result stays bit-exact."""
    from paper_2201_11840_b200 import gc3
    from gpu_util import make_input, oracle_collective, run_collective, to_np_bits
    names = ["ring_ar_8_ch1", "ring_ar_8_ch8_inst4"]
    count = 32 * 65536
    preds = {n: gc3.IR(read_ir(n)).predict_us(count * 4 // {"ring_ar_8_ch1": 8, "ring_ar_8_ch8_inst4": 32}[n],
                                             "simple", 64 if n == "ring_ar_8_ch1" else 2) for n in names}
    comms = gc3.init_all([0] * 8)
    try:
        for c in comms:
            c.set_config("select", 1)
            for n in names:
                c.register_ir(ir_path(n))
        chosen = comms[0].query_plan("allreduce", count, "float32")["name"]
        assert chosen in names
        irj = json.loads(read_ir(chosen))
        inputs = [make_input(count, "float32", 60 + r) for r in range(8)]
        expected = oracle_collective(irj, "allreduce", [x.clone() for x in inputs], count, "float32")
        outs = run_collective(comms, "allreduce", inputs, count, "float32")
        torch.cuda.synchronize()
        assert comms[0].async_error()[0] == 0
        for r in range(8):
            assert np.array_equal(to_np_bits(outs[r], "float32"), expected[r])
    finally:
        for c in comms:
            c.destroy()
    assert preds  # (predictions exercised on the host as well)


def test_small_messages_switch_to_ll():
    """ll_max_bytes: a Simple IR runs the LL protocol for messages up to the threshold (per rank),
    Simple above it; both bit-exact."""
    from paper_2201_11840_b200 import gc3
    comms, irj = _setup("ring_ar_8_ch8_inst4", ll_max_bytes=256 << 10)
    try:
        assert comms[0].query_plan("allreduce", 32 * 1024, "float32")["protocol"] == 1   # 128 KiB per rank
        assert comms[0].query_plan("allreduce", 32 * 65536, "float32")["protocol"] == 0  # 8 MiB per rank
    finally:
        for c in comms:
            c.destroy()
    _check("ring_ar_8_ch8_inst4", 32 * 1024, ll_max_bytes=256 << 10)
    _check("ring_ar_8_ch8_inst4", 32 * 65536, ll_max_bytes=256 << 10)


@pytest.mark.parametrize("name,count,dtype", [
    ("ring_ar_8_ch1", 8 * 4096, "float32"), ("ring_ar_8_ch8_inst4", 32 * 4096, "float32"), ("hier_ar_2x4_par1", 8 * 6000, "bfloat16"),
    ("hier_ar_2x4_par2", 16 * 512, "float32"), ("allpairs_ar_8", 8 * 777, "float32"), ("ring_ar_8_inst4_auto", 32 * 1000, "int32"),
    ("ring_ag_8", 4096, "float32"), ("ring_rs_8", 4096, "bfloat16"), ("twostep_a2a_2x4", 4096, "float32"),
    ("ring_ar_8_ch8_inst1.unfused", 8 * 1024, "float32"), ("hier_ar_2x4_par1.unfused", 8 * 2048, "float16"),
])
@pytest.mark.parametrize("df,tile", [(2, 0), (2, 1024), (2, 128), (0, 0)])
def test_dataflow_mode(name, count, dtype, df, tile):
    """Dataflow execution (interp_df_kernel: ready (op, tile) items, mailed messages for rrs) vs
    static lanes: bit-exact vs the oracle for every family, tile size and dtype."""
    _check(name, count, dtype, df=df, tile_bytes=tile, df_min_tile=128)


def test_dataflow_mode_is_selected_and_mails_rrs_messages():
    comms, irj = _setup("hier_ar_2x4_par1")
    try:
        plan = comms[0].query_plan("allreduce", 32 << 20, "float32")
        assert plan["mode"] == 2
        assert plan["mail_messages"] == 8  # one rrs -> rrc message per rank
        # small messages (fewer than two items per unit) stay on static lanes by default
        assert comms[0].query_plan("allreduce", 8 * 65536, "float32")["mode"] == 0
    finally:
        for c in comms:
            c.destroy()
    comms, irj = _setup("hier_ar_2x4_par1", df=0)
    try:
        assert comms[0].query_plan("allreduce", 32 << 20, "float32")["mode"] == 0
    finally:
        for c in comms:
            c.destroy()


@pytest.mark.parametrize("waves", [1, 0])
def test_dataflow_whole_wave_tiles(waves):
    """Dataflow tile count rounded to one wave of units per level (config df_waves, runtime.cpp
    plan_launch): C4's program (width 32: 480 nodes over 15 levels) at 64 KiB chunks with 4 KiB
    minimum tiles takes units / 32 tiles per chunk (18 on a B200, the last one ragged) instead of
    16; bit-exact vs the oracle either way."""
    count = 32 * 16384  # 2 MiB per rank, 64 KiB chunks
    cfg = dict(df_min_tile=4096, df_waves=waves, ll_max_bytes=0, ll128_max_bytes=0)  # Simple at 2 MiB
    comms, _ = _setup("ring_ar_8_ch8_inst4", **cfg)
    try:
        plan = comms[0].query_plan("allreduce", count, "float32")
        assert plan["mode"] == 2
        units = plan["grid"] * (512 // (32 * plan["unit_warps"]))
        if waves:
            assert 16 <= plan["ntiles"] and plan["ntiles"] * 32 <= units
            assert plan["ntiles"] == units // 32 or units // 32 < 16
        else:
            assert plan["ntiles"] == 16
    finally:
        for c in comms:
            c.destroy()
    _check("ring_ar_8_ch8_inst4", count, **cfg)


@pytest.mark.parametrize("name,count", [("ring_ar_8_ch1", 8 * 1000 + 3), ("ring_rs_8", 777), ("ring_ag_8", 1001)])
def test_dataflow_ragged_and_repeated(name, count):
    from gpu_util import make_input, oracle_collective, run_collective, to_np_bits
    comms, irj = _setup(name, df=2)
    try:
        coll = irj["collective"]
        R = len(comms)
        for it, n in enumerate([count, 8 * 64, count * 3, 8]):
            from gpu_util import input_len
            inputs = [make_input(input_len(coll, n, R), "float32", 17 * it + r) for r in range(R)]
            expected = oracle_collective(irj, coll, [x.clone() for x in inputs], n, "float32")
            outs = run_collective(comms, coll, inputs, n, "float32")
            torch.cuda.synchronize()
            assert comms[0].async_error()[0] == 0
            for r in range(R):
                assert np.array_equal(to_np_bits(outs[r], "float32"), expected[r]), (it, r)
    finally:
        for c in comms:
            c.destroy()


@pytest.mark.parametrize("algo,R,C,K", [("allpairs", 8, 1, 1), ("hier", 8, 4, 1), ("hier", 8, 2, 1), ("ring", 8, 8, 4),
                                        ("ring", 8, 2, 2), ("ring", 4, 4, 2)])
@pytest.mark.parametrize("dtype,proto", [("float32", None), ("bfloat16", None), ("float32", "ll"), ("float32", "ll128")])
def test_generated_programs_on_the_gpu(algo, R, C, K, dtype, proto):
    """Comm-time generated programs (gc3IrGenerate: ring channels x instances, all-pairs,
    hierarchical) registered as IR text and run through the C ABI: bit-exact vs the oracle running
    the same program."""
    from paper_2201_11840_b200 import gc3
    from gpu_util import make_input, oracle_collective, run_collective, to_np_bits
    text = gc3.IR.generate(algo, "allreduce", R, C, K).serialize()
    irj = json.loads(text)
    comms = gc3.init_all([0] * R)
    try:
        for c in comms:
            i = c.register_ir(text)
            if proto:
                c.set_protocol(i, proto)
        count = irj["nchunks"]["input"] * 3000 + 7
        inputs = [make_input(count, dtype, 50 + r) for r in range(R)]
        expected = oracle_collective(irj, "allreduce", [x.clone() for x in inputs], count, dtype)
        outs = run_collective(comms, "allreduce", inputs, count, dtype)
        torch.cuda.synchronize()
        assert comms[0].async_error()[0] == 0
        for r in range(R):
            assert np.array_equal(to_np_bits(outs[r], dtype), expected[r]), (algo, r)
    finally:
        for c in comms:
            c.destroy()


@pytest.mark.parametrize("name", ["ring_ar_8_ch1", "ring_ar_8_ch8_inst4", "allpairs_ar_8", "ring_ar_4_ch4_inst4"])
@pytest.mark.parametrize("proto,cfg", [(None, {}), ("ll", {}), ("ll128", {}), (None, {"df": 2, "df_min_tile": 4096}),
                                       (None, {"clip": 0})])
@pytest.mark.parametrize("size", ["big", "small"])
def test_ragged_allreduce_clipped_in_place(name, proto, cfg, size):
    """Ragged AllReduce (count not divisible by the IR's chunks) runs on the caller's buffer with
    tiles clipped at the block's end (LaunchArgs::clip_elems, 16-byte multiples) -- including chunks
    that are cut short or left empty -- bit-exact vs the oracle's padded semantics; clip 0 stages
    through the padded work buffers instead."""
    irj = json.loads(read_ir(name))
    c = irj["nchunks"]["input"]
    # f32, 16-byte multiples. big: chunks of 4096 elements, the last one 4 short; small: chunks of 8
    # elements, the block short by the largest multiple of 4 below c (several chunks empty when c > 8)
    count = c * 4096 - 4 if size == "big" else 8 * c - 4 * ((c - 1) // 4)
    assert -(-count // c) == (4096 if size == "big" else 8) and count % c
    _check(name, count, "float32", proto=proto, **cfg)
    _check(name, count, "float32", proto=proto, inplace=True, **cfg)
