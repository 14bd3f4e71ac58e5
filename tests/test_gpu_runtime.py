"""Runtime behaviour on the GPU beyond the per-IR parity tests: launch ordering across streams,
the watchdog's sticky error, and a ReduceScatter whose owned block is written by direct messages."""
import json

import numpy as np
import pytest

from conftest import ir_path, read_ir

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def rs2_direct_final_recv():
    """A 2-rank ReduceScatter whose final write of each owned chunk is a plain recv from the peer
    (the peer reduces the chunk and sends it back). That recv is both a direct message (the sender
    can store straight into the receiver's span) and the final write of the owned block (result
    buffer = recvbuff): the sender must store into recvbuff."""
    def op(step, opcode, buf_off):
        return {"count": 1, "deps": [], "dst_buf": "input", "dst_off": buf_off, "has_dep": False, "opcode": opcode,
                "src_buf": "input", "src_off": buf_off, "step": step}

    def gpu(r):
        mine, other = r, 1 - r
        return {"rank": r, "threadblocks": [{"channel": 0, "id": 0, "recv_peer": other, "send_peer": other, "ops": [
            op(0, "send", mine), op(1, "rrc", other), op(2, "send", other), op(3, "recv", mine)]}]}
    return {"collective": "reducescatter", "gpus": [gpu(0), gpu(1)], "inplace": True, "name": "rs2_direct_final_recv",
            "nchunks": {"input": 2, "output": 2, "scratch": 0}, "protocol": "simple",
            "size_range": {"max_bytes": 1 << 40, "min_bytes": 0}}


@pytest.mark.parametrize("proto", ["simple", "ll", "ll128"])
@pytest.mark.parametrize("count", [4096, 1 << 18])
def test_reducescatter_direct_final_write_lands_in_recvbuff(proto, count):
    from paper_2201_11840_b200 import gc3
    from gpu_util import make_input, oracle_collective, run_collective, to_np_bits
    irj = rs2_direct_final_recv()
    comms = gc3.init_all([0, 0])
    try:
        for c in comms:
            c.register_ir(json.dumps(irj))
            c.set_protocol(0, proto)
        inputs = [make_input(2 * count, "float32", 5 + r) for r in range(2)]
        expected = oracle_collective(irj, "reducescatter", [x.clone() for x in inputs], count, "float32")
        outs = run_collective(comms, "reducescatter", inputs, count, "float32")
        torch.cuda.synchronize()
        assert comms[0].async_error()[0] == 0
        for r in range(2):
            assert np.array_equal(to_np_bits(outs[r], "float32"), expected[r]), r
    finally:
        for c in comms:
            c.destroy()


def test_collectives_on_different_streams_do_not_overlap():
    """Two collectives of one communicator issued back to back on different streams share FIFO
    counters, scratch and work buffers: the runtime orders them (the second waits for the first)."""
    from paper_2201_11840_b200 import gc3
    from gpu_util import make_input, oracle_collective, run_collective, to_np_bits
    irj = json.loads(read_ir("ring_ar_8_ch1"))
    comms = gc3.init_all([0] * 8)
    try:
        for c in comms:
            c.register_ir(ir_path("ring_ar_8_ch1"))
        s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        counts = [8 * (1 << 18), 8 * 1000, 8 * (1 << 16)]
        inputs = [[make_input(n, "float32", 100 * k + r) for r in range(8)] for k, n in enumerate(counts)]
        expected = [oracle_collective(irj, "allreduce", [x.clone() for x in inp], n, "float32") for inp, n in zip(inputs, counts)]
        torch.cuda.synchronize()
        outs = [run_collective(comms, "allreduce", inp, n, "float32", stream=s) for inp, n, s in zip(inputs, counts, (s1, s2, s3))]
        torch.cuda.synchronize()
        assert comms[0].async_error()[0] == 0
        for k in range(3):
            for r in range(8):
                assert np.array_equal(to_np_bits(outs[k][r], "float32"), expected[k][r]), (k, r)
    finally:
        for c in comms:
            c.destroy()


def test_watchdog_error_is_sticky():
    """After a watchdog timeout the device abort flag stays raised; the next collective on the
    communicator must fail (not return success and leave recvbuff unwritten)."""
    from paper_2201_11840_b200 import gc3
    from gpu_util import make_input, run_collective
    comms = gc3.init_all([0] * 8)
    try:
        for c in comms:
            for k, v in dict(slots=1, timeout_ms=1500, lanes=1, tile_bytes=4096).items():
                c.set_config(k, v)
            c.register_ir(ir_path("ring_ar_8_ch1"))
        inputs = [make_input(8 * 65536, "float32", r) for r in range(8)]
        run_collective(comms, "allreduce", inputs, 8 * 65536, "float32")
        torch.cuda.synchronize()
        err, msg = comms[0].async_error()
        assert err != 0 and "watchdog" in msg
        with pytest.raises(gc3.NcclError):
            run_collective(comms, "allreduce", inputs, 8 * 1024, "float32")
    finally:
        for c in comms:
            c.abort()


@pytest.mark.parametrize("name,coll,count,dtype,cfg", [
    ("ring_ar_8_ch8_inst4", "allreduce", 8 * 4 * 8192, "float32", {}),               # static lanes, op-major groups
    ("ring_ar_8_ch8_inst4", "allreduce", 8 * 4 * 8192, "float32", {"df": 2}),        # dataflow
    ("hier_ar_2x4_par1", "allreduce", 8 * 65536, "bfloat16", {}),
    ("twostep_a2a_2x4", "alltoall", 65536, "float32", {}),                          # work queue
    ("ring_ar_8_ch1", "allreduce", 8 * 4096, "float32", {"proto": "ll"}),
    ("ring_rs_8", "reducescatter", 40000, "int32", {"proto": "ll128"})])
def test_cuda_graph_replays_are_fresh_launches(name, coll, count, dtype, cfg):
    """Collectives captured in a CUDA graph and replayed: every replay must behave like a new launch
    (semaphore / progress epochs come from a device-side counter, not a baked-in argument), bit-exact
    against the oracle for new input contents at every replay."""
    from paper_2201_11840_b200 import gc3
    from gpu_util import input_len, make_input, oracle_collective, run_collective, to_np_bits
    irj = json.loads(read_ir(name))
    R = len(irj["gpus"])
    comms = gc3.init_all([0] * R)
    try:
        for c in comms:
            for k, v in cfg.items():
                if k != "proto":
                    c.set_config(k, v)
            i = c.register_ir(ir_path(name))
            if "proto" in cfg:
                c.set_protocol(i, cfg["proto"])
        n = input_len(coll, count, R)
        bufs = [make_input(n, dtype, 0, device="cuda") for _ in range(R)]
        stream = torch.cuda.Stream()
        stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(stream):
            run_collective(comms, coll, bufs, count, dtype)  # warm-up: buffers and tables allocated
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            outs = run_collective(comms, coll, bufs, count, dtype)
        for rep in range(3):
            fresh = [make_input(n, dtype, 100 * rep + r) for r in range(R)]
            for b, f in zip(bufs, fresh):
                b.copy_(f)
            torch.cuda.synchronize()
            expected = oracle_collective(irj, coll, [f.clone() for f in fresh], count, dtype)
            g.replay()
            torch.cuda.synchronize()
            assert comms[0].async_error()[0] == 0
            for r in range(R):
                assert np.array_equal(to_np_bits(outs[r], dtype), expected[r]), (rep, r)
        del g
    finally:
        for c in comms:
            c.destroy()
