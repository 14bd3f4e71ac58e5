"""IR buffer shapes the NCCL entry points accept (runtime.cpp register_program; SURVEY.md §8(b),
core.hpp:305-397): AllReduce / ReduceScatter IRs must be in place with nchunks.output ==
nchunks.input (ReduceScatter: divisible by the ranks), AllGather out of place with output = ranks x
input, AlltoAll out of place with output == input divisible by the ranks. Anything else is rejected
at registration (ncclInvalidUsage) instead of writing past recvbuff at launch. Host-only: the
check runs before any device allocation."""
import json

import pytest

from conftest import read_ir


def _mutated(name, **kw):
    irj = json.loads(read_ir(name))
    for k, v in kw.items():
        if k in ("input", "output", "scratch"):
            irj["nchunks"][k] = v
        else:
            irj[k] = v
    return irj


@pytest.mark.parametrize("name,kw,msg", [
    ("ring_ar_8_ch1", dict(inplace=False), "in place"),
    ("ring_ar_8_ch1", dict(output=16), "output"),
    ("ring_rs_8", dict(inplace=False), "in place"),
    ("ring_ag_8", dict(inplace=True), ""),  # (the validator already rejects it)
    ("ring_ag_8", dict(output=16), "ranks x nchunks.input"),
    ("twostep_a2a_1x8", dict(inplace=True), "out of place"),
    ("twostep_a2a_1x8", dict(output=16), "output"),
])
def test_register_rejects_unsupported_buffer_shapes(gc3lib, name, kw, msg):
    gc3 = gc3lib
    irj = _mutated(name, **kw)
    comms = gc3.init_all([0] * len(irj["gpus"]))
    try:
        with pytest.raises(gc3.NcclError) as ei:
            comms[0].register_ir(json.dumps(irj))
        assert msg in str(ei.value) or msg in gc3.lib().ncclGetLastError(None).decode()
    finally:
        for c in comms:
            c.destroy()


def test_direct_final_write_of_reducescatter_is_flagged(gc3lib):
    """The IR of tests/test_gpu_runtime.py: its final recv of each owned chunk is both a direct
    message and a result write (runtime.cpp result_writes / direct_messages), the case in which the
    sender must store into the result buffer."""
    from test_gpu_runtime import rs2_direct_final_recv
    gc3 = gc3lib
    ir = gc3.IR(json.dumps(rs2_direct_final_recv()))
    complete, res = ir.result_writes()
    direct = ir.direct_messages()
    assert complete
    for r in range(2):
        assert res[r][0][3] == 1
        assert direct[r][0][3] & 1  # kInDirect
        assert direct[1 - r][0][2] & 2  # kOutDirect on the peer's send
