"""Timed model (SPEC.md:464-481 run_timed as an alpha-beta model over the happens-before graph;
runtime.cpp predict_us): calibrated on the C4 sweep measured on a B200 and
checked here against that sweep and the other measured configurations, and for the orderings the
runtime relies on when config "select" ranks matching IRs."""
import json
import math
import os

import pytest

from conftest import read_ir

gc3 = pytest.importorskip("paper_2201_11840_b200.gc3")
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (protocol, bytes per rank, lanes, measured us) from profiles/r01f3_sweep_c4.jsonl
SWEEP = os.path.join(REPO, "profiles", "r01f3_sweep_c4.jsonl")


def _sweep():
    out = []
    for ln in open(SWEEP):
        try:
            d = json.loads(ln)
        except ValueError:
            continue
        out.append((d["proto"], d["bytes"], d["lanes"], d["us"]))
    return out


def test_model_tracks_the_measured_sweep():
    ir = gc3.IR(read_ir("ring_ar_8_ch8_inst4"))
    errs = [math.log(ir.predict_us(b // 32, p, ln) / us) for p, b, ln, us in _sweep()]
    rms = math.sqrt(sum(e * e for e in errs) / len(errs))
    assert rms < 0.15, rms                       # ~9% rms on the 42 points
    assert max(abs(e) for e in errs) < math.log(1.6)


def test_model_on_other_measured_configs():
    # (ir, chunk bytes, protocol, lanes, measured us) from profiles/r01f3_quick.jsonl
    cases = [("hier_ar_2x4_par1", (256 << 20) // 8, "simple", 9, 1612.0),
             ("ring_ag_8", (64 << 20) // 8, "simple", 64, 167.3),
             ("ring_rs_8", (64 << 20) // 8, "simple", 64, 229.5),
             ("twostep_a2a_2x4", (64 << 20) // 8, "simple", 11, 288.4),
             ("ring_ar_8_ch1", (4 << 20) // 8, "ll", 64, 144.0)]
    for name, cb, proto, lanes, us in cases:
        pred = gc3.IR(read_ir(name)).predict_us(cb, proto, lanes)
        assert abs(math.log(pred / us)) < math.log(1.5), (name, pred, us)


def test_protocol_crossover_and_monotonicity():
    ir = gc3.IR(read_ir("ring_ar_8_ch8_inst4"))
    sizes = [1 << k for k in range(10, 31)]
    for proto in ("simple", "ll"):
        t = [ir.predict_us(s // 32, proto, 2) for s in sizes]
        assert all(b >= a - 1e-9 for a, b in zip(t, t[1:])), proto
    assert ir.predict_us(1024 // 32, "ll", 1) < ir.predict_us(1024 // 32, "simple", 1)
    assert ir.predict_us((256 << 20) // 32, "ll", 2) > ir.predict_us((256 << 20) // 32, "simple", 2)
