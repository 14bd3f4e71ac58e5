import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

# the parity tests pin each protocol explicitly: no size-based switch of Simple IRs to LL
os.environ.setdefault("GC3_LL_MAX_BYTES", "0")

GOLDEN = os.path.join(REPO, "tests", "golden")
IR_DIR = os.path.join(GOLDEN, "ir")
REF_LIB = os.path.join(REPO, "oracle", "_ref", "libref.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running")


def golden_names(include_unfused=False, include_ll=False):
    out = []
    for f in sorted(os.listdir(IR_DIR)):
        if not f.endswith(".ir.json"):
            continue
        if f.endswith(".unfused.ir.json") and not include_unfused:
            continue
        if f.endswith(".ll.ir.json") and not include_ll:
            continue
        out.append(f[: -len(".ir.json")])
    return out


def ir_path(name):
    return os.path.join(IR_DIR, name + ".ir.json")


def read_ir(name):
    with open(ir_path(name)) as f:
        return f.read()


@pytest.fixture(scope="session")
def reflib():
    """The reference harness (oracle/_ref/libref.so, compiled from /root/reference headers)."""
    import ctypes
    if not os.path.exists(REF_LIB):
        pytest.skip("oracle/_ref/libref.so not built (reference not available)")
    L = ctypes.CDLL(REF_LIB)
    for fn in ("ref_load", "ref_check_slots", "ref_symbolic", "ref_compile", "ref_fixture_names"):
        getattr(L, fn).restype = ctypes.c_void_p
    L.ref_load.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.ref_check_slots.argtypes = [ctypes.c_char_p, ctypes.c_int]
    L.ref_symbolic.argtypes = [ctypes.c_char_p]
    L.ref_compile.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int]
    L.ref_free.argtypes = [ctypes.c_void_p]

    class Ref:
        @staticmethod
        def _take(p):
            s = ctypes.string_at(p).decode()
            L.ref_free(p)
            return s

        def load(self, text, nodes, gpn, max_tb=0, max_ch=0):
            import json
            return json.loads(self._take(L.ref_load(text.encode(), nodes, gpn, max_tb, max_ch)))

        def check_slots(self, text, slots):
            import json
            return json.loads(self._take(L.ref_check_slots(text.encode(), slots)))

        def compile(self, name, fused=True, proto=0):
            import json
            p = L.ref_compile(name.encode(), int(fused), proto)
            if not p:
                raise KeyError(name)
            s = self._take(p)
            if s.startswith("ERROR"):
                raise RuntimeError(s)
            return json.loads(s)

        def symbolic(self, text):
            import json
            return json.loads(self._take(L.ref_symbolic(text.encode())))

    return Ref()


@pytest.fixture(scope="session")
def gc3lib():
    from paper_2201_11840_b200 import gc3
    if not os.path.exists(gc3.LIB_PATH):
        from paper_2201_11840_b200 import build
        build.build()
    return gc3
