"""B200-native GC3-IR runtime (arXiv 2201.11840) — Python host bindings.

The product is libgc3.so (C ABI, include/gc3.h): the IR loader/validator, the communicator +
FIFO arenas + CUDA IPC runtime and the sm_100a interpreter kernel. This package only binds that
library with ctypes and offers thin helpers for tests and the bench; torch is used for device
memory and streams. There is no CPU fallback: every collective goes through libgc3.so, and the
import fails loudly if the library is missing.
"""
from .gc3 import (  # noqa: F401
    LIB_PATH,
    NCCL_DTYPES,
    NcclError,
    Comm,
    IR,
    PlanInfo,
    coll_id,
    group,
    init_all,
    init_rank,
    get_unique_id,
    lib,
)
