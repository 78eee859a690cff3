"""Host fp32->bf16 conversion throughput (the async upload's host path)."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2603_13289_b200.engine import _check, lib  # noqa: E402

n = 60_000_000
x = np.random.default_rng(0).standard_normal(n).astype(np.float32)
y = np.empty(n, np.uint16)
for t in (1, 2, 4, 8, 12, 16):
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        _check(lib().rk_debug_f32_to_bf16_host(x.ctypes.data_as(C.POINTER(C.c_float)),
                                               y.ctypes.data_as(C.POINTER(C.c_uint16)), C.c_uint64(n), t))
        best = min(best, time.perf_counter() - t0)
    print(f"threads={t}: {best * 1e3:.2f} ms  {n * 4 / best / 1e9:.1f} GB/s fp32 read")
