"""Timeline of CTA 0 of one GEMM (rk_debug_trace_gemm): per k-block producer /
MMA times and per-unit epilogue times, in SM clocks from the first event.
  python tools/gemm_trace.py M N K [epi]"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2603_13289_b200.engine import Engine, P, _check, lib  # noqa: E402

if __name__ == "__main__":
    M, N, K = (int(x) for x in sys.argv[1:4])
    epi = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    e = Engine(0)
    out = np.zeros(3 * 512, np.uint64)
    _check(lib().rk_debug_trace_gemm(P(e.ptr), M, N, K, epi, out.ctypes.data_as(C.POINTER(C.c_uint64))))
    tr = out.reshape(3, 512).astype(np.int64)
    t0 = tr[tr > 0].min()
    prod, mma, epi_t = tr[0], tr[1], tr[2]
    n = int((mma > 0).sum())
    print(f"GEMM M={M} N={N} K={K} epi={epi}: CTA 0, {n} k-blocks")
    for i in range(n):
        print(f"  kb {i:3d}: slot {prod[i] - t0 if prod[i] else -1:7d}  full {mma[i] - t0:7d}"
              + (f"  (+{mma[i] - mma[i - 1]})" if i else ""))
    extra = [(i, int(epi_t[i] - t0)) for i in range(100, 130) if epi_t[i]]
    if extra:
        print("  epilogue warp 2 marks:", extra)
    for u in range(50):
        if epi_t[2 * u]:
            print(f"  unit {u}: acc ready {epi_t[2 * u] - t0:7d}  drained {epi_t[2 * u + 1] - t0:7d}")
