"""Dump the clock64 timeline of one attention CTA (rk_debug_trace_attention)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2603_13289_b200.engine import Engine, P, _check, lib  # noqa: E402

EV_SM = ["start", "s_full", "s_free", "max", "P stored", "p_full", "exp done", "o_done"]
EV_MMA = ["-", "S issue", "-", "-", "PV issue", "-", "-", "-"]

if __name__ == "__main__":
    M, T, H, Hkv, dh = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (4032, 4032, 32, 8, 64)))
    e = Engine(0)
    out = np.zeros(3 * 64 * 8, np.uint64)
    _check(lib().rk_debug_trace_attention(P(e.ptr), M, T, H, Hkv, dh, out.ctypes.data_as(C.POINTER(C.c_uint64))))
    tr = out.reshape(3, 64, 8).astype(np.int64)
    t0 = tr[tr > 0].min()
    print("grid-wide: CTA (head 0, last tile, split 0); timestamps in SM clocks from its first event")
    for role in range(3):
        names = EV_MMA if role == 2 else EV_SM
        print(f"role {role} ({'MMA' if role == 2 else 'softmax ' + str(role)})")
        for j in range(64):
            row = tr[role, j]
            if not row.any():
                continue
            print(f"  j={j:2d} " + " ".join(f"{n}={(v - t0) if v else '-':>7}" for n, v in zip(names, row)))
