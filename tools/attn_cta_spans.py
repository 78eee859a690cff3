"""Per-CTA global-timer spans of one attention launch (rk_debug_trace_attention_rows)
over the c2 row layouts: launch span, when CTAs start, how long each runs.
  python tools/attn_cta_spans.py [pre_suf|sparse|suffix64|prefix256 ...]"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2603_13289_b200.engine import Engine, P, _check, lib  # noqa: E402
from tools.microbench import c2_layout  # noqa: E402


def layout(kind, T=4032):
    if kind == "suffix64":
        pos = np.arange(T - 64, T, dtype=np.int32)
        return pos, 64, 64, 64, 64
    if kind == "prefix256":
        pos = np.arange(256, dtype=np.int32)
        return pos, 256, 256, 256, 256
    return c2_layout(kind, T)


def spans(e, kind, H=32, Hkv=8, dh=64, T=4032, max_ctas=1 << 15):
    pos, M, g1, g2, live = layout(kind, T)
    out = np.zeros(1536 + 4 * max_ctas, np.uint64)
    n = C.c_int()
    _check(lib().rk_debug_trace_attention_rows(P(e.ptr), pos.ctypes.data_as(C.POINTER(C.c_int32)), M, live, g1, g2,
                                                T, H, Hkv, dh, out.ctypes.data_as(C.POINTER(C.c_uint64)), max_ctas,
                                                C.byref(n)))
    ev = out[:1536].reshape(3, 64, 8).astype(np.int64)
    t = out[1536:].reshape(-1, 4).astype(np.int64)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    entry, wait, end = t[:, 0] - t0, t[:, 1] - t0, t[:, 2] - t0
    nk, partial, parts, rows = t[:, 3] & 0xFF, (t[:, 3] >> 8) & 1, (t[:, 3] >> 16) & 0xFFFF, t[:, 3] >> 32
    print(f"{kind}: {len(t)} live CTAs, launch span {end.max() / 1e3:.2f} us (first entry -> last end)")
    q = lambda x: " ".join(f"{v / 1e3:6.2f}" for v in np.percentile(x, [0, 10, 50, 90, 100]))
    print(f"  entry      (p0 p10 p50 p90 p100, us): {q(entry)}")
    print(f"  wait done  : {q(wait - entry)}")
    print(f"  run        : {q(end - wait)}")
    print(f"  end        : {q(end)}")
    for k in sorted(set(nk.tolist())):
        sel = nk == k
        print(f"  nk={k:2d}: {sel.sum():4d} CTAs (partial {int(partial[sel].sum())}), run p50 "
              f"{np.median(end[sel] - wait[sel]) / 1e3:.2f} us, max {(end[sel] - wait[sel]).max() / 1e3:.2f}")
    pm = ev[1, 0]  # CTA (0,0,0): entry, prologue done, TMEM ready, last O, partial ticket, output done, end
    if pm[0]:
        names = ["entry", "pos/kmax", "tmem+bar", "last O", "ticket", "out done", "end"]
        print("  CTA(0,0,0) clocks from entry: " + " ".join(f"{n}={pm[i] - pm[0] if pm[i] else '-'}"
                                                          for i, n in enumerate(names)))
        sm = ev[0]
        js = [j for j in range(64) if sm[j, 1]]
        if js:
            print(f"  first loop start {sm[js[0], 0] - pm[0]}, first S full {sm[js[0], 1] - pm[0]}, "
                  f"last P stored {sm[js[-1], 4] - pm[0]} ({len(js)} blocks)")
    return t


if __name__ == "__main__":
    e = Engine(0)
    for kind in sys.argv[1:] or ["pre_suf", "suffix64", "prefix256", "sparse"]:
        spans(e, kind)
