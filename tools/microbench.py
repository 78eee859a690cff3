"""Device-resident microbenchmarks of the bf16 tensor-core kernels (CUDA events)."""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2603_13289_b200.engine import Engine, P, _check, lib  # noqa: E402


def attn(e, M, T, H, Hkv, dh, iters=20):
    ms = C.c_float()
    _check(lib().rk_debug_bench_attention(P(e.ptr), M, T, H, Hkv, dh, iters, C.byref(ms)))
    flops = 4.0 * dh * H * sum(p + 1 for p in range(T - M, T))
    return ms.value, flops / ms.value / 1e9


def gemm(e, M, N, K, epi=3, iters=20):
    ms = C.c_float()
    _check(lib().rk_debug_bench_gemm(P(e.ptr), M, N, K, epi, iters, C.byref(ms)))
    return ms.value, 2.0 * M * N * K / ms.value / 1e9


if __name__ == "__main__":
    e = Engine(0)
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "attn"):
        for case in [(4032, 4032, 32, 8, 64), (1856, 4032, 32, 8, 64), (64, 4032, 32, 8, 64), (4096, 4096, 32, 8, 128),
                     (2048, 8192, 32, 8, 128)]:
            ms, tf = attn(e, *case)
            print(f"attn M={case[0]} T={case[1]} H={case[2]} Hkv={case[3]} dh={case[4]}: {ms * 1e3:.1f} us  {tf:.1f} TFLOP/s", flush=True)
    if which in ("all", "gemm"):
        for case in [(4032, 2048, 2048, 1), (1356, 2048, 2048, 1), (320, 2048, 2048, 1), (1356, 2048, 8192, 1),
                     (4032, 3072, 2048, 0), (320, 3072, 2048, 0), (1356, 3072, 2048, 0),
                     (4032, 16384, 2048, 2), (4032, 2048, 8192, 1), (4032, 3072, 2048, 3), (320, 16384, 2048, 2),
                     (320, 2048, 8192, 1), (320, 3072, 2048, 3), (1356, 2048, 2048, 1), (8192, 8192, 8192, 3)]:
            ms, tf = gemm(e, *case)
            print(f"gemm M={case[0]} N={case[1]} K={case[2]} epi={case[3]}: {ms * 1e3:.1f} us  {tf:.1f} TFLOP/s", flush=True)


def c2_layout(kind, T=4032, n_pre=256, n_suf=64, sel=1040, seed=3):
    """Row layouts of the c2 step: 'pre_suf' (prefix + suffix rows only) or
    'sparse' (prefix | suffix | ~25% of the segment rows, live count on the device)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    pre, suf = np.arange(n_pre), np.arange(T - n_suf, T)
    if kind == "pre_suf":
        return np.concatenate([pre, suf]).astype(np.int32), n_pre + n_suf, n_pre, n_pre + n_suf, n_pre + n_suf
    seg = np.sort(rng.choice(np.arange(n_pre, T - n_suf), sel, replace=False))
    pos = np.zeros(T, np.int32)
    pos[:n_pre + n_suf + sel] = np.concatenate([pre, suf, seg])
    return pos, T, n_pre, n_pre + n_suf, n_pre + n_suf + sel


def attn_rows(e, kind, H=32, Hkv=8, dh=64, T=4032, iters=20):
    pos, M, g1, g2, live = c2_layout(kind, T)
    ms = C.c_float()
    _check(lib().rk_debug_bench_attention_rows(P(e.ptr), pos.ctypes.data_as(C.POINTER(C.c_int32)), M, live, g1, g2, T,
                                               H, Hkv, dh, iters, C.byref(ms)))
    flops = 4.0 * dh * H * float((pos[:live].astype(float) + 1).sum())
    return ms.value, flops / ms.value / 1e9


if __name__ == "__main__" and "rows" in sys.argv[1:]:
    e = Engine(0)
    for kind in ("pre_suf", "sparse"):
        ms, tf = attn_rows(e, kind)
        print(f"attn c2 {kind}: {ms * 1e3:.1f} us  {tf:.1f} TFLOP/s", flush=True)
