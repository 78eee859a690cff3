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
        for case in [(4032, 16384, 2048, 2), (4032, 2048, 8192, 1), (4032, 3072, 2048, 3), (320, 16384, 2048, 2),
                     (320, 2048, 8192, 1), (320, 3072, 2048, 3), (1356, 2048, 2048, 1), (8192, 8192, 8192, 3)]:
            ms, tf = gemm(e, *case)
            print(f"gemm M={case[0]} N={case[1]} K={case[2]} epi={case[3]}: {ms * 1e3:.1f} us  {tf:.1f} TFLOP/s", flush=True)
