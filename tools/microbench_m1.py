import sys; sys.path.insert(0, ".")
from tools.microbench import gemm, attn, Engine
e = Engine(0)
for (M, N, K, epi) in [(1, 2048, 2048, 1), (1, 16384, 2048, 2), (1, 2048, 8192, 1), (1, 128256, 2048, 3), (1, 3072, 2048, 0)]:
    for it in (1, 20):
        ms, tf = gemm(e, M, N, K, epi, it)
        print(f"gemv M={M} N={N} K={K} epi={epi} iters={it}: {ms*1e3:.2f} us  {N*K*2/ms/1e9:.0f} GB/s", flush=True)
for it in (1, 20):
    ms, tf = attn(e, 1, 4032, 32, 8, 64, it)
    print(f"attn M=1 T=4032 iters={it}: {ms*1e3:.2f} us", flush=True)
