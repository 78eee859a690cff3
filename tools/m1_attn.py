import sys; sys.path.insert(0, ".")
from tools.microbench import attn, Engine
e = Engine(0)
for T in (4032, 1000):
    ms, tf = attn(e, 1, T, 32, 8, 64, 5)
    print(f"attn M=1 T={T}: {ms*1e3:.2f} us", flush=True)
