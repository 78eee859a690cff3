"""Time the c2 (and c3) GEMM shapes of one relay step under several GEMM
policies (env settings read once per process, so one subprocess each).
Weights rotate over >= 256 MB of copies (streamed from HBM as in the step).
  python tools/gemm_sweep.py [ENV=VAL,ENV=VAL ...]   (one policy per argument)"""
import json
import os
import subprocess
import sys

SHAPES = {
    "m320": [(320, 3072, 2048, 3), (320, 2048, 2048, 1), (320, 16384, 2048, 2), (320, 2048, 8192, 1)],
    "c2": [  # (M, N, K, epi): 0 qkv-shaped store, 1 residual, 2 silu, 3 store
        (320, 3072, 2048, 3), (320, 2048, 2048, 1), (320, 16384, 2048, 2), (320, 2048, 8192, 1),
        (1360, 3072, 2048, 3), (1360, 2048, 2048, 1), (1360, 16384, 2048, 2), (1360, 2048, 8192, 1),
        (4032, 3072, 2048, 3), (4032, 2048, 2048, 1), (4032, 16384, 2048, 2), (4032, 2048, 8192, 1)],
    "c3": [(320, 6144, 4096, 3), (320, 4096, 4096, 1), (320, 28672, 4096, 2), (320, 4096, 14336, 1)],
}

CHILD = r"""
import json, sys
sys.path.insert(0, ".")
from tools.microbench import gemm
from paper_2603_13289_b200.engine import Engine
e = Engine(0)
out = []
for (M, N, K, epi) in json.loads(sys.argv[1]):
    gemm(e, M, N, K, epi, iters=3)
    ms, tf = gemm(e, M, N, K, epi, iters=30)
    out.append(dict(M=M, N=N, K=K, epi=epi, us=round(ms * 1e3, 2), tflops=round(tf, 1)))
print("RESULT " + json.dumps(out))
"""


def main():
    policies = sys.argv[1:] or ["RK_GEMM_SWAP=0", "RK_GEMM_SWAP=2"]
    which = os.environ.get("SWEEP_SET", "c2,c3").split(",")
    shapes = [x for w in which for x in SHAPES[w]]
    for pol in policies:
        env = dict(os.environ)
        for kv in pol.split(","):
            if kv:
                k, v = kv.split("=")
                env[k] = v
        r = subprocess.run([sys.executable, "-c", CHILD, json.dumps(shapes)], env=env, capture_output=True, text=True,
                           timeout=600)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
        if not line:
            print(pol, "FAILED", r.stdout[-2000:], r.stderr[-2000:])
            continue
        for rec in json.loads(line[0][7:]):
            rec["policy"] = pol
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
