"""Sweep forced GEMM tile configs (RK_GEMM_OVERRIDE) on the full c2 step:
one bench.py subprocess per candidate, reporting the step time and the summed
time of the forced shape's launches (kernel_detail prefix match).
  python tools/gemm_override_sweep.py [set ...]   (sets: sparse, m320, band)"""
import json
import os
import subprocess
import sys

# shape key (RK_GEMM_OVERRIDE "M[d]:N:K"), kernel_detail name prefix, candidates bn/pair/splits
SETS = {
    "sparse": [
        ("4032d:3072:2048", "gemm_qkv_m4032dyn_n3072", ["128/2/1", "256/2/1", "64/2/1", "128/1/1", "256/1/1", "64/1/1"]),
        ("4032d:2048:2048", "gemm_add", ["128/2/1", "256/2/1", "64/2/1", "128/1/1", "256/1/1", "64/1/1", "256/1/2",
                                          "128/1/2"]),
        ("4032d:2048:8192", "gemm_add", ["256/1/3", "256/1/2", "256/1/4", "128/1/2", "128/1/3", "256/2/1", "128/2/1",
                                          "256/2/2", "256/2/3"]),
        ("4032d:16384:2048", "gemm_silu_m4032dyn", ["256/1/1", "256/2/1", "128/2/1", "128/1/1"]),
    ],
    "m320": [
        ("320:3072:2048", "gemm_qkv_m320", ["64/1/1", "128/1/1", "64/2/1", "128/2/1"]),
        ("320:2048:2048", "gemm_add", ["64/1/1", "128/1/1", "64/2/1", "128/2/1", "64/1/2", "128/1/2", "256/1/4"]),
        ("320:2048:8192", "gemm_add", ["256/1/6", "256/1/4", "256/1/8", "128/1/4", "128/1/6", "64/1/2", "64/1/4"]),
    ],
    "m320pair": [
        ("320:2048:8192", "gemm_add", ["256/1/6", "256/2/2", "256/2/4", "256/2/6", "128/2/4", "128/2/8"]),
        ("320:2048:2048", "gemm_add", ["64/1/1", "256/2/2", "128/2/2", "256/2/4", "64/2/2"]),
        ("4032d:2048:8192", "gemm_add", ["256/2/1", "256/2/2", "128/2/2", "256/2/3"]),
        ("4032d:2048:2048", "gemm_add", ["256/2/1", "256/2/2", "128/2/2"]),
    ],
    "sparse192": [
        ("4032d:2048:2048", "gemm_add", ["192/2/1", "256/2/1", "128/2/1", "64/2/1", "128/1/1", "128/1/2", "256/1/2"]),
        ("4032d:2048:8192", "gemm_add", ["192/2/1", "256/2/1", "128/2/1", "256/1/2", "256/1/3", "128/1/3"]),
        ("4032d:3072:2048", "gemm_qkv_m4032dyn_n3072", ["256/2/1", "192/2/1", "128/2/1"]),
        ("4032d:16384:2048", "gemm_silu_m4032dyn", ["192/2/1", "256/2/1", "128/2/1"]),
    ],
    "band": [
        ("4032:3072:2048", "gemm_qkv_m4032_", ["256/2/1", "128/2/1", "256/1/1"]),
        ("4032:2048:2048", "gemm_add", ["256/2/1", "128/2/1", "128/1/1", "256/1/1"]),
        ("4032:2048:8192", "gemm_add", ["256/2/1", "128/2/1", "256/1/2"]),
    ],
}


def run(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "bench.py", "--steps", "8", "--warmup", "3", "--no-cpu", "--exact-leg", "off"],
                       env=env, capture_output=True, text=True, timeout=600)
    try:
        return json.loads(r.stdout.strip().splitlines()[-1])
    except Exception:
        return {"error": (r.stdout + r.stderr)[-800:]}


def main():
    sets = sys.argv[1:] or ["sparse", "m320"]
    base = run({})
    print(json.dumps({"baseline": base.get("ms_per_step")}), flush=True)
    for st in sets:
        for key, prefix, cands in SETS[st]:
            for c in cands:
                d = run({"RK_GEMM_OVERRIDE": f"{key}={c}"})
                if "error" in d:
                    print(json.dumps({"shape": key, "cfg": c, "error": d["error"]}), flush=True)
                    continue
                kk = key.split(":")
                m_tag = ("m" + kk[0].rstrip("d") + ("dyn" if kk[0].endswith("d") else "")) + "_n" + kk[1] + "_k" + kk[2]
                tot = sum(x["ms"] for x in d.get("kernel_detail", []) if m_tag[:20] in x["name"] and
                          x["name"].startswith(prefix[:8]) and ("_k" + kk[2])[:3] in x["name"])
                print(json.dumps({"shape": key, "cfg": c, "step_ms": d["ms_per_step"], "shape_ms": round(tot, 4),
                                  "first_token": d.get("first_tokens"), "sel": d.get("selected_per_segment")}),
                      flush=True)


if __name__ == "__main__":
    main()
