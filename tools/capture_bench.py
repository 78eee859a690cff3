"""Decode-time capture on the device (RelayRecorder, relay_cache.cpp:68-127):
greedy-decode N tokens after a prompt, recording K_pre, V, the snapshot hidden
row and influence, at the c2 / c3 model shapes. Prints tokens/s."""
import json
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2603_13289_b200.engine import Engine  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    bench.set_workload(cfg)
    eng = Engine(0)
    w = eng.weights(bench.spec_obj(), bench.SEED, "bf16")
    pr = bench.prompts(0)
    for rep in range(2):
        ctx = w.context()
        logits = ctx.prefill(pr["a0_prefix"])
        eng.synchronize()
        t0 = time.perf_counter()
        c = ctx.capture_decode(logits, n, bench.WL["profile"][0])
        eng.synchronize()
        dt = time.perf_counter() - t0
        del c, ctx
    print(json.dumps({"config": cfg, "decode_tokens": n, "ms": round(dt * 1e3, 2),
                      "tokens_per_s": round(n / dt, 1), "ms_per_token": round(dt * 1e3 / n, 3)}))


if __name__ == "__main__":
    main()
