"""Probe: host-side timing of async cache upload vs relay prefill (diagnostic)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from bench import SEED, build_session, options, pin_host, spec_obj  # noqa: E402

bench.set_workload(sys.argv[1] if len(sys.argv) > 1 else "c2")
import torch  # noqa: E402

from paper_2603_13289_b200.engine import Engine  # noqa: E402

torch.cuda.set_device(0)
eng = Engine(0)
w = eng.weights(spec_obj(), SEED, "bf16")
sess = build_session(w, 0)
prof, opts = options()
hosts = [pin_host(c.to_host()) for c in sess["caches"]]
ctx = sess["ctx"]


def run(tag, asynchronous, wait_first):
    for it in range(5):
        t0 = time.perf_counter()
        ups = [w.upload_cache(h, asynchronous=asynchronous) for h in hosts]
        if wait_first and asynchronous:
            for c in ups:
                c.wait()
        t1 = time.perf_counter()
        ctx.reset()
        out = ctx.agent_prefill(sess["prefix"], ups, sess["suffix"], prof, opts, want_logits=True, outputs=True)
        t2 = time.perf_counter()
        del ups
    wall = out["segments"][0]["stats"].get("wall")
    print(f"{tag}: upload {1e3 * (t1 - t0):.2f} ms, prefill {1e3 * (t2 - t1):.2f} ms, total {1e3 * (t2 - t0):.2f}; "
          f"device phases {wall}")


run("sync upload", False, False)
run("async, wait first", True, True)
run("async overlapped", True, False)
eng.set_fused(False)
run("async overlapped, sequential schedule", True, False)
