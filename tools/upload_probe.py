"""Per-iteration timing of the asynchronous cache upload alone (bench.py's upload_only diagnostic)."""
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2603_13289_b200.engine import Engine  # noqa: E402

eng = Engine(0)
w = eng.weights(bench.spec_obj(), bench.SEED, "bf16")
sess = bench.build_session(w, 0)
hosts = [bench.pin_host(c.to_host()) for c in sess["caches"]]
prof, opts = bench.options()
def e2e_step():
    ups = [w.upload_cache(h, asynchronous=True) for h in hosts]
    sess["ctx"].reset()
    return sess["ctx"].agent_prefill(sess["prefix"], ups, sess["suffix"], prof, opts, want_logits=True)["first_token"]


for i in range(6):  # bench.py's e2e loop first
    t0 = time.perf_counter()
    e2e_step()
    print(f"e2e {i}: {1e3*(time.perf_counter()-t0):.2f} ms", flush=True)
for i in range(8):
    t0 = time.perf_counter()
    ups = [w.upload_cache(h, asynchronous=True) for h in hosts]
    t1 = time.perf_counter()
    for c in ups:
        c.wait()
    t2 = time.perf_counter()
    del ups
    t3 = time.perf_counter()
    print(f"iter {i}: enqueue {1e3*(t1-t0):.2f} ms, wait {1e3*(t2-t1):.2f} ms, destroy {1e3*(t3-t2):.2f} ms", flush=True)
    if i == 3:  # one relay step in between, as in bench.py
        sess["ctx"].reset()
        sess["ctx"].agent_prefill(sess["prefix"], [w.upload_cache(h, asynchronous=True) for h in hosts],
                                  sess["suffix"], prof, opts, want_logits=True)
