#!/usr/bin/env python
"""One-off measurement of the REFERENCE CPU path on the FULL c2 workload
("measure c2 once"), to validate the FLOP-model
extrapolation bench.py uses for its bounded CPU sample.

Same model (c2: L16 d2048 H32/8 dh64 ff8192 V128256, seed 1234), same
Reviewer prompt shape as bench.py (prefix 256 + 2 relayed segments x 1856 +
suffix 64 = 4032 tokens), profile (1,2,9), thresholds (1.5, 1.45, 10). The
two upstream caches are the reference's own decode-time captures
(ref_scenario_create: prefill the agent's 256-token prefix, greedy-decode
1856 tokens with RelayRecorder) -- the bench's GPU caches are teacher-forced
captures of synthetic outputs, so the token ids differ but every shape and
the profile are identical.

    python tools/cpu_full_c2.py capture 0 &   # the two captures run in parallel
    python tools/cpu_full_c2.py capture 1 &
    python tools/cpu_full_c2.py relay         # timed: one session, one core

Output: profiles/r02_cpu_full_c2.json. Test infrastructure: imports oracle/.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

CACHE = "/tmp/rk_c2_full_cache_{}.rkrc"


def main():
    stage = sys.argv[1]
    bench.set_workload("c2")
    orc = Oracle("reference")
    t0 = time.time()
    w = orc.weights(bench.spec_obj(), bench.SEED, checked=True)
    print(f"weights {time.time() - t0:.1f}s", flush=True)
    pr = bench.prompts(0)
    snap = bench.WL["profile"][0]
    if stage == "capture":
        a = int(sys.argv[2])
        t0 = time.time()
        host = orc.scenario(w, pr[f"a{a}_prefix"], bench.WL["segment"], snap)
        orc.save_cache(host, CACHE.format(a))
        print(f"capture {a}: {time.time() - t0:.1f}s", flush=True)
        return
    caches = [orc.load_cache(CACHE.format(a)) for a in range(bench.WL["agents"] - 1)]
    prof, opts = bench.options()
    last = bench.WL["agents"] - 1
    prefix, suffix = pr[f"a{last}_prefix"], pr[f"a{last}_suffix"]
    tokens = len(prefix) + sum(c.segment_len for c in caches) + len(suffix)
    t0 = time.perf_counter()
    logits, tok, ctx = orc.agent_prefill(w, prefix, caches, suffix, prof, opts)
    ms = (time.perf_counter() - t0) * 1e3
    segs = orc.ctx_segments(ctx)
    spec = bench.spec_obj()
    selected = [int(s[2][prof.l_det + 1].sum()) for s in segs]
    flops = bench.reference_work(spec, len(prefix), [c.segment_len for c in caches], len(suffix), selected,
                                 bench.WL["profile"])
    out = {
        "what": "reference CPU path (oracle/_ref, the reference library built from its sources), FULL c2 "
                "Reviewer TTFT, one session on one core",
        "workload": f"c2 model, prefix {len(prefix)} + {len(caches)} x {bench.WL['segment']} + suffix {len(suffix)} "
                    f"= {tokens} tokens, profile {bench.WL['profile']}",
        "ttft_ms": round(ms, 1), "tokens_per_s_one_core": round(tokens / (ms / 1e3), 4),
        "flops_model": flops, "gflops_per_s": round(flops / (ms / 1e3) / 1e9, 3),
        "selected_per_segment": selected,
        "first_token": int(tok), "host": bench.host_info(),
        "measured_in": "build container (no GPU), 2026-10",
    }
    path = os.path.join(ROOT, "profiles", "r02_cpu_full_c2.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
