"""BASELINE config 5: recompute-ratio x reused-segment-length sweep on the
Llama-3-8B shape, against the full-recompute prefill.

  python tools/sweep.py [--lengths 1024,2048,...] [--ratios 0.05,0.1,...] [--steps 3] > sweep.jsonl

One downstream agent relays one upstream segment of N tokens (captured on the
device), prefix 256 + suffix 64. Recompute ratio = BLEND's blend_alpha with
top_k_by_score (relay_engine.cpp:318-332; the reference's only ratio knob);
RELAY (threshold selection, tau_dev swept) reports its achieved ratio;
FULL = prefill of the whole prompt. TTFT is CUDA-event device time per call.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_13289_b200.abi import LayerProfile, ModelSpec, RelayOptions  # noqa: E402

SPEC = dict(num_layers=32, d_model=4096, num_heads=32, num_kv_heads=8, d_head=128, d_ff=14336,
            vocab_size=128256, theta_base=500000.0)
PROFILE = (1, 3, 18)  # PAPER.md:867 (Llama-3.1-8B)
PREFIX, SUFFIX = 256, 64


def tokens(seed, n, vocab):
    rng = np.random.default_rng(seed)
    return rng.integers(0, vocab, n).astype(np.int32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lengths", default="1024,2048,4096,8192,16384,32768")
    ap.add_argument("--ratios", default="0.05,0.1,0.2,0.3,0.5")
    ap.add_argument("--taus", default="1.0,1.5,2.0")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    args = ap.parse_args()
    import torch

    from paper_2603_13289_b200.engine import Engine, flops_segment_schedule, flops_span_full
    lengths = [int(x) for x in args.lengths.split(",")]
    maxpos = 2 * PREFIX + max(lengths) + SUFFIX + 64
    spec = ModelSpec.make(SPEC["num_layers"], SPEC["d_model"], SPEC["num_heads"], SPEC["num_kv_heads"],
                          SPEC["d_head"], SPEC["d_ff"], SPEC["vocab_size"], SPEC["theta_base"], maxpos)
    eng = Engine(0)
    w = eng.weights(spec, 1234, "bf16")
    stream = torch.cuda.ExternalStream(eng.stream)
    V = SPEC["vocab_size"]

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        eng.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            out = fn()
        t1.record(stream)
        t1.synchronize()
        return t0.elapsed_time(t1) / args.steps, out

    for n in lengths:
        up = w.context()
        up.prefill(tokens(1, PREFIX, V), logits=False)
        cache = up.capture_prefill(tokens(2, n, V), PROFILE[0])
        del up
        ctx = w.context()
        prefix, suffix = tokens(3, PREFIX, V), tokens(4, SUFFIX, V)
        total = PREFIX + n + SUFFIX

        def run(opts, prof=LayerProfile(*PROFILE), outputs=False):
            def f():
                ctx.reset()
                return ctx.agent_prefill(prefix, [cache], suffix, prof, opts, want_logits=False, outputs=outputs)
            return f

        full_ms, _ = timed(run(RelayOptions.make(mode="full")))
        full_flops = flops_span_full(spec, 0, total) + 2.0 * spec.d_model * spec.vocab_size
        rec = {"config": "c5", "n": n, "mode": "full", "ttft_ms": round(full_ms, 3),
               "tokens_per_s": round(total / (full_ms / 1e3), 1), "tflops": round(full_flops / full_ms / 1e9, 1)}
        print(json.dumps(rec), flush=True)
        for r in [float(x) for x in args.ratios.split(",")]:
            ms, _ = timed(run(RelayOptions.make(mode="blend", blend_alpha=r), LayerProfile()))
            out = run(RelayOptions.make(mode="blend", blend_alpha=r), LayerProfile(), True)()
            st = out["segments"][0]["stats"]
            sel = out["segments"][0]["selection_count"]
            print(json.dumps({"config": "c5", "n": n, "mode": "blend", "ratio": r, "selected": int(sel),
                              "reuse_rate": round(st["reuse_rate"], 4), "ttft_ms": round(ms, 3),
                              "speedup_vs_full": round(full_ms / ms, 3),
                              "tokens_per_s": round(total / (ms / 1e3), 1)}), flush=True)
        for tau in [float(x) for x in args.taus.split(",")]:
            opts = RelayOptions.make(mode="relay", tau_dev=tau, tau_inf=1.45, suffix_k=10)
            ms, _ = timed(run(opts))
            out = run(opts, outputs=True)()
            seg = out["segments"][0]
            st = seg["stats"]
            sel = int(seg["selection_count"])
            flops = (flops_span_full(spec, 0, PREFIX) + st["flops_cost"] + flops_span_full(spec, PREFIX + n, SUFFIX)
                     + 2.0 * spec.d_model * spec.vocab_size)
            print(json.dumps({"config": "c5", "n": n, "mode": "relay", "tau_dev": tau, "selected": sel,
                              "recompute_ratio": round(sel / n, 4), "reuse_rate": round(st["reuse_rate"], 4),
                              "ttft_ms": round(ms, 3), "speedup_vs_full": round(full_ms / ms, 3),
                              "tokens_per_s": round(total / (ms / 1e3), 1),
                              "analytic_tflop": round(flops / 1e12, 3),
                              "tflops": round(flops / ms / 1e9, 1)}), flush=True)
        del cache, ctx


if __name__ == "__main__":
    main()
