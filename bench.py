#!/usr/bin/env python
"""Benchmark: downstream-agent TTFT and relay-prefill tokens/s (BASELINE.json
metric). Default workload: BASELINE config 2 -- a Llama-3.2-1B-shaped
random-init model, the 3-agent Architect/Developer/Reviewer chain with ~4K
accumulated context. --config c3 (Llama-3-8B shape, 8-turn chain, 16K context)
and c4 (Qwen2.5-7B shape, 64 sessions sharded over the GPUs) run the larger
BASELINE configs. One process per GPU, sessions sharded, weak scaling, no
data-path collective.

One step = the last agent's TTFT sequence through the engine (run_workflow's
relay branch, workflow.cpp:316-369): prefix prefill -> relay_extend of every
upstream agent's decode-time cache -> suffix prefill -> last-row logits ->
argmax, first token read back on the host.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|c3|c4]

Prints ONE JSON line on rank 0.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2603_13289_b200.abi import LayerProfile, ModelSpec, RelayOptions  # noqa: E402

# ---- workloads (BASELINE.json configs) --------------------------
# The default (c2) is the config the metric is quoted on; c3/c4 are the larger
# single-GPU shapes, run with --config (the driver runs the default).
WORKLOADS = {
    "c2": dict(title="c2: Llama-3.2-1B-shaped random init (L16 d2048 H32/8 dh64 ff8192 V128256), "
                     "Architect->Developer->Reviewer chain",
               spec=dict(num_layers=16, d_model=2048, num_heads=32, num_kv_heads=8, d_head=64, d_ff=8192,
                         vocab_size=128256, theta_base=500000.0, max_positions=8192),
               agents=3, prefix=256, segment=1856, suffix=64, profile=(1, 2, 9), cpu=(4, 4, 2)),
    "c3": dict(title="c3: Llama-3-8B-shaped bf16 GQA random init (L32 d4096 H32/8 dh128 ff14336 V128256), "
                     "8-turn chain",
               spec=dict(num_layers=32, d_model=4096, num_heads=32, num_kv_heads=8, d_head=128, d_ff=14336,
                         vocab_size=128256, theta_base=500000.0, max_positions=16384),
               agents=8, prefix=256, segment=2240, suffix=64, profile=(1, 3, 18), cpu=(2, 1, 1)),
    "c4": dict(title="c4: Qwen2.5-7B-shaped random init (L28 d3584 H28/4 dh128 ff18944 V152064), "
                     "3-agent chain per session",
               spec=dict(num_layers=28, d_model=3584, num_heads=28, num_kv_heads=4, d_head=128, d_ff=18944,
                         vocab_size=152064, theta_base=1000000.0, max_positions=8192),
               agents=3, prefix=256, segment=1856, suffix=64, profile=(3, 4, 22), cpu=(2, 1, 1), sessions=64),
}
WL = WORKLOADS["c2"]
SEED = 1234


def set_workload(name):
    global WL
    WL = WORKLOADS[name]


def spec_obj():
    S = WL["spec"]
    return ModelSpec.make(S["num_layers"], S["d_model"], S["num_heads"], S["num_kv_heads"], S["d_head"], S["d_ff"],
                          S["vocab_size"], S["theta_base"], S["max_positions"])


def prompt_tokens():
    """Tokens in the downstream agent's prompt: prefix + upstream segments + suffix."""
    return WL["prefix"] + (WL["agents"] - 1) * WL["segment"] + WL["suffix"]


def synthetic_tokens(seed, salt, count, vocab):
    """metrics.cpp:255-263 (vectorised SplitMix64)."""
    state = np.uint64((seed ^ ((salt * 0x9E3779B97F4A7C15 + 0x1234567) & 0xFFFFFFFFFFFFFFFF)))
    with np.errstate(over="ignore"):
        z = state + np.arange(1, count + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z % np.uint64(vocab)).astype(np.int32)


def prompts(session=0):
    """Per agent a: prefix, suffix and its output segment (captured as its cache)."""
    V = WL["spec"]["vocab_size"]
    base = SEED + 7919 * session
    out = {}
    for a in range(WL["agents"]):
        out[f"a{a}_prefix"] = synthetic_tokens(base, 3 * a, WL["prefix"], V)
        out[f"a{a}_suffix"] = synthetic_tokens(base, 3 * a + 1, WL["suffix"], V)
        out[f"a{a}_out"] = synthetic_tokens(base, 3 * a + 2, WL["segment"], V)
    return out


def options(mode="relay"):
    return LayerProfile(*WL["profile"]), RelayOptions.make(mode=mode, tau_dev=1.5, tau_inf=1.45, suffix_k=10)


# ---- clocks -------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, device):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "samples": len(self.rows), "reasons": reasons}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p["bf16_tflops_sustained"], "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ---- distributed plumbing (torch.distributed over NCCL; results gather only) --
def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "ours":
            torch.cuda.set_device(local)
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")
    return world, rank, local, dist


def reduce_max(dist, value, local):
    if dist is None:
        return value
    import torch
    dev = f"cuda:{local}" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(argv, gpus):
    """`python bench.py --gpus N` outside torchrun: re-launch this script as N
    ranks (one process per GPU, torch.distributed.run on 127.0.0.1) and pass
    rank 0's JSON line through. Returns the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + argv
    return subprocess.call(cmd)


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ---- the reference CPU path ------------------------------------------------------
def reference_work(spec, prefix, seg_lens, suffix, selected, profile):
    """FLOPs the reference spends on the downstream agent's TTFT, by its own
    FLOP model (relay_engine.cpp:72-128: flops_span_full for the prefix and
    suffix prefills, flops_segment_schedule per relayed segment at its base)
    plus the all-row logits its prefill computes (model.cpp:328, 2*d*V per
    prefix and suffix row; the engine computes only the last row). The CPU
    reference is a plain i-k-j fp32 loop (tensor.cpp:66-86) whose time per
    FLOP barely depends on the shape, which is what makes a bounded sample
    extrapolate (checked against a full c2 run: profiles/r02_cpu_full_c2.json)."""
    d, kv, ff = spec.d_model, spec.num_kv_heads * spec.d_head, spec.d_ff
    L, dhH, V = spec.num_layers, spec.d_head * spec.num_heads, spec.vocab_size
    pm = 2.0 * d * (2.0 * d + 2.0 * kv) + 6.0 * d * ff

    def attn(b, n):
        return 4.0 * dhH * (n * b + n * (n + 1.0) / 2.0)

    def span(b, n):
        return L * n * pm + L * attn(b, n)

    l_start, l_det, l_end = profile
    total, base = span(0, prefix), prefix
    for n, sel in zip(seg_lens, selected):
        avg = base + (n + 1.0) / 2.0
        total += (l_det - l_start + 1) * (n * pm + attn(base, n)) + (l_end - l_det) * sel * (pm + 4.0 * dhH * avg)
        base += n
    total += span(base, suffix)
    total += 2.0 * d * V * (prefix + suffix)
    return total


def full_c2_reference_run():
    """The committed one-off run of the reference on the FULL c2 prompt (tools/cpu_full_c2.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_cpu_full_c2.json")) as f:
            return json.load(f)
    except Exception:
        return None


def cpu_sample(gpu_caches=None, threads=None, steps=1, warmup=0, kind="reference", full_selected=None):
    """Time the reference's own relay path (oracle/_ref: the reference library
    built from its sources) -- or the restatement if _ref is absent -- on a
    bounded sample of the workload: same model, prefix/segments/suffix cut to
    WL["cpu"] tokens. One session on one core (latency), then one independent
    session per host core (throughput). Both are extrapolated to the FULL
    prompt of the GPU arm with the reference's FLOP model (reference_work),
    and labelled as such. Returns (full-prompt tokens/s on all cores, meta)."""
    from oracle.oracle import Oracle, available
    if kind == "reference" and not available("reference"):
        kind = "restatement"
    orc = Oracle(kind)
    spec = spec_obj()
    w = orc.weights(spec, SEED, checked=(kind == "reference"))
    pr = prompts(0)
    cp, cs, cx = WL["cpu"]
    last = WL["agents"] - 1
    if gpu_caches is None:  # the reference's own decode-time captures of the cut segments
        caches = [orc.scenario(w, pr[f"a{a}_prefix"][:cp], cs, WL["profile"][0]) for a in range(last)]
    else:
        caches = []
        for host in gpu_caches:
            c = host.copy()
            c.segment_tokens = c.segment_tokens[:cs].copy()
            c.k_pre = np.ascontiguousarray(c.k_pre[:, :cs])
            c.v = np.ascontiguousarray(c.v[:, :cs])
            c.hidden_snapshot = np.ascontiguousarray(c.hidden_snapshot[:cs])
            c.influence = np.ascontiguousarray(c.influence[:cs])
            c.decode_steps_observed = cs
            caches.append(c)
    prof, opts = options()
    prefix, suffix = pr[f"a{last}_prefix"][:cp], pr[f"a{last}_suffix"][:cx]
    tokens = len(prefix) + sum(c.segment_len for c in caches) + len(suffix)
    # one core, one session (also yields the sample's selection for its work figure)
    t0 = time.perf_counter()
    _, _, ctx = orc.agent_prefill(w, prefix, caches, suffix, prof, opts)
    ms1 = (time.perf_counter() - t0) * 1e3
    l_det = WL["profile"][1]
    sel = [int(sg[2][l_det + 1].sum()) if l_det + 1 < spec.num_layers else 0 for sg in orc.ctx_segments(ctx)]
    work_sample = reference_work(spec, len(prefix), [c.segment_len for c in caches], len(suffix), sel, WL["profile"])
    threads = threads or (os.cpu_count() or 1)
    times = []
    for i in range(warmup + steps):
        if kind == "reference":
            ms, _ = orc.agent_prefill_parallel(w, threads, prefix, caches, suffix, prof, opts)
            used = threads
        else:
            ms, used = ms1, 1
        if i >= warmup:
            times.append(ms)
    ms = sum(times) / len(times)
    # the full prompt of the GPU arm
    n_full = prompt_tokens()
    full_sel = full_selected or [int(round(0.25 * WL["segment"]))] * last
    work_full = reference_work(spec, WL["prefix"], [WL["segment"]] * last, WL["suffix"], full_sel, WL["profile"])
    scale = work_full / work_sample
    ttft1_ms = ms1 * scale           # one session, one core
    ttftN_ms = ms * scale            # `used` concurrent sessions (memory-bandwidth shared)
    tps = used * n_full / (ttftN_ms / 1e3)
    meta = {"kind": "reference" if kind == "reference" else "port", "cores": used,
            "extrapolated": True,
            "sample": f"{WL['title'].split(':')[0]} model, measured on prefix {cp} + {len(caches)} relayed segments x "
                      f"{cs} + suffix {cx} = {tokens} tokens per session ({used} concurrent sessions); extrapolated "
                      f"to the GPU arm's {n_full}-token prompt by the reference's FLOP model (relay_engine.cpp:72-128 "
                      f"+ all-row prefill logits): x{scale:.1f} work",
            "sample_ms_per_session": round(ms, 3), "sample_ms_one_core": round(ms1, 3),
            "sample_tokens_per_s": round(used * tokens / (ms / 1e3), 4),
            "sample_gflop_per_s_per_core": round(work_sample / (ms1 / 1e3) / 1e9, 3),
            "full_prompt_selected_per_segment": full_sel,
            "full_prompt_ttft_ms_one_core_extrapolated": round(ttft1_ms, 1),
            "full_prompt_ttft_ms_all_cores_extrapolated": round(ttftN_ms, 1),
            "host": host_info()}
    ref = full_c2_reference_run() if WL is WORKLOADS["c2"] else None
    if ref:
        meta["full_prompt_measured_once"] = {k: ref.get(k) for k in ("ttft_ms", "tokens_per_s_one_core",
                                                                    "gflops_per_s", "first_token", "workload",
                                                                    "host", "measured_in")}
        if ref.get("sample_gflop_per_s_same_host"):
            # the sample runs less efficiently per FLOP than the full prompt (small
            # matrices): scale the extrapolated time by the ratio both measured
            # on one host (profiles/r02_cpu_full_c2.json)
            f = ref["sample_gflop_per_s_same_host"] / ref["gflops_per_s"]
            tps /= f
            meta["calibrated_by_full_run"] = round(f, 4)
            meta["full_prompt_ttft_ms_one_core_extrapolated"] = round(ttft1_ms * f, 1)
            meta["full_prompt_ttft_ms_all_cores_extrapolated"] = round(ttftN_ms * f, 1)
    return tps, meta


def host_info():
    """The host the CPU arm ran on (the oracle's glibc expf/cos/sin are part of
    the reference's numerics)."""
    import platform
    cpu = ""
    try:
        with open("/proc/cpuinfo") as f:
            cpu = next((l.split(":", 1)[1].strip() for l in f if l.startswith("model name")), "")
    except OSError:
        pass
    return {"cpu": cpu, "logical_cpus": os.cpu_count(), "libc": "-".join(platform.libc_ver())}


def pin_host(host):
    """Move a HostRelayCache's arrays into page-locked memory (torch pinned
    tensors; the tensors are kept alive on the object)."""
    import torch
    keep = []
    for f in ("segment_tokens", "k_pre", "v", "hidden_snapshot", "influence"):
        a = getattr(host, f)
        t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
        t.numpy()[...] = a
        keep.append(t)
        setattr(host, f, t.numpy())
    host._pinned = keep
    return host


def merge_kernel_stats(stats):
    """Collapse per-shape labels (gemm_qkv_m320_..., attn_m...) into kernel families."""
    fam = {}
    for k in stats:
        name = "gemm_bf16_tcgen05" if k["name"].startswith("gemm") else \
            "gemv_bf16" if k["name"].startswith("gemv") else \
            "attention_bf16_tcgen05" if k["name"].startswith("attn") else k["name"]
        f = fam.setdefault(name, {"name": name, "launches": 0, "total_ms": 0.0, "flops": 0.0, "bytes": 0.0})
        for key in ("launches", "total_ms", "flops", "bytes"):
            f[key] += k[key]
    return list(fam.values())


# ---- our engine ------------------------------------------------------------------
def build_session(w, session):
    """One collaboration session: the decode-time caches of agents 0..A-2
    (captured on the device; each agent relays all upstream segments,
    workflow.cpp:285-288) and the last agent's prompt parts."""
    pr = prompts(session)
    prof, opts = options()
    snap = WL["profile"][0]
    caches = []
    for a in range(WL["agents"] - 1):
        ctx = w.context()
        if caches:
            ctx.agent_prefill(pr[f"a{a}_prefix"], caches, pr[f"a{a}_suffix"], prof, opts, want_logits=False)
        else:
            ctx.prefill(pr[f"a{a}_prefix"], logits=False)
        caches.append(ctx.capture_prefill(pr[f"a{a}_out"], snap))
        del ctx
    last = WL["agents"] - 1
    return {"caches": caches, "prefix": pr[f"a{last}_prefix"], "suffix": pr[f"a{last}_suffix"],
            "ctx": w.context(), "session": session}


def _rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def exact_leg(eng, w, timed):
    """The fp32-exact mode (bit-identical to the reference: tests/test_gpu_wide.py
    at c2/c3 width) on the SAME workload: its TTFT, and the bf16 throughput
    mode's own error against it on the same relay caches (north_star: "a bf16
    throughput mode reports its own max error"): logits, first token, per
    segment selection Jaccard and |I|, K/V and segment hidden rel-L2."""
    wx = eng.weights(spec_obj(), SEED, "fp32")
    sx = build_session(wx, 0)  # fp32-exact captures of the upstream agents' segments
    hosts = [c.to_host() for c in sx["caches"]]
    prof, opts = options()

    def run(ctx, caches, outputs=False):
        ctx.reset()
        return ctx.agent_prefill(sx["prefix"], caches, sx["suffix"], prof, opts, want_logits=True, outputs=outputs)

    rx = run(sx["ctx"], sx["caches"], True)
    dev_ms, _, launches = timed(lambda: run(sx["ctx"], sx["caches"]), 2, 1)
    Kx, Vx = sx["ctx"].all()
    cb = [w.upload_cache(h) for h in hosts]
    ctxb = w.context()
    rb = run(ctxb, cb, True)
    Kb, Vb = ctxb.all()
    segs = []
    for sb, sxg in zip(rb["segments"], rx["segments"]):
        a, b = set(int(i) for i in sb["selection"]), set(int(i) for i in sxg["selection"])
        segs.append({"selected_bf16": len(a), "selected_exact": len(b),
                     "selection_jaccard": round(len(a & b) / max(1, len(a | b)), 4),
                     "hidden_rel_l2": _rel_l2(sb["hidden"][sb["depth"] == sxg["depth"]],
                                              sxg["hidden"][sb["depth"] == sxg["depth"]]),
                     "s_dev_max_abs": float(np.max(np.abs(sb["s_dev"] - sxg["s_dev"])))})
    err = {
        "against": "fp32-exact run of the same prompt and relay caches (bit-equal to the reference CPU path)",
        "logits_max_abs": float(np.max(np.abs(rb["logits"].astype(np.float64) - rx["logits"]))),
        "logits_rel_l2": _rel_l2(rb["logits"], rx["logits"]),
        "first_token_match": rb["first_token"] == rx["first_token"],
        "k_rel_l2": _rel_l2(Kb, Kx), "v_rel_l2": _rel_l2(Vb, Vx),
        "kv_max_abs": float(max(np.max(np.abs(Kb - Kx)), np.max(np.abs(Vb - Vx)))),
        "segments": segs,
    }
    n_tokens = prompt_tokens()
    eng.profile(True)  # where the exact step's time goes (CUDA events per launch)
    run(sx["ctx"], sx["caches"])
    kst = eng.profile_read()
    eng.profile(False)
    split = {}
    for k in kst:
        key = "attention" if k["name"].startswith("attn_exact") else (
            "gemm" if k["name"].startswith("gemm_exact") else k["name"])
        split[key] = split.get(key, 0.0) + k["total_ms"]
    exact = {"ttft_ms": round(dev_ms / 2, 3), "tokens_per_s": round(n_tokens / (dev_ms / 2 / 1e3), 1),
             "ms_by_kind": {k: round(v, 3) for k, v in split.items()},
             "gpu_launches_per_step": int(launches // 2),
             "selected_per_segment": [int(x["selection_count"]) for x in rx["segments"]],
             "note": "RK_FP32_EXACT: SIMT kernels replaying the reference's fp32 operation order"}
    del cb, ctxb
    # fp32-accurate tensor-core mode (RK_FP32_TC: 3xTF32 tcgen05 GEMMs + fp32
    # flash attention) on the same relay caches: TTFT and error vs the exact run
    tc = None
    try:
        wt = eng.weights(spec_obj(), SEED, "fp32tc")
        ct = [wt.upload_cache(h) for h in hosts]
        ctxt = wt.context()
        rt = run(ctxt, ct, True)
        Kt, Vt = ctxt.all()
        tc_ms, _, tc_launches = timed(lambda: run(ctxt, ct), 3, 1)
        eng.profile(True)
        run(ctxt, ct)
        kst = eng.profile_read()
        eng.profile(False)
        tsplit = {}
        for k in kst:
            key = "attention" if k["name"].startswith("attn") else (
                "gemm" if k["name"].startswith("tc_split_gemm") else (
                    "inner_gemm" if k["name"].startswith("gemm") else k["name"]))
            tsplit[key] = tsplit.get(key, 0.0) + k["total_ms"]
        same_sel = all(np.array_equal(a["selection"], b["selection"]) for a, b in zip(rt["segments"], rx["segments"]))
        tc = {"ttft_ms": round(tc_ms / 3, 3), "tokens_per_s": round(n_tokens / (tc_ms / 3 / 1e3), 1),
              "ms_by_kind": {k: round(v, 3) for k, v in tsplit.items()},
              "gpu_launches_per_step": int(tc_launches // 3),
              "error_vs_exact": {"logits_rel_l2": _rel_l2(rt["logits"], rx["logits"]),
                                 "logits_max_abs": float(np.max(np.abs(rt["logits"].astype(np.float64) - rx["logits"]))),
                                 "kv_rel_l2": max(_rel_l2(Kt, Kx), _rel_l2(Vt, Vx)) if same_sel else None,
                                 "first_token_match": rt["first_token"] == rx["first_token"],
                                 "selection_equal": same_sel,
                                 "selected_per_segment": [int(x["selection_count"]) for x in rt["segments"]]},
              "note": "RK_FP32_TC: 3xTF32 tcgen05 GEMMs (hi/lo split, K chunked into <=1536-element TMEM "
                      "accumulations summed in fp32) + fp32 flash attention; exact-path storage and relay kernels"}
        del ct, ctxt, wt
    except Exception as ex:
        tc = {"error": f"{type(ex).__name__}: {str(ex)[:200]}"}
    exact["fp32_tc"] = tc
    del sx, wx
    return exact, err


def run_ours(args, world, rank, local, dist):
    import torch
    from paper_2603_13289_b200.engine import Engine
    from paper_2603_13289_b200.sessions import gather_records, shard
    torch.cuda.set_device(local)
    eng = Engine(local)
    w = eng.weights(spec_obj(), SEED, "bf16")
    n_sessions = args.sessions or WL.get("sessions", world)
    mine = [build_session(w, sid) for sid in shard(n_sessions, world, rank)]
    prof, opts = options()
    _, full_opts = options("full")
    stream = torch.cuda.ExternalStream(eng.stream)
    n_tokens = prompt_tokens()
    # first local session carries the single-session diagnostics
    caches, ctx = mine[0]["caches"], mine[0]["ctx"]

    def run_session(sess, o=opts, want_outputs=False):
        sess["ctx"].reset()
        return sess["ctx"].agent_prefill(sess["prefix"], sess["caches"], sess["suffix"], prof, o,
                                         want_logits=False, outputs=want_outputs)

    def step(o=opts):
        import torch
        torch.cuda.nvtx.range_push("relay_step")  # ncu --nvtx --nvtx-include relay_step/
        for sess in mine:
            run_session(sess, o)
        torch.cuda.nvtx.range_pop()

    def timed(fn, K, W):
        for _ in range(W):
            fn()
        barrier(dist)
        torch.cuda.synchronize()
        eng.synchronize()
        launches0 = eng.launches
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        h0 = time.perf_counter()
        for _ in range(K):
            fn()
        t1.record(stream)
        t1.synchronize()
        host_ms = (time.perf_counter() - h0) * 1e3
        torch.cuda.synchronize()
        barrier(dist)
        return t0.elapsed_time(t1), host_ms, eng.launches - launches0

    # correctness / reuse diagnostics of one session
    diag = run_session(mine[0], want_outputs=True)
    segs = diag["segments"]
    reuse = [s["stats"]["reuse_rate"] for s in segs]
    selected = [int(s["selection_count"]) for s in segs]

    with ClockSampler(local) as clk:
        dev_ms, host_ms, launches = timed(step, args.steps, args.warmup)
    dev_ms = reduce_max(dist, dev_ms, local)
    ms_step = dev_ms / args.steps
    if args.lean:
        if rank == 0:
            print(json.dumps({"lean": True, "ms_per_step": round(ms_step, 4), "gpu_launches": int(launches)}), flush=True)
        return
    value = n_sessions * n_tokens * args.steps / (dev_ms / 1e3)
    ttft = ms_step / len(mine)  # per session, sessions of a GPU run back to back

    full_ms, _, _ = timed(lambda: run_session(mine[0], full_opts), max(2, args.steps // 2), 1)
    full_ms = reduce_max(dist, full_ms, local) / max(2, args.steps // 2)

    # end to end through the C ABI with HOST buffers: RelayCache fp32 arrays
    # (the reference's struct, in pinned host memory) uploaded every step
    # (rk_cache_upload), tokens staged, logits read back.
    hosts = [pin_host(c.to_host()) for c in caches]

    # layers l_start..l_det-1 of every cache are never read by the relay (the
    # band recomputes them; l_det is read by the deviation score): they are
    # held back (rk_cache_upload_async_defer) and never cross PCIe
    l_start, l_det = WL["profile"][0], WL["profile"][1]
    defer = (l_start, l_det - 1) if l_det > l_start else None

    def e2e_step():
        # layer-streamed uploads: the relay prefill starts while later layers
        # of the caches are still crossing PCIe (rk_cache_upload_async)
        ups = [w.upload_cache(h, asynchronous=True, defer=defer) for h in hosts]
        ctx.reset()
        out = ctx.agent_prefill(mine[0]["prefix"], ups, mine[0]["suffix"], prof, opts, want_logits=True)
        return out["first_token"]

    e2e_K = max(2, args.steps // 2)
    for _ in range(max(1, args.warmup // 2)):
        e2e_step()
    barrier(dist)
    h0 = time.perf_counter()
    for _ in range(e2e_K):
        e2e_step()
    e2e_ms = reduce_max(dist, (time.perf_counter() - h0) * 1e3, local) / e2e_K  # one session per rank
    # the upload alone (diagnostic: how much of e2e is PCIe); median of
    # per-iteration times (an nvidia-smi sample of the clock sampler can stall
    # the driver's enqueue for tens of ms)
    ups_ms = []
    for _ in range(max(e2e_K, 5)):
        h0 = time.perf_counter()
        ups = [w.upload_cache(h, asynchronous=True, defer=defer) for h in hosts]
        for c in ups:
            c.xfer_wait()
        ups_ms.append((time.perf_counter() - h0) * 1e3)
        del ups
    upload_ms = statistics.median(ups_ms)
    # bytes that cross PCIe: fp32 K/V, unless RK_HOST_CONVERT=1 converts them
    # to bf16 on the host first (rk_cache_upload_async), then half of that
    kv_div = 2 if os.environ.get("RK_HOST_CONVERT", "0") != "0" else 1
    sent = 1.0 - ((defer[1] - defer[0] + 1) / WL["spec"]["num_layers"] if defer else 0.0)
    h2d = sum(int((h.k_pre.nbytes + h.v.nbytes) * sent) // kv_div + h.hidden_snapshot.nbytes + h.influence.nbytes +
              h.segment_tokens.nbytes for h in hosts) + 4 * (WL["prefix"] + WL["suffix"])
    d2h = 4 * WL["spec"]["vocab_size"] + 4

    # per-kernel instrumentation pass (same step, CUDA events per launch)
    eng.profile(True)
    run_session(mine[0])
    kstats = eng.profile_read()
    eng.profile(False)

    exact, bf16_err = None, None
    if args.exact_leg == "on" or (args.exact_leg == "auto" and args.config == "c2"):
        try:
            exact, bf16_err = exact_leg(eng, w, timed)
        except Exception as ex:
            exact = {"error": f"{type(ex).__name__}: {str(ex)[:200]}"}

    # results gather over NCCL (after timing; no collective on the hot path)
    recs = []
    for sess in mine:
        o = run_session(sess, want_outputs=True)
        recs.append({"session": sess["session"], "first_token": o["first_token"], "segments": len(o["segments"]),
                     "selected_total": sum(int(x["selection_count"]) for x in o["segments"]),
                     "reuse": sum(x["stats"]["reuse_rate"] for x in o["segments"]) / len(o["segments"]),
                     "ttft_ms": ttft})
    gathered = gather_records(recs, n_sessions, dist, device=f"cuda:{local}")

    hbm, tf_burst, tf_sus, src = peaks()
    traffic = {}  # ncu DRAM bytes per launch, from the committed capture of this workload
    try:
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as f:
            traffic = json.load(f)["kernels"] if args.config == "c2" else {}
    except Exception:
        traffic = {}
    detail = sorted(kstats, key=lambda k: -k["total_ms"])
    kstats = merge_kernel_stats(kstats)
    gemm = next((k for k in kstats if k["name"].startswith("gemm")), None)
    roofline = None
    clocks = clk.summary()
    # burst peak when the SMs ran at (near) their max clock during the timed
    # region, the sustained (power-capped) figure otherwise (B200_PROFILING.md)
    near_max = bool(clocks.get("sm_mhz") and clocks.get("sm_max_mhz") and
                    clocks["sm_mhz"] >= 0.95 * clocks["sm_max_mhz"])
    tf_peak, peak_kind = (tf_burst, "bf16_tflops (burst; SM clock near max)") if near_max else \
        (tf_sus, "bf16_tflops_sustained (SM clock below max)")
    if gemm and gemm["total_ms"] > 0:
        achieved = gemm["flops"] / (gemm["total_ms"] / 1e3) / 1e12
        roofline = {"kernel": "gemm_bf16_tcgen05", "bound": "tensor", "achieved": round(achieved, 1),
                    "peak": tf_peak, "peak_source": f"{src} {peak_kind}", "unit": "TFLOP/s",
                    "frac": round(achieved / tf_peak, 4),
                    "traffic": traffic.get("gemm_bf16_tcgen05", {}).get("traffic_bytes"),
                    "traffic_launch": traffic.get("gemm_bf16_tcgen05", {}).get("launch"),
                    "launches_per_step": gemm["launches"],
                    "gemm_ms_per_step": round(gemm["total_ms"], 4),
                    "gemm_tflop_per_step": round(gemm["flops"] / 1e12, 4)}
    kernels = {}
    for k in kstats:
        e = {"launches": k["launches"], "ms": round(k["total_ms"], 4)}
        if k["flops"]:
            e["tflops"] = round(k["flops"] / (k["total_ms"] / 1e3) / 1e12, 1) if k["total_ms"] else None
        if k["bytes"] and not k["name"].startswith(("gemm", "attention")):
            e["gbs"] = round(k["bytes"] / (k["total_ms"] / 1e3) / 1e9, 1) if k["total_ms"] else None
            e["hbm_frac"] = round(e["gbs"] / hbm, 4) if e.get("gbs") else None
            e["bytes_per_launch"] = round(k["bytes"] / max(1, k["launches"]))
        if k["name"] in traffic:
            e["ncu_traffic_bytes"] = traffic[k["name"]]["traffic_bytes"]
        kernels[k["name"]] = e

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            tps, meta = cpu_sample(hosts, steps=1, warmup=0, kind="reference", full_selected=selected)
            cpu = {"value": round(tps, 4), "unit": "tokens/s", **meta}
        except Exception as ex:  # the CPU leg is a reported baseline, not the product
            cpu = {"value": None, "unit": "tokens/s", "error": str(ex)[:200]}

    out = {
        "metric": "relay-prefill tokens/s (downstream-agent TTFT at ~80% KV reuse)",
        "value": round(value, 1), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"{WL['title']}, last agent's TTFT at a {n_tokens}-token prompt "
                               f"(prefix {WL['prefix']} + {WL['agents'] - 1} relayed segments x {WL['segment']} + "
                               f"suffix {WL['suffix']}), profile {WL['profile']}, thresholds (1.5, 1.45, 10)",
                   "config_id": args.config,
                   "sessions_per_gpu": len(mine), "l2": "inputs larger than L2 (bf16 weights streamed per step)",
                   "parallelism": f"sessions sharded, {world} GPU(s), no hot-path collective"},
        "ttft_ms": round(ttft, 4),
        "full_prefill_ttft_ms": round(full_ms, 4),
        "speedup_vs_full_prefill": round(full_ms / ttft, 3),
        "sessions": n_sessions, "sessions_gathered": len(gathered),
        "first_tokens": [r["first_token"] for r in gathered][:16],
        "reuse_rate_per_segment": [round(r, 4) for r in reuse],
        "selected_per_segment": selected,
        "host_ms_per_step": round(host_ms / args.steps, 4),
        "e2e": {"value": round(world * n_tokens / (e2e_ms / 1e3), 1), "unit": "tokens/s",
                "ttft_ms": round(e2e_ms, 3), "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "upload_only_ms": round(upload_ms, 3), "h2d_gbs": round(h2d / (upload_ms / 1e3) / 1e9, 1)},
        "gpu_launches": int(launches),
        "roofline": roofline,
        "kernels": kernels,
        "kernel_detail": [{"name": k["name"], "launches": k["launches"], "ms": round(k["total_ms"], 4),
                           "tflops": round(k["flops"] / (k["total_ms"] / 1e3) / 1e12, 1) if k["flops"] and k["total_ms"] else None}
                          for k in detail[:40]],
        "cpu_baseline": cpu,
        "fp32_exact": exact,
        "bf16_error": bf16_err,
        "clocks": clocks,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)


def run_reference(args, world, rank, local, dist):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref, built from /root/reference sources) on this box's host cores,
    same metric/unit: each step runs one independent session per host core on
    a bounded sample of the workload (the reference's own decode-time captures
    of the cut segments), extrapolated to the GPU arm's full prompt with the
    reference's FLOP model (cpu_sample; labelled "extrapolated")."""
    if rank != 0:
        return
    try:
        from oracle.oracle import available
        if not available("reference"):
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference "
                                                                  "at build time)"}))
            return
        ref = full_c2_reference_run() if args.config == "c2" else None
        full_sel = ref.get("selected_per_segment") if ref else None
        value, meta = cpu_sample(None, steps=args.steps, warmup=args.warmup, kind="reference",
                                 full_selected=full_sel)
        ms = meta["full_prompt_ttft_ms_all_cores_extrapolated"]
        print(json.dumps({
            "impl": "reference", "metric": "relay-prefill tokens/s (downstream-agent TTFT at ~80% KV reuse)",
            "value": round(value, 4), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "config": {"workload": f"{WL['title']}, last agent's TTFT at a {prompt_tokens()}-token prompt, "
                                   f"profile {WL['profile']} (CPU: measured sample, FLOP-model extrapolated)",
                       "config_id": args.config, "sample": meta["sample"]},
            "ttft_ms_one_core": meta["full_prompt_ttft_ms_one_core_extrapolated"],
            "cpu_baseline": {"value": round(value, 4), "unit": "tokens/s", **meta},
            "e2e": {"value": round(value, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }), flush=True)
    except Exception as ex:
        print(json.dumps({"impl": "reference", "unavailable": f"{type(ex).__name__}: {str(ex)[:200]}"}))


def run_stub(args, world, rank, local, dist):
    """The multi-rank plumbing of run_ours without a GPU (CPU tests, gloo):
    sessions sharded contiguously, a timed loop of no-op sessions bracketed by
    barriers, max-over-ranks time, one all_gather of the per-session records
    after timing, one JSON line on rank 0."""
    from paper_2603_13289_b200.sessions import gather_records, shard
    n_sessions = args.sessions or WL.get("sessions", world)
    mine = list(shard(n_sessions, world, rank))
    barrier(dist)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for sid in mine:
            sum(range(1000))
    ms = reduce_max(dist, (time.perf_counter() - t0) * 1e3, local)
    barrier(dist)
    recs = [{"session": sid, "first_token": 1000 + sid, "segments": WL["agents"] - 1, "ttft_ms": ms} for sid in mine]
    gathered = gather_records(recs, n_sessions, dist)
    if rank == 0:
        print(json.dumps({"impl": "stub", "n_gpus": world, "steps": args.steps, "sessions": n_sessions,
                          "sessions_per_rank": len(mine), "sessions_gathered": len(gathered),
                          "gathered_ids": [r["session"] for r in gathered],
                          "first_tokens_ok": all(r["first_token"] == 1000 + r["session"] for r in gathered)}),
              flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference", "stub"], default="ours",
                    help="stub: the launcher/shard/gather plumbing with a CPU no-op session (tests only)")
    ap.add_argument("--config", choices=sorted(WORKLOADS), default="c2",
                    help="workload (default c2: the config BASELINE.json's metric is quoted on)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--exact-leg", choices=["auto", "on", "off"], default="auto",
                    help="fp32-exact TTFT + bf16 error leg (auto: c2 only)")
    ap.add_argument("--lean", action="store_true",
                    help="timed relay steps only (for ncu launch lists): no full-prefill, e2e or profiling legs")
    ap.add_argument("--sessions", type=int, default=0,
                    help="collaboration sessions in total, sharded contiguously over the GPUs (default: one per GPU)")
    args = ap.parse_args()
    set_workload(args.config)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(sys.argv[1:], args.gpus))
    world, rank, local, dist = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank, local, dist)
    elif args.impl == "stub":
        run_stub(args, world, rank, local, dist)
    else:
        run_ours(args, world, rank, local, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
