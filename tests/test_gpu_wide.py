"""Parity at the MEASURED model widths: BASELINE config 2 (Llama-3.2-1B shape,
the bench's default workload) and config 3 (Llama-3-8B shape), against
golden vectors the REFERENCE wrote (tests/golden/wide/*.npz, made by
tests/golden/make_golden_wide.py from oracle/_ref).

1. fp32-exact mode: the device's decode-time capture hits the reference's
   cache digests, and the relay chain (prefix prefill -> relay_extend per
   upstream -> suffix prefill, workflow.cpp:316-369, fused layer-major
   schedule) is BIT-EQUAL to the reference: selection + tags, s_dev,
   s_key_dev, depth, marks, stats, segment hidden states, merged KV context,
   end logits, first token. This is the north_star's "bit-exact
   recompute-token selection versus the CPU reference" at c2/c3 width.
2. bf16 throughput mode on the SAME (reference-identical) relay caches:
   its own error is measured and bounded -- logits max-abs / rel-L2 against
   the reference's logits, first-token agreement, per-segment selection
   Jaccard and |I| difference against the reference's selection, K/V and
   hidden rel-L2 against the exact run (which equals the reference bitwise).
   The numbers are written to gpurun_out/bf16_error_<case>.json.
"""
import glob
import json
import os

import numpy as np
import pytest

from tests.compare import assert_bit_equal
from tests.golden.cases import WIDE_CASES
from tests.golden.make_golden_wide import cache_digest, digest

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "wide")
FILES = sorted(glob.glob(os.path.join(HERE, "*.npz")))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# bf16-mode bounds (north_star: "a bf16 throughput mode reports its own max
# error"); measured values are reported, these are the asserted ceilings.
BF16_BOUNDS = {"logits_rel_l2": 3e-2, "kv_rel_l2": 2e-2, "hidden_rel_l2": 3e-2, "selection_jaccard_min": 0.6}


def load(path):
    z = np.load(path)
    meta = json.loads(bytes(z["meta"]).decode())
    return meta, {k: z[k] for k in z.files if k != "meta"}


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def jaccard(a, b):
    a, b = set(int(x) for x in a), set(int(x) for x in b)
    return 1.0 if not a and not b else len(a & b) / len(a | b)


@pytest.fixture(scope="module", params=FILES, ids=[os.path.basename(f)[:-4] for f in FILES])
def wide(request, engine):
    """Exact weights + the device's decode-time captures for one wide case."""
    meta, arr = load(request.param)
    case = WIDE_CASES[meta["name"]]
    spec = case["spec"]()
    w = engine.weights(spec, case["seed"], "fp32")
    hosts = []
    for (old, n, snap) in case["upstream"]:
        ctx = w.context()
        logits = ctx.prefill(old)
        hosts.append(ctx.capture_decode(logits, n, snap).to_host())
        del ctx
    yield meta, arr, case, w, hosts
    del w


def run_chain(w, case, hosts):
    ctx = w.context()
    caches = [w.upload_cache(h) for h in hosts]
    r = ctx.agent_prefill(case["prefix"], caches, case["suffix"], case["profile"], case["opts"],
                          want_logits=True, outputs=True)
    K, V = ctx.all()
    return r, K, V


def test_wide_capture_matches_reference(wide):
    meta, arr, case, w, hosts = wide
    assert [cache_digest(h) for h in hosts] == meta["cache_digests"], \
        "fp32-exact decode-time capture differs from the reference's RelayRecorder"


def test_wide_exact_bit_equal(wide):
    meta, arr, case, w, hosts = wide
    r, K, V = run_chain(w, case, hosts)
    name = meta["name"]
    for i, (seg, want) in enumerate(zip(r["segments"], meta["segments"])):
        for k in ("selection", "tags", "s_dev", "s_key_dev", "depth", "origin"):
            got = seg[k].astype(arr[f"seg{i}_{k}"].dtype)
            assert_bit_equal(got, arr[f"seg{i}_{k}"], f"{name}.seg{i}.{k}")
        assert digest(seg["hidden"]) == want["hidden_digest"], f"{name}.seg{i}: segment hidden differs"
        for k, v in want["stats"].items():
            assert seg["stats"][k] == v, f"{name}.seg{i}.stats.{k}: {seg['stats'][k]} vs {v}"
    assert_bit_equal(r["logits"], arr["logits"], f"{name}.logits")
    assert r["first_token"] == meta["first_token"]
    assert K.shape[1] == meta["ctx_size"]
    assert digest(K, V) == meta["ctx_digest"], f"{name}: merged KV context differs"


def test_wide_bf16_error_report(wide, engine):
    meta, arr, case, w, hosts = wide
    name = meta["name"]
    rx, Kx, Vx = run_chain(w, case, hosts)  # == reference bitwise (test above)
    wb = engine.weights(case["spec"](), case["seed"], "bf16")
    rb, Kb, Vb = run_chain(wb, case, hosts)
    ref_logits = arr["logits"]
    rep = {
        "case": meta["case"], "compared_against": "reference goldens (oracle/_ref) and the fp32-exact run "
                                                  "(bit-equal to the reference)",
        "logits_max_abs": float(np.max(np.abs(rb["logits"].astype(np.float64) - ref_logits))),
        "logits_ref_max_abs": float(np.max(np.abs(ref_logits))),
        "logits_rel_l2": rel_l2(rb["logits"], ref_logits),
        "first_token_bf16": rb["first_token"], "first_token_ref": meta["first_token"],
        "first_token_match": rb["first_token"] == meta["first_token"],
        "kv_rel_l2": max(rel_l2(Kb, Kx), rel_l2(Vb, Vx)),
        "k_max_abs": float(np.max(np.abs(Kb.astype(np.float64) - Kx))),
        "v_max_abs": float(np.max(np.abs(Vb.astype(np.float64) - Vx))),
        "segments": [],
    }
    hid = []
    for i, (sb, sx) in enumerate(zip(rb["segments"], rx["segments"])):
        ref_sel = arr[f"seg{i}_selection"]
        same = sb["depth"] == sx["depth"]  # rows whose selection differs stop at different layers
        hid.append(rel_l2(sb["hidden"][same], sx["hidden"][same]))
        rep["segments"].append({
            "selected_bf16": int(sb["selection_count"]), "selected_ref": int(len(ref_sel)),
            "selection_jaccard": jaccard(sb["selection"], ref_sel),
            "selection_equal": bool(np.array_equal(sb["selection"], ref_sel)),
            "s_dev_max_abs": float(np.max(np.abs(sb["s_dev"] - arr[f"seg{i}_s_dev"]))),
            "hidden_rel_l2": hid[-1],
            "reuse_bf16": sb["stats"]["reuse_rate"], "reuse_ref": meta["segments"][i]["stats"]["reuse_rate"],
        })
    rep["hidden_rel_l2"] = max(hid)
    rep["selection_jaccard_min"] = min(s["selection_jaccard"] for s in rep["segments"])
    rep["bounds"] = BF16_BOUNDS
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"bf16_error_{name}.json"), "w") as f:
        json.dump(rep, f, indent=1)
    print(json.dumps(rep))
    assert rep["logits_rel_l2"] < BF16_BOUNDS["logits_rel_l2"], rep
    assert rep["kv_rel_l2"] < BF16_BOUNDS["kv_rel_l2"], rep
    assert rep["hidden_rel_l2"] < BF16_BOUNDS["hidden_rel_l2"], rep
    assert rep["selection_jaccard_min"] >= BF16_BOUNDS["selection_jaccard_min"], rep
