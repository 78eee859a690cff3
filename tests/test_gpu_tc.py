"""fp32-accurate tensor-core mode (RK_FP32_TC): 3xTF32 matmuls on tcgen05 +
fp32 flash attention over the fp32-exact path's storage and relay kernels.

north_star: "fp32-accumulate mode <= 1e-4 relative". The bar here: logits,
K/V context and hidden states within 1e-4 relative L2 of the bit-exact fp32
path (which equals the reference bitwise, tests/test_gpu_wide.py), and the
recompute selection equal to the reference's except for tokens whose
deviation score sits within 1e-3 (relative) of the selection threshold --
those are the only ones a ~1e-6 perturbation can flip, and they are counted
and reported, not hidden."""
import json
import os

import numpy as np
import pytest

from paper_2603_13289_b200.abi import LayerProfile, ModelSpec, RelayOptions
from tests.scenarios import pattern_tokens, triple

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TC_BOUND = 1e-4


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def threshold_flips(sel_got, sel_ref, s_dev_ref, tau, s_dev_got=None, noise=1e-6):
    """Tokens selected by one side only, and the largest relative distance of
    their (reference) deviation score from the mean-relative threshold. A flip
    whose deviations sit below the fp32 noise floor on both sides (a segment
    the upstream computed identically: the exact path's cosines are exactly 1,
    the tensor-core path's 1 - O(1e-12), and the mean-relative threshold scales
    that noise) counts at distance 0."""
    diff = np.setxor1d(np.asarray(sel_got, np.int64), np.asarray(sel_ref, np.int64))
    if len(diff) == 0:
        return 0, 0.0
    s_ref = np.asarray(s_dev_ref, np.float64)
    thr = tau * float(np.mean(s_ref))
    dist = []
    for j in diff:
        if s_dev_got is not None and abs(float(s_dev_got[j])) < noise and abs(float(s_ref[j])) < noise:
            dist.append(0.0)
        elif thr > 0:
            dist.append(abs(float(s_ref[j]) / thr - 1.0))
        else:
            dist.append(float("inf"))
    return len(diff), max(dist)


SPECS = [
    ("d256_h4_kv2_dh64", ModelSpec.make(4, 256, 4, 2, 64, 512, 256, 10000.0, 2048)),
    ("d512_h4_kv4_dh128", ModelSpec.make(3, 512, 4, 4, 128, 1024, 320, 500000.0, 2048)),
    ("d512_h8_kv2_dh64", ModelSpec.make(3, 512, 8, 2, 64, 1536, 384, 10000.0, 2048)),
]


@pytest.mark.parametrize("name,spec", SPECS, ids=[s[0] for s in SPECS])
@pytest.mark.parametrize("mode", ["relay", "full", "blend"])
def test_tc_relay_prefill_vs_exact(engine, oracle, name, spec, mode):
    ow = oracle.weights(spec, 99)
    cache = oracle.scenario(ow, pattern_tokens(40, spec.vocab_size, 1), 300, 1)
    prefix = pattern_tokens(57, spec.vocab_size, 2)
    # (l_det > l_start: the first recomputed layer reads the grafted snapshot,
    # so deviations are measured one layer later and are not identically 0)
    prof = triple(1, 2, 2) if mode == "relay" else LayerProfile()
    opts = RelayOptions.make(mode=mode, suffix_k=8, blend_alpha=0.25)
    res = {}
    for prec in ("fp32", "fp32tc"):
        w = engine.weights(spec, 99, prec)
        ctx = w.context()
        out = ctx.relay_prefill(prefix, w.upload_cache(cache), prof, opts)
        res[prec] = (out, ctx.all())
    (e, (Ke, Ve)), (t, (Kt, Vt)) = res["fp32"], res["fp32tc"]
    same = t["depth"] == e["depth"]
    # context rows of tokens selected by one mode only hold fresh vs reused K/V
    # by design; compare the rows both modes treated alike (segment = last 300)
    keep = np.ones(Ke.shape[1], bool)
    keep[Ke.shape[1] - 300 + np.setxor1d(t["selection"], e["selection"]).astype(np.int64)] = False
    errs = {"logits": rel(t["logits"], e["logits"]), "K": rel(Kt[:, keep], Ke[:, keep]),
            "V": rel(Vt[:, keep], Ve[:, keep]), "hidden": rel(t["hidden"][same], e["hidden"][same])}
    print(name, mode, errs, "sel", len(e["selection"]), len(t["selection"]))
    for k, v in errs.items():
        assert v < TC_BOUND, f"{k} rel err {v}"
    if mode == "relay":
        n, dist = threshold_flips(t["selection"], e["selection"], e["s_dev"], 1.5, t["s_dev"])
        assert n == 0 or dist < 1e-3, f"{n} selection flips, farthest {dist} from the threshold"
        assert float(np.max(np.abs(t["s_dev"] - e["s_dev"]))) < 1e-5
    else:
        assert np.array_equal(t["selection"], e["selection"])


def test_tc_agent_chain_matches_exact(engine, oracle):
    """Multi-upstream fused schedule (prefix -> relay_extend x2 -> suffix)."""
    spec = ModelSpec.make(4, 256, 4, 2, 64, 512, 256, 10000.0, 4096)
    ow = oracle.weights(spec, 5)
    caches = [oracle.scenario(ow, pattern_tokens(30 + 7 * i, spec.vocab_size, i), 200, 1) for i in range(2)]
    prefix = pattern_tokens(48, spec.vocab_size, 9)
    suffix = pattern_tokens(12, spec.vocab_size, 10)
    prof, opts = triple(1, 2, 3), RelayOptions.make(suffix_k=6)
    out = {}
    for prec in ("fp32", "fp32tc"):
        w = engine.weights(spec, 5, prec)
        ctx = w.context()
        r = ctx.agent_prefill(prefix, [w.upload_cache(c) for c in caches], suffix, prof, opts, want_logits=True,
                              outputs=True)
        out[prec] = (r, ctx.all())
    (e, (Ke, Ve)), (t, (Kt, Vt)) = out["fp32"], out["fp32tc"]
    assert rel(t["logits"], e["logits"]) < TC_BOUND
    if all(np.array_equal(a["selection"], b["selection"]) for a, b in zip(t["segments"], e["segments"])):
        assert max(rel(Kt, Ke), rel(Vt, Ve)) < TC_BOUND  # (else fresh vs reused rows differ by design)
    assert t["first_token"] == e["first_token"]


def test_tc_wide_error_report(engine):
    """c2-width golden chain (reference-written, tests/golden/wide): the TC
    mode's error against the reference's own logits and selection."""
    from tests.golden.cases import WIDE_CASES
    from tests.test_gpu_wide import FILES, jaccard, load, rel_l2, run_chain
    path = [f for f in FILES if "c2w" in os.path.basename(f)][0]
    meta, arr = load(path)
    case = WIDE_CASES[meta["name"]]
    spec = case["spec"]()
    wx = engine.weights(spec, case["seed"], "fp32")
    hosts = []
    for (old, n, snap) in case["upstream"]:
        ctx = wx.context()
        hosts.append(ctx.capture_decode(ctx.prefill(old), n, snap).to_host())
        del ctx
    rx, Kx, Vx = run_chain(wx, case, hosts)
    del wx
    wt = engine.weights(spec, case["seed"], "fp32tc")
    rt, Kt, Vt = run_chain(wt, case, hosts)
    rep = {"case": meta["case"], "mode": "fp32tc (3xTF32 tcgen05 GEMMs + fp32 flash attention)",
           "logits_rel_l2": rel_l2(rt["logits"], arr["logits"]),
           "logits_max_abs": float(np.max(np.abs(rt["logits"].astype(np.float64) - arr["logits"]))),
           "first_token_match": rt["first_token"] == meta["first_token"],
           "kv_rel_l2": max(rel_l2(Kt, Kx), rel_l2(Vt, Vx)), "segments": []}
    for i, (st, sx) in enumerate(zip(rt["segments"], rx["segments"])):
        ref_sel = arr[f"seg{i}_selection"]
        n, dist = threshold_flips(st["selection"], ref_sel, arr[f"seg{i}_s_dev"], case["opts"].tau_dev, st["s_dev"])
        same = st["depth"] == sx["depth"]
        rep["segments"].append({"selection_equal": bool(np.array_equal(st["selection"], ref_sel)),
                                "selection_jaccard": jaccard(st["selection"], ref_sel), "flips": n,
                                "flip_max_rel_dist_from_threshold": dist,
                                "hidden_rel_l2": rel_l2(st["hidden"][same], sx["hidden"][same]),
                                "s_dev_max_abs": float(np.max(np.abs(st["s_dev"] - arr[f"seg{i}_s_dev"])))})
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"fp32tc_error_{meta['name']}.json"), "w") as f:
        json.dump(rep, f, indent=1)
    print(json.dumps(rep))
    assert rep["logits_rel_l2"] < TC_BOUND, rep
    if all(x["flips"] == 0 for x in rep["segments"]):
        assert rep["kv_rel_l2"] < TC_BOUND, rep
    assert rep["first_token_match"], rep
    for s in rep["segments"]:
        assert s["hidden_rel_l2"] < TC_BOUND, rep
        assert s["flips"] == 0 or s["flip_max_rel_dist_from_threshold"] < 1e-3, rep


@pytest.mark.parametrize("shape", [(130, 256, 512), (320, 2048, 2048), (1000, 768, 8192)])
def test_tc_gemm_vs_fp64(engine, shape):
    """The 3xTF32 matmul alone against fp64, per element relative to the row's
    |A| . |B| scale (the accumulation error bound)."""
    import ctypes as C
    from paper_2603_13289_b200.engine import P, _check, lib
    M, N, K = shape
    rng = np.random.default_rng(M + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = (rng.standard_normal((K, N)) / np.sqrt(K)).astype(np.float32)
    out = np.zeros((M, N), np.float32)
    F = C.POINTER(C.c_float)
    _check(lib().rk_debug_gemm_tc(P(engine.ptr), A.ctypes.data_as(F), B.ctypes.data_as(F), out.ctypes.data_as(F),
                                  M, N, K, 0))
    ref = A.astype(np.float64) @ B.astype(np.float64)
    scale = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64)
    err = float(np.max(np.abs(out - ref) / scale))
    f32 = (A @ B).astype(np.float64)  # plain fp32 BLAS for comparison
    err_f32 = float(np.max(np.abs(f32 - ref) / scale))
    print(shape, "3xTF32 max err / (|A||B|):", err, "numpy fp32:", err_f32, "rel-L2", rel(out, ref))
    assert err < 2e-5 and rel(out, ref) < 1e-5
