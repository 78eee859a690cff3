"""Golden vectors from the reference itself (tests/golden/*.npz, made by
tests/golden/make_golden.py from oracle/_ref). The CPU restatement must
reproduce every one bit for bit (CPU test); the fp32-exact CUDA path too
(GPU test). The relay_accounting case also pins the reference's known answer
(test_engine.cpp:156-164): 450 recomputed entries, reuse 0.859375."""
import glob
import json
import os

import numpy as np
import pytest

from tests.compare import assert_bit_equal
from tests.golden.cases import CASES
from tests.golden.make_golden import digest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FILES = sorted(glob.glob(os.path.join(HERE, "*.npz")))


def load(path):
    z = np.load(path)
    meta = json.loads(bytes(z["meta"]).decode())
    return meta, {k: z[k] for k in z.files if k != "meta"}


def check_against(meta, arr, caches, out, what):
    assert [digest(c.segment_tokens, c.k_pre, c.v, c.hidden_snapshot, c.influence) for c in caches] == \
        meta["cache_digests"], f"{what}: decode-time capture differs from the reference"
    if "cache_k_pre" in arr:
        assert_bit_equal(caches[0].k_pre, arr["cache_k_pre"], f"{what}.cache.k_pre")
        assert_bit_equal(caches[0].influence, arr["cache_influence"], f"{what}.cache.influence")
    assert_bit_equal(out["logits"], arr["logits"], f"{what}.logits")
    assert out["ctx_digest"] == meta["ctx_digest"], f"{what}: KV context differs"
    if "selection" in arr:
        for k in ("selection", "tags", "s_dev", "s_key_dev", "depth", "origin"):
            assert_bit_equal(out[k].astype(arr[k].dtype), arr[k], f"{what}.{k}")
        assert out["hidden_digest"] == meta["hidden_digest"], f"{what}: segment hidden differs"
        for k, v in meta["stats"].items():
            assert out["stats"][k] == v, f"{what}.stats.{k}"
    else:
        assert out["first_token"] == meta["first_token"]
        for i, m in enumerate(out["marks"]):
            assert_bit_equal(m, arr[f"marks_{i}"], f"{what}.marks{i}")


def run_oracle(orc, case):
    from tests.golden.make_golden import run_case
    return run_case(orc, case)


@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(f)[:-4] for f in FILES])
def test_restatement_matches_golden(oracle, path):
    meta, arr = load(path)
    caches, out = run_oracle(oracle, CASES[meta["name"]])
    check_against(meta, arr, caches, out, meta["name"])


def test_known_answers_in_golden():
    meta, arr = load(os.path.join(HERE, "relay_accounting_L32.npz"))
    st = meta["stats"]
    assert st["total_entries"] == 3200 and st["recomputed_entries"] == 450 and st["reuse_rate"] == 0.859375
    assert list(arr["selection"]) == list(range(90, 100))


@pytest.mark.gpu
@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(f)[:-4] for f in FILES])
def test_gpu_exact_matches_golden(engine, oracle, path):
    """The CUDA fp32-exact path on the reference's golden inputs."""
    meta, arr = load(path)
    case = CASES[meta["name"]]
    spec = case["spec"]()
    ow = oracle.weights(spec, case["seed"])
    caches = [oracle.scenario(ow, old, n, snap) for (old, n, snap) in case["upstream"]]
    w = engine.weights(spec, case["seed"], "fp32")
    ctx = w.context()
    dev = [w.upload_cache(c) for c in caches]
    if case["kind"] == "relay_prefill":
        o = ctx.relay_prefill(case["prefix"], dev[0], case["profile"], case["opts"])
        K, V = ctx.all()
        o["ctx_digest"] = digest(K, V)
        o["hidden_digest"] = digest(o["hidden"])
        o["stats"] = {k: v for k, v in o["stats"].items() if k != "wall"}
    else:
        r = ctx.agent_prefill(case["prefix"], dev, case["suffix"], case["profile"], case["opts"])
        K, V = ctx.all()
        o = {"logits": r["logits"], "first_token": r["first_token"], "ctx_digest": digest(K, V),
             "marks": [s[2] for s in ctx.segments()]}
    check_against(meta, arr, caches, o, meta["name"] + "[gpu]")
