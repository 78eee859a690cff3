"""Pin the C restatement (oracle/relay_oracle.c) to the reference itself
(oracle/_ref, compiled from /root/reference/proj/src): bit-identical caches,
selections, marks, hidden states, contexts and logits on the reference's own
test scenarios (test_engine.cpp) and on BASELINE config 1."""
import numpy as np
import pytest

from paper_2603_13289_b200.abi import (InvalidArgument, LayerProfile, RelayOptions, SchemaError)
from tests.compare import assert_bit_equal, assert_outputs_equal
from tests.scenarios import c1_spec, parity_scenarios, pattern_tokens, spec_of, synthetic_tokens, triple

SCEN = parity_scenarios()


@pytest.mark.parametrize("scen", SCEN, ids=[s[0] for s in SCEN])
def test_restatement_equals_reference(oracle, reference, scen):
    name, spec, seed, old, n, snap, new, prof, opts = scen
    res = {}
    for tag, orc in (("restatement", oracle), ("reference", reference)):
        w = orc.weights(spec, seed)
        cache = orc.scenario(w, old, n, snap)
        out, ctx = orc.relay_prefill(w, new, cache, prof, opts)
        K, V = orc.ctx_all(ctx)
        res[tag] = (cache, out, K, V, orc.ctx_segments(ctx))
    (ca, oa, Ka, Va, sa), (cb, ob, Kb, Vb, sb) = res["restatement"], res["reference"]
    for f in ("k_pre", "v", "hidden_snapshot", "influence", "segment_tokens"):
        assert_bit_equal(getattr(ca, f), getattr(cb, f), f"{name}.cache.{f}")
    assert_outputs_equal(oa, ob, name)
    assert_bit_equal(oa["logits"], ob["logits"], f"{name}.logits")
    assert_bit_equal(Ka, Kb, f"{name}.ctx.K")
    assert_bit_equal(Va, Vb, f"{name}.ctx.V")
    assert len(sa) == len(sb) and all(x[0] == y[0] and x[1] == y[1] for x, y in zip(sa, sb))
    for x, y in zip(sa, sb):
        assert_bit_equal(x[2], y[2], f"{name}.marks")


def test_weights_init_mirror(oracle, reference):
    spec = spec_of(6, 32, 4)
    w1 = oracle.weights(spec, 77)
    w2 = reference.weights(spec, 77, checked=True)  # the reference's own init_weights
    for i in range(1 + 9 * 6 + 2):
        assert_bit_equal(oracle.weights_tensor(w1, i), reference.weights_tensor(w2, i), f"tensor {i}")


def test_c1_two_agent_relay(oracle, reference):
    """BASELINE config 1: 2 layers, d=256, 4 heads, 512-token decode segment."""
    spec = c1_spec()
    out = {}
    for tag, orc in (("restatement", oracle), ("reference", reference)):
        w = orc.weights(spec, 1234)
        cache = orc.scenario(w, synthetic_tokens(1234, 1, 64, 256), 512, 0)
        o, ctx = orc.relay_prefill(w, synthetic_tokens(1234, 2, 48, 256), cache, triple(0, 0, 1),
                                   RelayOptions.make())
        out[tag] = (cache, o, orc.ctx_all(ctx))
    (ca, oa, (Ka, Va)), (cb, ob, (Kb, Vb)) = out["restatement"], out["reference"]
    assert_bit_equal(ca.k_pre, cb.k_pre, "c1.cache.k_pre")
    assert_bit_equal(ca.influence, cb.influence, "c1.cache.influence")
    assert_outputs_equal(oa, ob, "c1")
    assert_bit_equal(oa["logits"], ob["logits"], "c1.logits")
    assert_bit_equal(Ka, Kb, "c1.K")
    assert_bit_equal(Va, Vb, "c1.V")


def test_agent_prefill_multi_segment(oracle, reference):
    """Two upstream segments + suffix (workflow.cpp:316-369)."""
    spec = spec_of(8, 32, 4)
    got = {}
    for tag, orc in (("restatement", oracle), ("reference", reference)):
        w = orc.weights(spec, 55)
        c1 = orc.scenario(w, pattern_tokens(9, 64, 1), 12, 1)
        c2 = orc.scenario(w, pattern_tokens(7, 64, 2), 9, 1)
        logits, tok, ctx = orc.agent_prefill(w, pattern_tokens(5, 64, 3), [c1, c2], pattern_tokens(4, 64, 4),
                                             triple(1, 2, 5), RelayOptions.make(suffix_k=3))
        got[tag] = (logits, tok, orc.ctx_all(ctx), orc.ctx_segments(ctx))
    a, b = got["restatement"], got["reference"]
    assert_bit_equal(a[0], b[0], "agent.logits")
    assert a[1] == b[1]
    assert_bit_equal(a[2][0], b[2][0], "agent.K")
    assert_bit_equal(a[2][1], b[2][1], "agent.V")


@pytest.mark.parametrize("which", ["restatement", "reference"])
def test_validation_error_types(oracle, reference, which):
    """relay validates profile, snapshot layer and capacity (test_engine.cpp:272-296)."""
    orc = oracle if which == "restatement" else reference
    spec = spec_of(8, 32, 4)
    w = orc.weights(spec, 107)
    cache = orc.scenario(w, pattern_tokens(10, 64, 0), 8, 2)
    prefix = pattern_tokens(4, 64, 1)
    with pytest.raises(SchemaError):
        orc.relay_prefill(w, prefix, cache, triple(1, 2, 20), RelayOptions.make())
    with pytest.raises(InvalidArgument):
        orc.relay_prefill(w, prefix, cache, triple(1, 2, 5), RelayOptions.make())
    with pytest.raises(InvalidArgument):
        orc.relay_prefill(w, prefix, cache, LayerProfile(), RelayOptions.make(mode="blend", blend_alpha=0.0))


def test_reference_unit_suite_passes():
    """The reference's own 88 non-CLI doctest cases pass against oracle/_ref."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                       "ref_unit_tests")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref not built")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "passed: 88 | failed: 0" in p.stdout
