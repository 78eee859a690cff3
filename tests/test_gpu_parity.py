"""GPU parity: the fp32-exact CUDA path through the C ABI against the oracle
on identical seeded inputs. Bar: BIT-EXACT for everything (contexts, marks,
selection + tags, s_dev/s_key_dev, hidden states, depths, logits, caches),
which is stronger than the north_star's 1e-4 fp32 tolerance."""
import glob
import json
import os

import numpy as np
import pytest

from paper_2603_13289_b200.abi import InvalidArgument, LayerProfile, RelayOptions, SchemaError
from tests.golden.cases import CASES
from tests.compare import assert_bit_equal, assert_outputs_equal
from tests.scenarios import c1_spec, parity_scenarios, pattern_tokens, spec_of, synthetic_tokens, triple

pytestmark = pytest.mark.gpu
SCEN = parity_scenarios()


def test_weights_init_bit_exact(engine, oracle):
    for spec in (spec_of(8, 32, 4), c1_spec()):
        w = engine.weights(spec, 1234)
        ow = oracle.weights(spec, 1234)
        for i in range(w.num_tensors()):
            want = oracle.weights_tensor(ow, i)
            assert_bit_equal(w.tensor(i, want.size), want, f"tensor {i}")


@pytest.mark.parametrize("scen", SCEN, ids=[s[0] for s in SCEN])
def test_relay_prefill_bit_exact(engine, oracle, scen):
    name, spec, seed, old, n, snap, new, prof, opts = scen
    ow = oracle.weights(spec, seed)
    cache = oracle.scenario(ow, old, n, snap)
    want, octx = oracle.relay_prefill(ow, new, cache, prof, opts)
    w = engine.weights(spec, seed)
    ctx = w.context()
    got = ctx.relay_prefill(new, w.upload_cache(cache), prof, opts)
    assert_outputs_equal(got, want, name)
    assert_bit_equal(got["logits"], want["logits"], f"{name}.logits")
    K, V = ctx.all()
    Ko, Vo = oracle.ctx_all(octx)
    assert_bit_equal(K, Ko, f"{name}.ctx.K")
    assert_bit_equal(V, Vo, f"{name}.ctx.V")
    segs, osegs = ctx.segments(), oracle.ctx_segments(octx)
    assert [(b, l) for b, l, _ in segs] == [(b, l) for b, l, _ in osegs]
    for (_, _, a), (_, _, b) in zip(segs, osegs):
        assert_bit_equal(a, b, f"{name}.marks")
    # marks agree with the accounting identity (relay_engine.cpp:347-358)
    assert int(segs[0][2].sum()) == got["stats"]["recomputed_entries"]


def test_c1_bit_exact_and_capture(engine, oracle):
    """BASELINE config 1 (2 layers, d=256, 4 heads, 512-token segment): GPU
    decode-time capture == oracle capture, and the relay prefill is bit-exact."""
    spec = c1_spec()
    ow = oracle.weights(spec, 1234)
    old = synthetic_tokens(1234, 1, 64, 256)
    cache = oracle.scenario(ow, old, 512, 0)
    w = engine.weights(spec, 1234)
    dctx = w.context()
    logits = dctx.prefill(old)
    gcache = dctx.capture_decode(logits, 512, 0).to_host()
    for f in ("segment_tokens", "k_pre", "v", "hidden_snapshot", "influence"):
        assert_bit_equal(getattr(gcache, f), getattr(cache, f), f"c1.capture.{f}")
    new = synthetic_tokens(1234, 2, 48, 256)
    want, octx = oracle.relay_prefill(ow, new, cache, triple(0, 0, 1), RelayOptions.make())
    ctx = w.context()
    got = ctx.relay_prefill(new, w.upload_cache(cache), triple(0, 0, 1), RelayOptions.make())
    assert_outputs_equal(got, want, "c1")
    assert_bit_equal(got["logits"], want["logits"], "c1.logits")
    K, V = ctx.all()
    Ko, Vo = oracle.ctx_all(octx)
    assert_bit_equal(K, Ko, "c1.K")
    assert_bit_equal(V, Vo, "c1.V")


@pytest.mark.parametrize("fused", [1, 0], ids=["fused", "sequential"])
@pytest.mark.parametrize("mode", ["relay", "full", "blend", "zero"])
def test_agent_prefill_bit_exact(engine, oracle, mode, fused):
    """The downstream agent's prompt (prefix + 2 relayed segments + suffix, or
    no suffix): the engine's layer-major fused schedule and its sequential
    schedule are both bit-identical to the oracle's sequential order."""
    engine.set_fused(fused)
    spec = spec_of(8, 32, 4)
    ow = oracle.weights(spec, 55)
    c1 = oracle.scenario(ow, pattern_tokens(9, 64, 1), 12, 1)
    c2 = oracle.scenario(ow, pattern_tokens(7, 64, 2), 9, 1)
    opts = RelayOptions.make(mode=mode, suffix_k=3, blend_alpha=0.25)
    prof = triple(1, 2, 5)
    if mode == "zero":
        c1 = oracle.scenario(ow, pattern_tokens(9, 64, 1), 12, 1)
    for suffix in (pattern_tokens(4, 64, 4), np.zeros(0, np.int32)):
        logits, tok, octx = oracle.agent_prefill(ow, pattern_tokens(5, 64, 3), [c1, c2], suffix, prof, opts)
        w = engine.weights(spec, 55)
        ctx = w.context()
        got = ctx.agent_prefill(pattern_tokens(5, 64, 3), [w.upload_cache(c1), w.upload_cache(c2)], suffix,
                                prof, opts)
        assert_bit_equal(got["logits"], logits, f"agent.{mode}.logits")
        assert got["first_token"] == tok
        K, V = ctx.all()
        Ko, Vo = oracle.ctx_all(octx)
        assert_bit_equal(K, Ko, f"agent.{mode}.K")
        assert_bit_equal(V, Vo, f"agent.{mode}.V")
        segs, osegs = ctx.segments(), oracle.ctx_segments(octx)
        assert len(segs) == len(osegs)
        for (b, l, a), (ob, ol, oa) in zip(segs, osegs):
            assert (b, l) == (ob, ol)
            assert_bit_equal(a, oa, f"agent.{mode}.marks")
    engine.set_fused(1)


def test_agent_prefill_many_segments_bit_exact(engine, oracle):
    """Ten relayed segments (a deep agent chain) through the fused schedule:
    bit-identical to the oracle's sequential order (the fused schedule takes
    up to 32 segments; relay and blend)."""
    spec = spec_of(8, 32, 4)
    ow = oracle.weights(spec, 56)
    caches = [oracle.scenario(ow, pattern_tokens(5 + i, 64, 10 + i), 6 + (i % 3), 1) for i in range(10)]
    prof = triple(1, 2, 5)
    for mode in ("relay", "blend"):
        opts = RelayOptions.make(mode=mode, suffix_k=2, blend_alpha=0.25)
        suffix = pattern_tokens(3, 64, 40)
        logits, tok, octx = oracle.agent_prefill(ow, pattern_tokens(4, 64, 41), caches, suffix, prof, opts)
        w = engine.weights(spec, 56)
        ctx = w.context()
        got = ctx.agent_prefill(pattern_tokens(4, 64, 41), [w.upload_cache(c) for c in caches], suffix, prof, opts)
        assert_bit_equal(got["logits"], logits, f"many.{mode}.logits")
        assert got["first_token"] == tok
        K, V = ctx.all()
        Ko, Vo = oracle.ctx_all(octx)
        assert_bit_equal(K, Ko, f"many.{mode}.K")
        assert_bit_equal(V, Vo, f"many.{mode}.V")
        assert len(ctx.segments()) == 10


def test_zero_mode_round_trip(engine, oracle):
    """ZERO with the unchanged prefix reproduces decode-time KV (test_engine.cpp:124-137)."""
    spec = spec_of(8, 32, 4)
    ow = oracle.weights(spec, 102)
    old = pattern_tokens(10, 64, 0)
    cache, dctx = oracle.scenario(ow, old, 8, 2, return_decode_ctx=True)
    w = engine.weights(spec, 102)
    ctx = w.context()
    got = ctx.relay_prefill(old, w.upload_cache(cache), LayerProfile(), RelayOptions.make(mode="zero"))
    K, V = ctx.all()
    Kd, Vd = oracle.ctx_all(dctx)
    assert_bit_equal(K, Kd, "zero.K")
    assert_bit_equal(V, Vd, "zero.V")
    assert got["stats"]["recomputed_entries"] == 0 and got["stats"]["reuse_rate"] == 1.0


def test_accounting_formula(engine, oracle):
    """(1,3,18) on 32 layers, N=100, |I|=10 -> 450 entries, reuse 0.859375 (test_engine.cpp:139-178)."""
    spec = spec_of(32, 16, 2)
    ow = oracle.weights(spec, 103)
    cache = oracle.scenario(ow, pattern_tokens(8, 64, 0), 100, 1)
    w = engine.weights(spec, 103)
    ctx = w.context()
    opts = RelayOptions.make(tau_dev=1e9, tau_inf=1e9, suffix_k=10)
    got = ctx.relay_prefill(pattern_tokens(12, 64, 3), w.upload_cache(cache), triple(1, 3, 18), opts)
    st = got["stats"]
    assert st["selected_count"] == 10 and st["total_entries"] == 3200
    assert st["recomputed_entries"] == 450 and st["reuse_rate"] == 0.859375
    marks = ctx.segments()[0][2]
    assert marks[1:4].all() and not marks[0].any() and not marks[19:].any()
    assert (marks[4:19, 90:] == 1).all() and not marks[4:19, :90].any()


def test_suffix_never_touches_segment_cells(engine, oracle):
    spec = spec_of(8, 32, 4)
    ow = oracle.weights(spec, 106)
    cache = oracle.scenario(ow, pattern_tokens(10, 64, 0), 8, 1)
    w = engine.weights(spec, 106)
    ctx = w.context()
    ctx.relay_prefill(pattern_tokens(6, 64, 4), w.upload_cache(cache), triple(1, 2, 5), RelayOptions.make())
    seg_end = ctx.size
    a, b = ctx.clone(), ctx.clone()
    a.prefill(pattern_tokens(5, 64, 11))
    b.prefill(pattern_tokens(5, 64, 12))
    Ka, _ = a.all()
    Kb, _ = b.all()
    assert_bit_equal(Ka[:, :seg_end], Kb[:, :seg_end], "suffix.K")


def test_validation_errors(engine, oracle):
    spec = spec_of(8, 32, 4)
    ow = oracle.weights(spec, 107)
    cache = oracle.scenario(ow, pattern_tokens(10, 64, 0), 8, 2)
    w = engine.weights(spec, 107)
    c = w.upload_cache(cache)
    prefix = pattern_tokens(4, 64, 1)
    with pytest.raises(SchemaError):
        w.context().relay_prefill(prefix, c, triple(1, 2, 20), RelayOptions.make())
    with pytest.raises(InvalidArgument):
        w.context().relay_prefill(prefix, c, triple(1, 2, 5), RelayOptions.make())
    with pytest.raises(InvalidArgument):
        w.context().relay_prefill(prefix, c, LayerProfile(), RelayOptions.make(mode="blend", blend_alpha=0.0))
    ctx = w.context()
    with pytest.raises(InvalidArgument):
        ctx.prefill(np.zeros(0, np.int32))
    with pytest.raises(InvalidArgument):
        ctx.prefill([64])  # outside vocab
    tiny = spec_of(8, 32, 4, max_positions=10)
    w2 = engine.weights(tiny, 107)
    ow2 = oracle.weights(tiny, 107)
    c2 = oracle.scenario(ow2, pattern_tokens(4, 64, 0), 4, 0)
    with pytest.raises(InvalidArgument):
        w2.context().relay_prefill(pattern_tokens(8, 64, 2), w2.upload_cache(c2), LayerProfile(),
                                   RelayOptions.make(mode="zero"))


@pytest.mark.parametrize("mode", ["relay", "zero", "blend"])
def test_async_upload_bit_exact(engine, oracle, mode):
    """rk_cache_upload_async (layers streamed on the copy stream, grafted layer
    by layer) gives the same bits as the synchronous upload."""
    spec = spec_of(6, 64, 4, kv_heads=2)
    ow = oracle.weights(spec, 31)
    c1 = oracle.scenario(ow, pattern_tokens(9, 64, 1), 16, 1)
    c2 = oracle.scenario(ow, pattern_tokens(7, 64, 2), 11, 1)
    prof = triple(1, 2, 4) if mode == "relay" else LayerProfile()
    opts = RelayOptions.make(mode=mode, suffix_k=3, blend_alpha=0.5)
    res = []
    for asynchronous in (False, True):
        w = engine.weights(spec, 31)
        ups = [w.upload_cache(c, asynchronous=asynchronous) for c in (c1, c2)]
        out = w.context().agent_prefill(pattern_tokens(5, 64, 3), ups, pattern_tokens(4, 64, 4), prof, opts)
        res.append(out["logits"])
    assert_bit_equal(res[1], res[0], f"async.{mode}.logits")


RKRC = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "*.rkrc")))


@pytest.mark.parametrize("path", RKRC, ids=os.path.basename)
@pytest.mark.parametrize("asynchronous", [False, True])
def test_rkrc_load_onto_device(engine, path, asynchronous):
    """load_relay_cache of a reference-written file straight onto the device
    (rk_cache_load; async = pinned blob streamed by layer) holds the file's bits."""
    from paper_2603_13289_b200.hostcache import HostRelayCache
    meta = json.load(open(path + ".json"))
    want = HostRelayCache.load(path)
    spec = CASES[meta["case"]]["spec"]()
    w = engine.weights(spec, meta["seed"])
    c = w.load_cache(path, asynchronous=asynchronous)
    got = c.to_host()
    for f in ("segment_tokens", "k_pre", "v", "hidden_snapshot", "influence"):
        assert_bit_equal(getattr(got, f), getattr(want, f), f"rkrc.{f}")
    assert (got.source_base_position, got.snapshot_layer) == (want.source_base_position, want.snapshot_layer)


@pytest.mark.parametrize("path", RKRC, ids=os.path.basename)
def test_rkrc_device_capture_saves_reference_bytes(engine, path, tmp_path):
    """Engine decode-time capture of the golden scenario, saved with
    rk_cache_save, is byte-identical to the file the reference saved."""
    meta = json.load(open(path + ".json"))
    spec = CASES[meta["case"]]["spec"]()
    w = engine.weights(spec, meta["seed"])
    dctx = w.context()
    logits = dctx.prefill(np.array(meta["old_prefix"], np.int32))
    cache = dctx.capture_decode(logits, meta["segment_len"], meta["snapshot_layer"])
    out = tmp_path / "engine.rkrc"
    cache.save(out)
    assert out.read_bytes() == open(path, "rb").read()


def test_rkrc_loaded_cache_relays_like_uploaded(engine, oracle):
    """A relay prefill through a loaded cache equals the reference's relay
    prefill through the same cache (bit-exact)."""
    path = [p for p in RKRC if "diag" in p][0]
    meta = json.load(open(path + ".json"))
    case = CASES[meta["case"]]
    spec = case["spec"]()
    from paper_2603_13289_b200.hostcache import HostRelayCache
    host = HostRelayCache.load(path)
    ow = oracle.weights(spec, meta["seed"])
    want, _ = oracle.relay_prefill(ow, case["prefix"], host, case["profile"], case["opts"])
    w = engine.weights(spec, meta["seed"])
    got = w.context().relay_prefill(case["prefix"], w.load_cache(path, asynchronous=True), case["profile"],
                                    case["opts"])
    assert_outputs_equal(got, want, "rkrc.relay")
    assert_bit_equal(got["logits"], want["logits"], "rkrc.relay.logits")


def test_token_deviation_bit_exact(engine, oracle):
    """token_deviation (metrics.cpp:118-159) on the device == the reference's,
    all four planes, bit for bit; identical caches give exact zeros."""
    from oracle.oracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref not built")
    ref = Oracle("reference")
    from paper_2603_13289_b200.profiler import token_deviation
    spec = spec_of(6, 64, 4, kv_heads=2)
    ow = oracle.weights(spec, 5)
    a = oracle.scenario(ow, pattern_tokens(9, 64, 1), 16, 1)
    b = oracle.scenario(ow, pattern_tokens(13, 64, 2), 16, 1)
    w = engine.weights(spec, 5)
    got = token_deviation(w.upload_cache(a), w.upload_cache(b))
    want = ref.token_deviation(a, b)
    for k in want:
        assert_bit_equal(got[k], want[k], f"token_deviation.{k}")
    zero = token_deviation(w.upload_cache(a), w.upload_cache(a))
    for k in zero:
        assert (zero[k] == 0.0).all(), k


@pytest.mark.parametrize("identical", [False, True])
def test_profile_model_bit_exact(engine, identical):
    """profile_model (profiler.cpp:157-175) with the captures, prefills and
    deviations on the device: same window, same fallbacks, bit-identical
    averaged curves as the reference run on the CPU."""
    from oracle.oracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref not built")
    ref = Oracle("reference")
    from paper_2603_13289_b200.profiler import ProfilerParams, TwoStageConfig, profile_model
    spec = spec_of(8, 32, 4)
    calib = TwoStageConfig.make(seed=3, instances=3, stage1_prefix=(8, 16), stage2_prefix=(6, 18), segment_len=12,
                                identical_prefix=identical, snapshot_layer=1)
    params = ProfilerParams.make(tau_start=0.95)
    got = profile_model(engine.weights(spec, 77), calib, params)
    want = ref.profile_model(ref.weights(spec, 77), calib, params)
    for k in ("l_start", "l_det", "l_end", "end_fallback", "det_fallback"):
        assert got[k] == want[k], (k, got, want)
    assert_bit_equal(got["curve_s"], want["curve_s"], "curve_s")
    assert_bit_equal(got["curve_rho"], want["curve_rho"], "curve_rho")


def test_profile_model_bf16_runs(engine):
    from paper_2603_13289_b200.profiler import TwoStageConfig, profile_model
    spec = spec_of(8, 256, 4)
    got = profile_model(engine.weights(spec, 9, "bf16"), TwoStageConfig.make(instances=2, segment_len=16))
    assert got["l_start"] <= got["l_det"] <= got["l_end"] < 8
    assert np.isfinite(got["curve_s"]).all()


@pytest.mark.parametrize("mode", ["relay", "zero", "blend"])
def test_deferred_layers_bit_exact(engine, oracle, mode):
    """rk_cache_upload_async_defer: the held-back layers are uploaded when a
    call first reads them (ZERO and BLEND read them, RELAY with the band over
    them does not) -- same bits as the plain upload, and export sees them."""
    spec = spec_of(6, 64, 4, kv_heads=2)
    ow = oracle.weights(spec, 31)
    c1 = oracle.scenario(ow, pattern_tokens(9, 64, 1), 16, 1)
    c2 = oracle.scenario(ow, pattern_tokens(7, 64, 2), 11, 1)
    prof = triple(1, 3, 4) if mode == "relay" else LayerProfile()
    opts = RelayOptions.make(mode=mode, suffix_k=3, blend_alpha=0.5)
    res = []
    for defer in (None, (1, 2)):
        w = engine.weights(spec, 31)
        ups = [w.upload_cache(c, asynchronous=True, defer=defer) for c in (c1, c2)]
        out = w.context().agent_prefill(pattern_tokens(5, 64, 3), ups, pattern_tokens(4, 64, 4), prof, opts)
        res.append(out["logits"])
        back = ups[0].to_host()
        assert_bit_equal(back.k_pre, c1.k_pre, f"defer.{mode}.export")
    assert_bit_equal(res[1], res[0], f"defer.{mode}.logits")
