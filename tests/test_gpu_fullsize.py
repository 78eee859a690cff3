"""Full-size (BASELINE configs 2 and 3) checks through size-independent properties, in
the bf16 throughput mode the bench measures: the oracle cannot run a 1B-model,
4,032-token relay in test time, so these pin what must hold at any size.

  - determinism: repeated relays give bit-identical logits, first token,
    selections, marks and contexts;
  - reused cells are the cache: every grafted V cell of every relayed segment
    is a bit copy of the cache's V (relay_engine.cpp:136-148), and every
    grafted K cell equals realign() of the cache's K_pre at its absolute
    position (checked against the realign restatement in numpy on the same
    bf16 values);
  - marks, selection and depths agree with each other and with the reuse
    accounting identity recomputed = N*(l_det-l_start+1) + |I|*(l_end-l_det)
    (test_engine.cpp:156);
  - the selection is sorted, unique, tagged, and contains the suffix window
    (selector.cpp:62-88), and every deviation-selected token clears the
    threshold tau_dev * mean(s_dev) (selector.cpp:32-50).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["c2", "c3"])
def full(engine, request):
    """BASELINE config 2 (the bench line) and config 3 (Llama-3-8B shape,
    8-agent chain, 16,000-token prompt)."""
    import bench
    bench.set_workload(request.param)
    w = engine.weights(bench.spec_obj(), bench.SEED, "bf16")
    sess = bench.build_session(w, 0)
    prof, opts = bench.options()
    yield bench, w, sess, prof, opts
    del sess, w
    bench.set_workload("c2")


def run(sess, prof, opts):
    sess["ctx"].reset()
    out = sess["ctx"].agent_prefill(sess["prefix"], sess["caches"], sess["suffix"], prof, opts, want_logits=True,
                                    outputs=True)
    return out


def test_fullsize_deterministic(full):
    bench, w, sess, prof, opts = full
    a = run(sess, prof, opts)
    Ka, Va = sess["ctx"].all()
    b = run(sess, prof, opts)
    Kb, Vb = sess["ctx"].all()
    assert a["first_token"] == b["first_token"]
    assert np.array_equal(a["logits"].view(np.uint32), b["logits"].view(np.uint32))
    for sa, sb in zip(a["segments"], b["segments"]):
        assert np.array_equal(sa["selection"], sb["selection"])
        assert np.array_equal(sa["origin"], sb["origin"])
        assert np.array_equal(sa["s_dev"].view(np.uint64), sb["s_dev"].view(np.uint64))
    assert np.array_equal(Ka.view(np.uint32), Kb.view(np.uint32))
    assert np.array_equal(Va.view(np.uint32), Vb.view(np.uint32))


def rope_table(theta, dh, positions):
    """cos/sin in double of the reference's rope_rotate (tensor.cpp:128-143)."""
    i = np.arange(dh // 2, dtype=np.float64)
    freq = np.power(np.float64(theta), -2.0 * i / dh)
    ang = positions[:, None].astype(np.float64) * freq[None, :]
    return np.cos(ang), np.sin(ang)


def bf16(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return (((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16).astype(np.uint32).view(np.float32)


def test_fullsize_reused_cells_are_the_cache(full):
    bench, w, sess, prof, opts = full
    out = run(sess, prof, opts)
    K, V = sess["ctx"].all()
    spec = w.spec
    dh, hkv = spec.d_head, spec.num_kv_heads
    l_start, l_det, l_end = prof.l_start, prof.l_det, prof.l_end
    for seg, cache in zip(out["segments"], sess["caches"]):
        host = cache.to_host()
        base, n = seg["segment_base"], seg["segment_len"]
        origin = seg["origin"]  # [L, n], 1 = recomputed
        reused = origin == 0
        for l in range(spec.num_layers):
            cells = np.nonzero(reused[l])[0]
            if cells.size == 0:
                continue
            assert np.array_equal(V[l, base + cells].view(np.uint32), host.v[l, cells].view(np.uint32)), l
            # realign: rotate K_pre (bf16 values) at absolute positions, double math, round to bf16
            kp = host.k_pre[l, cells].reshape(cells.size, hkv, dh // 2, 2).astype(np.float64)
            c, s = rope_table(spec.theta_base, dh, base + cells)
            c, s = c[:, None, :], s[:, None, :]
            r0 = (c * kp[..., 0] - s * kp[..., 1]).astype(np.float32)
            r1 = (s * kp[..., 0] + c * kp[..., 1]).astype(np.float32)
            want = bf16(np.stack([r0, r1], -1).reshape(cells.size, -1))
            got = K[l, base + cells]
            # the device builds its cos/sin table with glibc; numpy's libm may
            # differ in the last ulp of a few angles -> allow 1 bf16 ulp there
            diff = np.abs(got.view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64))
            assert (diff <= 1).all() and (diff == 0).mean() > 0.999, l
        # band layers [l_start, l_det] are recomputed for every token
        assert (origin[l_start:l_det + 1] == 1).all()
        assert (origin[:l_start] == 0).all() and (origin[l_end + 1:] == 0).all()


def test_fullsize_marks_selection_accounting(full):
    bench, w, sess, prof, opts = full
    out = run(sess, prof, opts)
    l_start, l_det, l_end = prof.l_start, prof.l_det, prof.l_end
    for seg in out["segments"]:
        n, sel, tags = seg["segment_len"], seg["selection"], seg["tags"]
        assert np.all(np.diff(sel) > 0) and (sel < n).all()
        assert (tags != 0).all()
        origin = seg["origin"]
        mask = np.zeros(n, bool)
        mask[sel] = True
        for l in range(l_det + 1, l_end + 1):
            assert np.array_equal(origin[l] == 1, mask), l
        assert np.array_equal(seg["depth"], np.where(mask, l_end + 1, l_det + 1))
        st = seg["stats"]
        assert st["recomputed_entries"] == n * (l_det - l_start + 1) + len(sel) * (l_end - l_det)
        assert st["recomputed_entries"] == int(origin.sum())
        assert abs(st["reuse_rate"] - (1 - st["recomputed_entries"] / (n * w.spec.num_layers))) < 1e-12
        # suffix window and deviation threshold
        assert set(range(n - min(opts.suffix_k, n), n)) <= set(sel.tolist())
        thr = seg["dev_threshold"]
        dev = sel[(tags & 1) != 0]
        assert (seg["s_dev"][dev] >= thr).all()
        assert (seg["s_dev"][np.setdiff1d(np.arange(n), dev)] < thr).all()


def test_fullsize_streamed_upload_matches_resident(full):
    """The e2e path at full size: host caches streamed in by layer (with the
    band layers deferred) while the relay runs -- every kernel launched with
    programmatic dependent launch behind a per-layer event wait -- gives the
    same bits as caches already resident on the device."""
    bench, w, sess, prof, opts = full
    ref = run(sess, prof, opts)
    hosts = [bench.pin_host(c.to_host()) for c in sess["caches"]]
    defer = (prof.l_start, prof.l_det - 1) if prof.l_det > prof.l_start else None
    for _ in range(2):
        ups = [w.upload_cache(h, asynchronous=True, defer=defer) for h in hosts]
        sess["ctx"].reset()
        got = sess["ctx"].agent_prefill(sess["prefix"], ups, sess["suffix"], prof, opts, want_logits=True)
        assert got["first_token"] == ref["first_token"]
        assert np.array_equal(got["logits"].view(np.uint32), ref["logits"].view(np.uint32))
