"""Offline layer profiler, host side (profiler.cpp:16-155, metrics.cpp:48-238):
make_layer_curve (similarity + adjacent-layer Spearman with average ranks),
average_curves and profile_from_curve (start / end / detection scans) against
the reference library (oracle/_ref) bit for bit, plus the scan fallbacks and
validation errors the reference's test_profiler.cpp exercises."""
import numpy as np
import pytest

from paper_2603_13289_b200.abi import InvalidArgument, SchemaError
from paper_2603_13289_b200.profiler import (ProfilerParams, average_curves, make_layer_curve,
                                            profile_from_curve)


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref not built")
    return Oracle("reference")


def same_curve(a, b):
    for k in ("s", "rho"):
        assert a[k].tobytes() == b[k].tobytes(), k
    assert np.array_equal(a["rho_degenerate"], b["rho_degenerate"])


def dev_matrix(seed, n, L, ties=False, const_layer=None):
    r = np.random.default_rng(seed)
    m = r.random((n, L)) * 0.3
    if ties:
        m = np.round(m * 8) / 8  # many equal values -> average ranks
    if const_layer is not None:
        m[:, const_layer] = 0.125  # constant column -> degenerate rho
    return m


CASES = [(0, 48, 32, False, None), (1, 20, 8, True, None), (2, 16, 12, False, 3), (3, 1, 6, False, None),
         (4, 2, 6, True, 0), (5, 100, 28, True, 27)]


@pytest.mark.parametrize("case", CASES, ids=[f"n{c[1]}-L{c[2]}" for c in CASES])
def test_layer_curve_bit_exact(ref, case):
    seed, n, L, ties, const = case
    m = dev_matrix(seed, n, L, ties, const)
    same_curve(make_layer_curve(m), ref.layer_curve(m))


def test_average_curves_bit_exact(ref):
    curves = [make_layer_curve(dev_matrix(s, 24, 10, s % 2 == 0, s if s < 10 else None)) for s in range(5)]
    same_curve(average_curves(curves), ref.average_curves(curves))


def synthetic_curve(L, kind):
    """Similarity curves of the shapes the scans meet: a dip then recovery
    (the paper's U-shape), a monotone decline (end-scan fallback), a flat
    tail (zero sigma)."""
    x = np.arange(L, dtype=np.float64)
    if kind == "u":
        s = 1.0 - 0.3 * np.exp(-((x - L * 0.4) ** 2) / (2 * (L / 8) ** 2))
    elif kind == "decline":
        s = 1.0 - 0.02 * x
    else:
        s = np.minimum(1.0, 0.7 + 0.05 * np.abs(x - 5))
        s[-6:] = s[-6]
    rho = np.concatenate([[np.nan], 0.5 + 0.4 * np.sin(x[1:] / 2.0)])
    deg = np.zeros(L, bool)
    deg[0] = True
    return {"s": s, "rho": rho, "rho_degenerate": deg}


@pytest.mark.parametrize("L", [8, 16, 32])
@pytest.mark.parametrize("kind", ["u", "decline", "flat_tail"])
@pytest.mark.parametrize("relaxed", [False, True])
def test_profile_from_curve_matches_reference(ref, L, kind, relaxed):
    c = synthetic_curve(L, kind)
    p = ProfilerParams.make(first_negative_alpha=relaxed)
    got = profile_from_curve(c, p)
    want = ref.profile_from_curve(c, p)
    for k in ("l_start", "l_det", "l_end", "end_fallback", "det_fallback"):
        assert got[k] == want[k], (k, got, want)
    assert got["curve_rho"].tobytes() == want["curve_rho"].tobytes()


def test_profile_from_averaged_random_curves(ref):
    for seed in range(6):
        curves = [make_layer_curve(dev_matrix(seed * 10 + i, 32, 16, i % 2 == 1)) for i in range(4)]
        avg = average_curves(curves)
        p = ProfilerParams.make(tau_start=0.8)
        got, want = profile_from_curve(avg, p), ref.profile_from_curve(avg, p)
        assert (got["l_start"], got["l_det"], got["l_end"]) == (want["l_start"], want["l_det"], want["l_end"])


def test_validation_errors(ref):
    c = synthetic_curve(16, "u")
    for bad in (ProfilerParams.make(tau_start=0.0), ProfilerParams.make(tail_layers=1),
                ProfilerParams.make(stability_lambda=0.0), ProfilerParams.make(consecutive=0),
                ProfilerParams.make(min_rise=0)):
        with pytest.raises(InvalidArgument):
            profile_from_curve(c, bad)
        with pytest.raises(InvalidArgument):
            ref.profile_from_curve(c, bad)
    short = synthetic_curve(5, "u")  # fewer than 6 layers
    with pytest.raises(InvalidArgument):
        profile_from_curve(short)
    with pytest.raises(InvalidArgument):
        make_layer_curve(np.zeros((0, 8)))
    assert issubclass(SchemaError, Exception)
