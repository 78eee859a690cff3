"""Bitwise comparison helpers for parity tests."""
import numpy as np


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint8)


def assert_bit_equal(a, b, what):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, f"{what}: shape {a.shape} vs {b.shape}"
    if not np.array_equal(bits(a), bits(b)):
        if a.dtype.kind == "f":
            diff = np.abs(a.astype(np.float64) - b.astype(np.float64))
            idx = np.unravel_index(np.argmax(diff), diff.shape)
            n = int(np.sum(bits(a).reshape(a.size, -1) != bits(b).reshape(b.size, -1)) if a.size else 0)
            raise AssertionError(f"{what}: not bit-equal; max |diff| {diff.max():.3e} at {idx} "
                                 f"({a[idx]!r} vs {b[idx]!r})")
        raise AssertionError(f"{what}: not equal")


def assert_outputs_equal(got, want, what, check_hidden=True):
    for key in ("selection", "tags", "s_dev", "s_key_dev", "depth", "origin"):
        assert_bit_equal(got[key], want[key], f"{what}.{key}")
    if check_hidden:
        assert_bit_equal(got["hidden"], want["hidden"], f"{what}.hidden")
    gs, ws = got["stats"], want["stats"]
    for key in ("total_entries", "recomputed_entries", "reuse_rate", "selected_count", "selected_deviation",
                "selected_influence_score", "selected_influence_suffix", "selected_blend", "flops_cost",
                "flops_selection", "flops_realign", "flops_full_equiv"):
        assert gs[key] == ws[key], f"{what}.stats.{key}: {gs[key]} vs {ws[key]}"
