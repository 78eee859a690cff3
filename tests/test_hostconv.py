"""The asynchronous upload's host-side fp32 -> bf16 conversion (hostconv.cpp):
round-to-nearest-even identical to the device's __float2bfloat16_rn (and to
numpy's reference rounding here), special values preserved, on 1 and 8
worker threads (chunked parallel_for covering every element exactly once)."""
import ctypes as C

import numpy as np
import pytest

from paper_2603_13289_b200.engine import _check, lib


def ref_bf16_bits(x):
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint32)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint32)
    return r.astype(np.uint16)


@pytest.mark.parametrize("threads", [1, 8])
@pytest.mark.parametrize("n", [0, 1, 4095, 1 << 20])
def test_f32_to_bf16_host(threads, n):
    rng = np.random.default_rng(n + threads)
    x = (rng.standard_normal(n) * np.exp(rng.uniform(-90, 90, n))).astype(np.float32)
    specials = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, -1e-45, 3.4028235e38, 1.0 + 2 ** -8,
                         1.0 + 3 * 2 ** -8, 1.0 + 2 ** -9], np.float32)
    if n >= len(specials):
        x[:len(specials)] = specials
    y = np.empty(n, np.uint16)
    _check(lib().rk_debug_f32_to_bf16_host(x.ctypes.data_as(C.POINTER(C.c_float)),
                                           y.ctypes.data_as(C.POINTER(C.c_uint16)), C.c_uint64(n), threads))
    assert np.array_equal(y, ref_bf16_bits(x))
