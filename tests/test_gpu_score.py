"""K2 deviation scores at l_det (relay_engine.cpp:270-277, metrics cosine):
the bf16 warp-per-row kernel and the fp32 exact kernel against a float64
numpy restatement (value cosines, and key cosines after the double RoPE
realignment of the cached pre-RoPE keys, rounded like realign())."""
import ctypes as C

import numpy as np
import pytest

from paper_2603_13289_b200.engine import P, _check, lib

pytestmark = pytest.mark.gpu


def bf16_bits(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def from_bits(b):
    return (b.astype(np.uint32) << 16).view(np.float32)


def rope_table(npos, dh, theta=10000.0):
    inv = 1.0 / theta ** (np.arange(0, dh, 2, dtype=np.float64) / dh)
    ang = np.arange(npos, dtype=np.float64)[:, None] * inv[None, :]
    return np.stack([np.cos(ang), np.sin(ang)], -1)  # [pos][dh/2][2]


def reference(cv, rv, ck, rk, heads, dh, rope, base, bf16):
    n = cv.shape[0]
    cs = rope[base:base + n]
    rk = rk.reshape(n, heads, dh // 2, 2).astype(np.float64)
    c, s_ = cs[:, None, :, 0], cs[:, None, :, 1]
    r0 = (c * rk[..., 0] - s_ * rk[..., 1]).astype(np.float32)
    r1 = (s_ * rk[..., 0] + c * rk[..., 1]).astype(np.float32)
    rot = np.stack([r0, r1], -1).reshape(n, heads * dh)
    if bf16:
        rot = from_bits(bf16_bits(rot))
    out = []
    for a, b in ((cv, rv), (ck, rot)):
        a = a.reshape(n, heads, dh).astype(np.float64)
        b = b.reshape(n, heads, dh).astype(np.float64)
        same = np.all(a == b, axis=2)
        na, nb = np.linalg.norm(a, axis=2), np.linalg.norm(b, axis=2)
        cos = np.clip((a * b).sum(2) / (na * nb), -1, 1)
        cos = np.where(same, 1.0, cos)
        cos = np.where((na < 1e-12) | (nb < 1e-12), 0.0, cos)
        out.append(1.0 - cos.mean(1))
    return out


@pytest.mark.parametrize("elem", [2, 4], ids=["bf16", "fp32"])
@pytest.mark.parametrize("heads,dh", [(8, 64), (8, 128), (4, 128), (16, 64), (32, 64)])
def test_score_deviation(engine, elem, heads, dh):
    n, base = 1000, 37
    rng = np.random.default_rng(heads * dh + elem)
    kv = heads * dh
    cv = rng.standard_normal((n, kv)).astype(np.float32)
    ck = rng.standard_normal((n, kv)).astype(np.float32)
    rv = (cv + 0.3 * rng.standard_normal((n, kv))).astype(np.float32)
    rk = rng.standard_normal((n, kv)).astype(np.float32)
    rope = rope_table(base + n, dh)
    if elem == 2:
        bits = [bf16_bits(x) for x in (cv, rv, ck, rk)]
        cv, rv, ck, rk = (from_bits(b) for b in bits)
        rv[::7] = cv[::7]  # identical value rows score exactly 0
        bits[1] = bf16_bits(rv)
        host = bits
    else:
        rv[::7] = cv[::7]
        host = [cv, rv, ck, rk]
    sd, sk = np.zeros(n), np.zeros(n)
    D = C.POINTER(C.c_double)
    _check(lib().rk_debug_score_deviation(P(engine.ptr), *[h.ctypes.data_as(C.c_void_p) for h in host], elem, n,
                                          heads, dh, np.ascontiguousarray(rope).ctypes.data_as(D), base,
                                          sd.ctypes.data_as(D), sk.ctypes.data_as(D)))
    ref_d, ref_k = reference(cv, rv, ck, rk, heads, dh, rope, base, elem == 2)
    assert np.abs(sd - ref_d).max() < 1e-12 and np.abs(sk - ref_k).max() < 1e-12
    assert (sd[::7] == 0).all()
