"""Kernel-level checks of the bf16 tensor-core kernels (tcgen05 GEMM, flash
attention) against fp64 numpy on bf16-rounded operands, and of the device
glibc-expf restatement against the host libm."""
import ctypes as C

import numpy as np
import pytest

from paper_2603_13289_b200.engine import P, _check, lib

pytestmark = pytest.mark.gpu
F32P = C.POINTER(C.c_float)


def bf16_round(x):
    x = np.ascontiguousarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def run_gemm(engine, A, B, C0, live, epi):
    M, K = A.shape
    N = B.shape[0]
    out = np.ascontiguousarray(C0, np.float32).copy()
    _check(lib().rk_debug_gemm_bf16(P(engine.ptr), np.ascontiguousarray(A, np.float32).ctypes.data_as(F32P),
                                    np.ascontiguousarray(B, np.float32).ctypes.data_as(F32P),
                                    out.ctypes.data_as(F32P), M, live, N, K, epi))
    return out


SHAPES = [(1, 64, 64), (7, 192, 128), (128, 256, 256), (200, 384, 512), (333, 1024, 2048),
          (1000, 128, 1024), (64, 3072, 2048), (256, 2048, 8192), (513, 16384, 256), (129, 64, 64),
          (4032, 3072, 2048), (320, 16384, 2048), (1, 16384, 2048), (1, 4096, 14336), (1, 128256, 2048)]


@pytest.mark.parametrize("shape", SHAPES, ids=[f"{m}x{n}x{k}" for m, n, k in SHAPES])
def test_gemm_store(engine, shape):
    M, N, K = shape
    rng = np.random.default_rng(M * 7 + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    got = run_gemm(engine, A, B, np.zeros((M, N)), M, 3)
    ref = bf16_round(A).astype(np.float64) @ bf16_round(B).astype(np.float64).T
    err = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30)
    assert err < 2e-5, f"rel err {err}"


@pytest.mark.parametrize("shape", [(128, 256, 8192), (256, 2048, 8192), (40, 512, 4096)])
def test_gemm_residual_split_k_deterministic(engine, shape):
    M, N, K = shape
    rng = np.random.default_rng(3)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    H = rng.standard_normal((M, N)).astype(np.float32)
    got = run_gemm(engine, A, B, H, M, 1)
    again = run_gemm(engine, A, B, H, M, 1)
    assert np.array_equal(got.view(np.uint32), again.view(np.uint32)), "split-K residual not deterministic"
    ref = H + bf16_round(A).astype(np.float64) @ bf16_round(B).astype(np.float64).T
    assert np.abs(got - ref).max() / np.abs(ref).max() < 2e-5


def test_gemm_live_rows(engine):
    M, N, K, live = 300, 256, 512, 77
    rng = np.random.default_rng(5)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32) / 20
    C0 = np.full((M, N), 7.0, np.float32)
    got = run_gemm(engine, A, B, C0, live, 3)
    ref = bf16_round(A[:live]).astype(np.float64) @ bf16_round(B).astype(np.float64).T
    assert np.abs(got[:live] - ref).max() / np.abs(ref).max() < 2e-5
    assert (got[live:] == 7.0).all(), "rows beyond the live count were written"


def ref_attention(q, k, v, pos, H, Hkv, dh):
    M, T = q.shape[0], k.shape[0]
    out = np.zeros((M, H * dh))
    g = H // Hkv
    qd, kd, vd = (bf16_round(x).astype(np.float64) for x in (q, k, v))
    for h in range(H):
        kh = h // g
        s = qd[:, h * dh:(h + 1) * dh] @ kd[:, kh * dh:(kh + 1) * dh].T / np.sqrt(dh)
        mask = np.arange(T)[None, :] > pos[:, None]
        s[mask] = -np.inf
        s -= s.max(1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(1, keepdims=True)
        out[:, h * dh:(h + 1) * dh] = p @ vd[:, kh * dh:(kh + 1) * dh]
    return out


ATT = [(64, 200, 4, 2, 64, "band"), (300, 700, 8, 2, 64, "sparse"), (130, 1000, 4, 4, 128, "band"),
       (1, 333, 4, 1, 128, "band"), (257, 1500, 32, 8, 64, "sparse"), (320, 4032, 32, 8, 64, "mixed"),
       (700, 2000, 16, 4, 128, "mixed"), (1356, 4032, 32, 8, 64, "mixed"), (900, 3000, 8, 2, 64, "live"),
       (600, 2500, 8, 4, 128, "live"), (4032, 4032, 32, 8, 64, "band"), (2048, 4096, 8, 2, 128, "band"),
       # GQA packing shapes: group 7 (Qwen2.5-7B: 28/4, 16 rows x 7 heads, 16 idle lanes), 16 (8 rows), 3, 8
       (500, 1800, 28, 4, 128, "live"), (333, 1200, 28, 4, 128, "mixed"), (260, 900, 32, 2, 64, "mixed"),
       (190, 640, 12, 4, 64, "sparse"), (450, 1500, 16, 2, 128, "live"),
       # few static rows (1-4; the top layer's last row, decode-capture steps)
       (1, 4032, 32, 8, 64, "band"), (4, 3000, 32, 8, 64, "sparse"), (2, 1000, 28, 4, 128, "band"),
       (3, 500, 8, 8, 64, "sparse"), (1, 1, 4, 2, 64, "band"), (1, 129, 16, 16, 128, "band"),
       (4, 129, 16, 2, 128, "sparse")]


@pytest.mark.parametrize("case", ATT, ids=[f"{c[5]}-M{c[0]}-T{c[1]}-dh{c[4]}" for c in ATT])
def test_attention(engine, case):
    M, T, H, Hkv, dh, kind = case
    rng = np.random.default_rng(M + T)
    live, g1, g2 = M, 0, 0
    if kind == "band":
        pos = np.arange(T - M, T, dtype=np.int32)
    elif kind in ("mixed", "live"):  # fused-schedule layout: [prefix | suffix | segment rows], unsorted
        n_pre, n_suf = M // 4, M // 8
        seg = np.sort(rng.choice(np.arange(n_pre, T - n_suf), M - n_pre - n_suf, replace=False))
        pos = np.concatenate([np.arange(n_pre), np.arange(T - n_suf, T), seg]).astype(np.int32)
        g1, g2 = n_pre, n_pre + n_suf
        if kind == "live":  # sparse pass: only the first `live` rows exist
            live = g2 + (M - g2) // 3
    else:
        pos = np.sort(rng.choice(T, M, replace=False)).astype(np.int32)
    q = rng.standard_normal((M, H * dh)).astype(np.float32)
    k = rng.standard_normal((T, Hkv * dh)).astype(np.float32)
    v = rng.standard_normal((T, Hkv * dh)).astype(np.float32)
    out = np.zeros((M, H * dh), np.float32)
    _check(lib().rk_debug_attention_bf16(P(engine.ptr), q.ctypes.data_as(F32P), k.ctypes.data_as(F32P),
                                         v.ctypes.data_as(F32P), pos.ctypes.data_as(C.POINTER(C.c_int32)),
                                         M, live, g1, g2, T, H, Hkv, dh, out.ctypes.data_as(F32P)))
    ref = ref_attention(q[:live], k, v, pos[:live], H, Hkv, dh)
    err = np.abs(out[:live] - ref).max()
    rel = np.linalg.norm(out[:live] - ref) / np.linalg.norm(ref)
    # bf16 operands are exact in the reference; the kernel rounds P and O to
    # bf16 (2^-9 relative each), so rel-L2 sits near 3e-3
    assert rel < 8e-3, f"rel-L2 err {rel}"
    assert err < 3e-2, f"max abs err {err}"
    assert (out[live:] == 0).all(), "rows beyond the live count were written"


def test_device_expf_matches_host_libm(engine):
    """The device restatement of glibc expf vs this host's libm, every 256th float."""
    from oracle.oracle import Oracle
    orc = Oracle("restatement")
    fn = orc.lib.orc_host_expf_array
    fn.argtypes = [F32P, F32P, C.c_uint64]
    x = (np.arange(0, 2 ** 32, 256, dtype=np.uint64).astype(np.uint32)).view(np.float32)
    x = np.ascontiguousarray(x[~np.isnan(x)])
    want = np.empty_like(x)
    fn(x.ctypes.data_as(F32P), want.ctypes.data_as(F32P), x.size)
    got = np.empty_like(x)
    _check(lib().rk_debug_expf(P(engine.ptr), x.ctypes.data_as(F32P), got.ctypes.data_as(F32P), C.c_uint64(x.size)))
    bad = np.flatnonzero(got.view(np.uint32) != want.view(np.uint32))
    assert bad.size == 0, f"{bad.size} mismatches, first x={x[bad[0]]!r}"


def ref_select(s_dev, infl, infl_mean, tau_dev, tau_inf, suffix_k):
    """selector.cpp:32-88 in plain Python (sequential double mean)."""
    n = len(s_dev)
    mean = 0.0
    for x in s_dev:
        mean += float(x)
    mean /= n
    thr = tau_dev * mean
    tags = {}
    if mean > 0:
        for j, x in enumerate(s_dev):
            if float(x) >= thr:
                tags[j] = tags.get(j, 0) | 1
    if infl_mean > 0:
        ti = tau_inf * infl_mean
        for j, x in enumerate(infl):
            if float(x) >= ti:
                tags[j] = tags.get(j, 0) | 2
    for j in range(max(0, n - suffix_k), n):
        tags[j] = tags.get(j, 0) | 4
    idx = sorted(tags)
    return np.array(idx, np.int32), np.array([tags[j] for j in idx], np.uint32), thr


@pytest.mark.parametrize("case", ["random", "ties", "zeros", "big"])
def test_select_certified_threshold(engine, case):
    """The certified parallel threshold must reproduce the sequential-mean
    selection bit for bit, including scores placed exactly on (and one ulp
    below) the reference's sequential threshold, which forces the fallback."""
    rng = np.random.default_rng(7)
    n = {"random": 1856, "ties": 1000, "zeros": 300, "big": 40000}[case]
    s = rng.random(n) * 0.02
    if case == "zeros":
        s[:] = 0.0
    infl = rng.random(n).astype(np.float32)
    infl_mean = float(np.mean(infl.astype(np.float64)))
    if case == "ties":
        _, _, thr = ref_select(s, infl, infl_mean, 1.5, 1.45, 10)
        for _ in range(8):  # the mean moves when scores change: iterate to a fixed point
            s[5] = thr
            s[6] = np.nextafter(thr, 0.0)
            s[7] = np.nextafter(thr, 1.0)
            _, _, thr = ref_select(s, infl, infl_mean, 1.5, 1.45, 10)
    want_idx, want_tags, thr = ref_select(s, infl, infl_mean, 1.5, 1.45, 10)
    idx = np.zeros(n, np.int32)
    tags = np.zeros(n, np.uint32)
    cnt = C.c_int32(0)
    dinfo = np.zeros(2, np.float64)
    _check(lib().rk_debug_select_relay(P(engine.ptr), s.ctypes.data_as(C.POINTER(C.c_double)),
                                       infl.ctypes.data_as(F32P), C.c_double(infl_mean), n, C.c_double(1.5),
                                       C.c_double(1.45), 10, idx.ctypes.data_as(C.POINTER(C.c_int32)),
                                       tags.ctypes.data_as(C.POINTER(C.c_uint32)), C.byref(cnt),
                                       dinfo.ctypes.data_as(C.POINTER(C.c_double))))
    assert np.array_equal(idx[:cnt.value], want_idx)
    assert np.array_equal(tags[:cnt.value], want_tags)
    if case != "zeros":
        assert dinfo[0] == thr, (dinfo[0], thr)


def test_gemm_single_cta_kernel():
    """The 1-CTA GEMM kernel (RK_GEMM_PAIR=0; the default uses CTA pairs for
    M > 128) on the store / residual / live-row shapes, in a subprocess."""
    import os
    import subprocess
    import sys
    code = f"""
import numpy as np, sys
sys.path.insert(0, {os.getcwd()!r})
from paper_2603_13289_b200.engine import Engine
from tests.test_gpu_kernels import run_gemm, bf16_round, SHAPES
e = Engine(0)
for (M, N, K) in SHAPES + [(1356, 2048, 2048), (320, 16384, 2048)]:
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    H = rng.standard_normal((M, N)).astype(np.float32)
    for epi, C0 in ((3, np.zeros((M, N))), (1, H)):
        got = run_gemm(e, A, B, C0, M, epi)
        ref = C0 + bf16_round(A).astype(np.float64) @ bf16_round(B).astype(np.float64).T
        err = np.abs(got - ref).max() / np.abs(ref).max()
        assert err < 2e-5, (M, N, K, epi, err)
print("ok")
"""
    env = dict(os.environ, RK_GEMM_PAIR="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("shape", [(1, 2048, 8192), (1, 4096, 14336), (1, 64, 64)])
def test_gemv_residual(engine, shape):
    """M = 1 residual GEMMs run as the CUDA-core GEMV; same result as fp64."""
    M, N, K = shape
    rng = np.random.default_rng(N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    H = rng.standard_normal((M, N)).astype(np.float32)
    got = run_gemm(engine, A, B, H, M, 1)
    ref = H + bf16_round(A).astype(np.float64) @ bf16_round(B).astype(np.float64).T
    assert np.abs(got - ref).max() / np.abs(ref).max() < 2e-5


SWAP_SHAPES = [(7, 256, 128), (200, 512, 512), (320, 16384, 2048), (333, 1024, 2048), (320, 2048, 8192),
               (64, 3072, 2048), (256, 2048, 8192), (129, 256, 64), (512, 768, 1024), (2, 256, 256)]


def test_gemm_swap_ab_pair():
    """The swap-AB CTA-pair kernel (weights on the MMA's M side, tokens on N;
    forced with RK_GEMM_SWAP=2 for every M <= 512, N % 256 == 0) on store and
    residual (split-K partials) GEMMs, in a subprocess: fp64 agreement and
    deterministic residuals."""
    import os
    import subprocess
    import sys
    code = f"""
import numpy as np, sys
sys.path.insert(0, {os.getcwd()!r})
from paper_2603_13289_b200.engine import Engine
from tests.test_gpu_kernels import run_gemm, bf16_round, SWAP_SHAPES
e = Engine(0)
for (M, N, K) in SWAP_SHAPES:
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    H = rng.standard_normal((M, N)).astype(np.float32)
    for epi, C0 in ((3, np.zeros((M, N))), (1, H)):
        got = run_gemm(e, A, B, C0, M, epi)
        ref = C0 + bf16_round(A).astype(np.float64) @ bf16_round(B).astype(np.float64).T
        err = np.abs(got - ref).max() / np.abs(ref).max()
        assert err < 2e-5, (M, N, K, epi, err)
        if epi == 1:
            again = run_gemm(e, A, B, C0, M, epi)
            assert np.array_equal(got.view(np.uint32), again.view(np.uint32)), (M, N, K)
print("ok")
"""
    env = dict(os.environ, RK_GEMM_SWAP="2", RK_GEMM_LOG="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
    assert "swap" in r.stderr, "the swap kernel was not selected"



@pytest.mark.parametrize("case", ["random", "ties", "zeros", "big", "none", "all", "over"])
def test_select_topk_radix(engine, case):
    """BLEND's top_k_by_score (selector.cpp:90-105) as a device radix select:
    the count largest scores, ties broken by ascending index (the reference's
    stable sort), returned ascending -- including heavy ties and k = 0 / n / > n."""
    rng = np.random.default_rng(13)
    n, k = {"random": (1856, 371), "ties": (1000, 333), "zeros": (300, 100), "big": (40000, 2000),
            "none": (500, 0), "all": (500, 500), "over": (64, 99)}[case]
    s = rng.random(n) * 3.0
    if case == "ties":
        s = np.round(s * 4) / 4  # a dozen distinct values
    if case == "zeros":
        s[:] = 0.0
    if case == "big":
        s[::7] = s[3]  # a large tie class straddling the cut
    order = sorted(range(n), key=lambda j: (-s[j], j))[:min(k, n)]
    want = np.array(sorted(order), np.int32)
    idx = np.zeros(n + 1, np.int32)
    cnt = C.c_int32(-1)
    _check(lib().rk_debug_select_topk(P(engine.ptr), np.ascontiguousarray(s).ctypes.data_as(C.POINTER(C.c_double)), n, k,
                                      idx.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(cnt)))
    assert cnt.value == len(want)
    assert np.array_equal(idx[:cnt.value], want)


@pytest.mark.parametrize("case", [(1360, 2048, 8192, 1, 1360), (700, 2048, 2048, 3, 700), (1500, 1600, 1024, 1, 1111),
                                  (900, 16384, 512, 3, 900)])
def test_gemm_pair_bn192_ragged_n(case, tmp_path):
    """CTA-pair tiles 192 columns wide with a ragged last N tile (N % 192 != 0:
    the tile's rows past N are TMA zero fill and are never stored), forced by
    RK_GEMM_OVERRIDE in a subprocess; residual (EPI_ADD, with live rows on the
    device) and plain-store epilogues against fp64."""
    import os
    import subprocess
    import sys
    M, N, K, epi, live = case
    rng = np.random.default_rng(M + N)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    H = rng.standard_normal((M, N)).astype(np.float32)
    np.savez(tmp_path / "in.npz", A=A, B=B, H=H)
    code = f"""
import numpy as np, sys
sys.path.insert(0, {os.getcwd()!r})
from paper_2603_13289_b200.engine import Engine
from tests.test_gpu_kernels import run_gemm
e = Engine(0)
d = np.load({str(tmp_path / "in.npz")!r})
np.save({str(tmp_path / "out.npy")!r}, run_gemm(e, d["A"], d["B"], d["H"], {live}, {epi}))
"""
    key = f"{M}{'d' if live < M else ''}:{N}:{K}=192/2/1"
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, RK_GEMM_OVERRIDE=key, RK_GEMM_LOG="1"),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bn=192 pair=2" in r.stderr, r.stderr
    got = np.load(tmp_path / "out.npy")
    prod = bf16_round(A[:live]).astype(np.float64) @ bf16_round(B).astype(np.float64).T
    ref = (H[:live] + prod) if epi == 1 else prod
    assert np.abs(got[:live] - ref).max() / np.abs(ref).max() < 2e-5
    if live < M:
        assert np.array_equal(got[live:], H[live:]), "rows past the live count were written"
