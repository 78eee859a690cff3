"""The C ABI library loads on a CPU-only host, exports every entry point the
headers in include/ declare, agrees with the ctypes struct layouts, and fails
loudly (a status + message, no crash, no fallback) when no GPU is present."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

from paper_2603_13289_b200 import abi
from paper_2603_13289_b200.engine import LIB_PATH, lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in ("relaykv_b200.h", "relaykv_b200_debug.h")]


def declared():
    names = set()
    for h in HEADERS:
        txt = open(h).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        names |= set(re.findall(r"\b(rk_[a-z0-9_]+)\s*\(", txt))
    return names


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = sorted(declared() - exported)
    assert not missing, f"declared but not exported: {missing}"
    assert len(declared()) >= 30


def test_library_loads_and_reports_version():
    assert lib().rk_abi_version() == 1


STRUCTS = {
    "rk_model_spec": abi.ModelSpec, "rk_layer_profile": abi.LayerProfile, "rk_relay_options": abi.RelayOptions,
    "rk_relay_cache_view": abi.RelayCacheView, "rk_phase_timings": abi.PhaseTimings,
    "rk_reuse_stats": abi.ReuseStats, "rk_relay_output": abi.RelayOutput,
}


def test_struct_layouts_match_header():
    src = '#include <stdio.h>\n#include <stddef.h>\n#include "relaykv_b200.h"\nint main(void){\n'
    for cname, py in STRUCTS.items():
        src += f'printf("{cname} %zu\\n", sizeof({cname}));\n'
        for f, _ in py._fields_:
            src += f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));\n'
    src += "return 0;}\n"
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "l.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "l")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        got = dict(line.split() for line in subprocess.run([exe], capture_output=True, text=True).stdout.splitlines())
    for cname, py in STRUCTS.items():
        assert int(got[cname]) == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, f"{cname}.{f}"


def test_flop_model_matches_reference_formula():
    """rk_flops_* restate relay_engine.cpp:72-110 (checked against oracle/_ref when built)."""
    from paper_2603_13289_b200.engine import flops_segment_schedule, flops_span_full
    from tests.scenarios import spec_of
    spec = spec_of(16, 128, 4)
    d, kv, ff, dhH = 128.0, 128.0, 256.0, 128.0
    pm = 2 * d * (2 * d + 2 * kv) + 6 * d * ff
    assert flops_span_full(spec, 64, 100) == 16 * 100 * pm + 16 * 4 * dhH * (100 * 64 + 100 * 101 / 2)
    # select-all full-range schedule == full prefill cost (test_engine.cpp:210-222)
    assert flops_segment_schedule(spec, 0, 100, 0, 0, 15, 100) + 0 == pytest.approx(flops_span_full(spec, 0, 100))
    from oracle.oracle import Oracle, available
    if available("reference"):
        ref = Oracle("reference")
        for args in [(64, 100, 1, 3, 10, 12), (0, 7, 0, 0, 15, 7), (300, 512, 2, 2, 9, 80)]:
            assert flops_segment_schedule(spec, *args) == ref.flops_segment_schedule(spec, *args)
        assert flops_span_full(spec, 17, 333) == ref.flops_span_full(spec, 17, 333)


def test_engine_create_fails_loudly_without_gpu():
    from tests.conftest import HAS_GPU
    if HAS_GPU:
        pytest.skip("a GPU is present")
    from paper_2603_13289_b200.engine import Engine
    with pytest.raises(abi.StatusError) as ei:
        Engine(0)
    assert ei.value.code != 0 and str(ei.value)
