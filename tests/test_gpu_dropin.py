"""The C++ drop-in (namespace relaykv over the C ABI) passes the reference's
relay-engine test scenarios, rewritten against it (tests/cpp/test_dropin.cpp),
on the B200 -- including a bitwise cross-check against the oracle."""
import os
import subprocess

import pytest

from paper_2603_13289_b200.build import DROPIN_TEST


def test_dropin_binary_is_built():
    assert os.path.exists(DROPIN_TEST), "run python -m paper_2603_13289_b200.build"


@pytest.mark.gpu
def test_dropin_reference_scenarios_on_gpu():
    p = subprocess.run([DROPIN_TEST], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "failed: 0" in p.stdout


REF_ENGINE_TESTS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                                "engine_tests_on_dropin")


@pytest.mark.gpu
def test_reference_engine_tests_unmodified_on_dropin():
    """The reference's OWN tests/test_engine.cpp (+ test_main.cpp), compiled
    unmodified against the drop-in headers (oracle/Makefile dropin_ref), run
    on the B200: every case -- degenerate FULL bit-equality, ZERO round trip,
    the accounting formula (450 entries, reuse 0.859375), BLEND counting
    (201-208), the FLOP-model identities (210-244), suffix isolation,
    validation throws, selection diagnostics and the 12-seed monotone
    fidelity ladder (331-378)."""
    if not os.path.exists(REF_ENGINE_TESTS):
        pytest.skip("built only where /root/reference exists (make -C oracle dropin_ref)")
    p = subprocess.run([REF_ENGINE_TESTS], capture_output=True, text=True, timeout=900)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-4000:]
    assert "CHECK FAILED" not in out, out[-4000:]
    print(out[-600:])
