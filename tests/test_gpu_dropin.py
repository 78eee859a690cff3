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
