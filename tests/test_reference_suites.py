"""The reference's own doctest suites (core, geometry, raster, grad, optimize),
compiled unmodified against the header shims (oracle/_ref/ref_tests).  Passing
them validates the shims and therefore the oracle build that pins everything
else.  CPU only."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "ref_tests")


@pytest.mark.skipif(not os.path.exists(BIN), reason="reference build missing")
@pytest.mark.parametrize("suite", ["core", "geometry", "raster", "grad", "optimize"])
def test_reference_suite(suite):
    r = subprocess.run([BIN, f"-ts={suite}"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout
