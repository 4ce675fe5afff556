"""Drop-in proof: the reference's OWN doctest suites (raster, grad, core,
geometry, optimize), compiled unmodified, linked against the GPU path through
the C++ adapter (paper_2412_11752_b200/adapter/drk_adapter.cpp) instead of the
reference's render / bin_primitives / backward_render.  Built by
oracle/Makefile.ref (target `adapter`) where /root/reference exists; the
binary travels to the GPU box."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_tests")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="adapter test binary not built")
@pytest.mark.parametrize("suite", ["raster", "grad", "core", "geometry", "optimize"])
def test_reference_suite_through_gpu_adapter(suite):
    r = subprocess.run([BIN, f"-ts={suite}"], capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "0 failed" in r.stdout
