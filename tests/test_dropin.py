"""Drop-in proof: the reference's OWN doctest suites (raster, grad, core,
geometry, optimize) and its acceptance suite (acceptance.cpp C1-C10), compiled
unmodified, linked against the GPU path through the C++ adapter
(paper_2412_11752_b200/adapter/drk_adapter.cpp) instead of the reference's
render / bin_primitives / backward_render / eval_sorting / losses.  Built by
oracle/Makefile.ref (target `adapter`) where /root/reference exists; the
binaries travel to the GPU box.

Two precisions: the adapter's default reference-precision mode (fp64 alpha:
cache-sorted and exact-sort renders are bitwise comparable, as the raster
suite's "cache-sorted render equals the exact-sort oracle" case requires) and
DRK_ADAPTER_PRECISION=fast (the fp32 fast kernels that bench.py measures; that
one bitwise cross-mode case is excluded — the fp32 cache path and the fp64
exact-sort path agree to the parity tolerance, not bitwise).  Both use the
deterministic parallel backward."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_tests")
ACC = os.path.join(ROOT, "oracle", "_ref", "acceptance_adapter")

pytestmark = pytest.mark.gpu

# Cases the fp32 fast path cannot meet by construction: bitwise equality of the
# fp32 cache path with the fp64 exact-sort path, and central differences of
# renders with h = 1e-4 (fp32 alpha noise ~1e-7 / 1e-4 = 1e-3 relative per
# probe; the cases' bars are 1e-2 and 1e-4) — they run in reference precision.
FAST_EXCLUDE = ",".join([
    "cache-sorted render equals the exact-sort oracle under low overlap",
    "end-to-end gradients match finite differences on a tiny render",
    "loss-level translation equivariance between centers and camera",
])
FAST_ACCEPTANCE_SKIP = ("C4", "C6")  # finite differences at h = 1e-4; bitwise cache vs exact sort


def _env(precision):
    env = dict(os.environ)
    env["DRK_ADAPTER_PRECISION"] = precision
    return env


@pytest.mark.skipif(not os.path.exists(BIN), reason="adapter test binary not built")
@pytest.mark.parametrize("precision", ["reference", "fast"])
@pytest.mark.parametrize("suite", ["raster", "grad", "core", "geometry", "optimize"])
def test_reference_suite_through_gpu_adapter(suite, precision):
    args = [BIN, f"-ts={suite}"]
    if precision == "fast":
        args.append(f"-tce={FAST_EXCLUDE}")
    r = subprocess.run(args, capture_output=True, text=True, timeout=1200, env=_env(precision))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "0 failed" in r.stdout


@pytest.mark.skipif(not os.path.exists(ACC), reason="acceptance binary not built")
@pytest.mark.parametrize("precision", ["reference", "fast"])
def test_reference_acceptance_through_gpu_adapter(precision):
    """acceptance.cpp criteria on the GPU path: C4 gradients (alpha FD + 8x8 scene FD
    through finite_diff_check -> render / backward_render), C5 culling
    (bin_primitives vs brute force, sigma up to e^0.75 at z ~ 2: near-clipped
    polygons), C6 sorting (bitwise cache vs exact, Kendall-tau ordering through
    eval_sorting), C10 determinism (two train runs: scene and image bytes equal),
    plus the cheap C1-C3 and C8 (mesh conversion rendered on the GPU)."""
    crit = ["C1", "C2", "C3", "C4", "C5", "C6", "C8", "C10"]
    if precision == "fast":
        crit = [c for c in crit if c not in FAST_ACCEPTANCE_SKIP]
    r = subprocess.run([ACC, *crit], capture_output=True, text=True, timeout=1200, env=_env(precision))
    out = r.stdout
    assert r.returncode == 0, out[-4000:] + r.stderr[-3000:]
    for c in crit:
        assert any(ln.startswith("PASS - " + c + " ") for ln in out.splitlines()), (c, out)
