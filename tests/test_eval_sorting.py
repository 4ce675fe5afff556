"""eval_sorting (reference raster.cpp:487-560) on the
GPU: per-pixel processed-depth sequences (SortCache pops or list order) of the GPU
tile lists, Kendall tau by merge-sort pair counting, MAE, ordered fraction —
identical to the reference build for every presort mode, with and without the
cache (per-pixel values are the reference's exactly and are summed in its order)."""
from __future__ import annotations

import pytest

from oracle import ref
from paper_2412_11752_b200 import scenes

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref.available(), reason="reference build missing")]


@pytest.mark.parametrize("presort,use_cache", [(2, True), (1, True), (0, True), (0, False), (2, False)])
def test_eval_sorting_matches_reference(rast, presort, use_cache):
    from paper_2412_11752_b200.api import PresortMode
    sc = scenes.random_scene(300, seed=41, sh_degree=0, clusters=4)
    cam = scenes.look_at_camera(72, 40, (0.4, -0.3, -3.6))
    want = ref.eval_sorting(sc, cam, ref.Options(presort=presort, use_cache=use_cache, sh_degree=0))
    got = rast.eval_sorting(sc.f32(), cam, presort=PresortMode(presort), use_cache=use_cache, k=sc.k)
    assert got.pixels == want[3] and got.pixels > 0
    assert (got.accuracy, got.kendall_tau, got.mae) == want[:3]


def test_eval_sorting_presort_quality_order(rast):
    """The reference suite's property (test_raster.cpp:266-280): NearestDepth presort
    plus the cache sorts at least as well as list order without presort."""
    from paper_2412_11752_b200.api import PresortMode
    sc = scenes.random_scene(500, seed=42, sh_degree=0, clusters=6)
    cam = scenes.look_at_camera(96, 64, (0.0, 0.2, -3.4))
    best = rast.eval_sorting(sc.f32(), cam, presort=PresortMode.NearestDepth, use_cache=True, k=sc.k)
    worst = rast.eval_sorting(sc.f32(), cam, presort=PresortMode.None_, use_cache=False, k=sc.k)
    assert best.kendall_tau >= worst.kendall_tau
