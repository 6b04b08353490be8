"""GPU coherence properties (tools/gpu/coherence.py at full
scale, profiles/r1_coherence.md): seeds attached to the surface keep the glint
pattern correlated under a small zoom, unlike re-seeding; and
output blending between LODs (the Zirr-style baseline, Eq. 7) lowers the count
variance at mid-blend while the distributed law keeps it (Fig. 4)."""
import importlib.util
import os

import pytest
import torch

pytestmark = pytest.mark.gpu

_HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def coh():
    spec = importlib.util.spec_from_file_location("coherence", os.path.join(_HERE, "..", "tools", "gpu", "coherence.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


@pytest.fixture(scope="module")
def ctx():
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import build
    build.build()
    c = pkg.Context(0)
    yield c
    c.close()


def test_zoom_pattern_correlation(ctx, coh):
    """8 steps of the C5 zoom (x1.245 area per step) on a 960x540 frame."""
    A = coh.zoom_experiment(ctx, torch.device("cuda", 0), 960, 540, steps=8, quad=6, zoom=1000.0 ** (7 / 63))
    m = A["methods"]
    assert m["ours"]["corr_1"] > 0.5 and m["zk"]["corr_1"] > 0.8
    assert abs(m["reseeded"]["corr_1"]) < 0.1
    assert m["ours"]["flicker"] < 0.7 * m["reseeded"]["flicker"]


def test_output_blending_lowers_variance(ctx, coh):
    B = coh.ghosting_experiment(ctx, torch.device("cuda", 0), n=512, steps=8)
    s = B["summary"]
    assert s["zk"]["var_rel_min"] < 0.5
    assert 0.75 < s["ours"]["var_rel_min"] and s["ours"]["var_rel_max"] < 1.6
