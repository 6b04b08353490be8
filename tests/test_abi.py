"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/glint.h declares, rejects bad arguments before touching the GPU, and
its host-built tables are bit-identical to the oracle's independently built
ones."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def glib():
    from paper_2306_05051_b200 import build
    build.build()
    import paper_2306_05051_b200 as pkg
    return pkg


def test_exports_match_header(glib):
    hdr = open(os.path.join(ROOT, "include", "glint.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char\*|int64_t)\s+\*?(glint_\w+)\s*\(", hdr, re.M))
    assert declared == set(glib._lib.EXPORTS)
    L = glib.lib()
    for name in declared:
        assert hasattr(L, name)
    assert glib.version() == 10000
    assert glib.strerror(-1) == "invalid argument"


def test_tables_bit_identical_to_oracle(glib, orc):
    z, c, s = glib.build_tables()
    assert np.array_equal(z.view(np.uint32), orc.ztable().view(np.uint32))
    assert np.array_equal(c.view(np.uint32), orc.costable().view(np.uint32))
    assert np.array_equal(s.view(np.uint32), orc.sintable().view(np.uint32))


def test_argument_errors_without_gpu(glib):
    L = glib.lib()
    sc = glib._lib.glint_scene()
    gb = glib._lib.glint_gbuffer()
    assert L.glint_eval(None, C.byref(gb), C.byref(sc), None, 0, None, None) == glib._lib.GLINT_EINVAL
    assert L.glint_create(None, 0) == glib._lib.GLINT_EINVAL
    h = C.c_void_p()
    import torch
    if not torch.cuda.is_available():
        assert L.glint_create(C.byref(h), 0) == glib._lib.GLINT_EDEVICE
        with pytest.raises(glib.GlintError):
            glib.Context(0)


def test_scene_struct_layout(glib):
    assert C.sizeof(glib._lib.glint_light) == 32
    assert C.sizeof(glib._lib.glint_scene) == 64 + 16 * 32
    assert C.sizeof(glib._lib.glint_gbuffer) == 5 * 8 + 4 + 4 + 8
