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
    assert glib.version() == 20100
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
    assert C.sizeof(glib._lib.glint_gbuffer) == 5 * 8 + 4 + 4 + 8 + 4 + 4   # + tile origin (x0, y0)


@pytest.mark.skipif(__import__("torch").cuda.is_available(),
                    reason="fake, never dereferenced addresses are safe only where the device check fails "
                           "(a passing call would dereference the fake context)")
def test_batch_validation_and_alias_rules_without_gpu(glib):
    """glint_eval_batch validates every frame and the output/input overlap
    rule before it touches the context or the device (include/glint.h), so
    the rules run here on fake, never dereferenced, 16-byte-aligned
    addresses: any output overlapping any frame's input plane or another
    output -> GLINT_EALIAS; disjoint (even adjacent) ranges pass validation
    and only then fail on the missing device."""
    import torch
    L = glib.lib()
    m = glib._lib
    W, H, pitch = 64, 8, 64
    plane = pitch * H * 16                      # bytes of one plane

    def frame(base):
        g = m.glint_gbuffer()
        g.duv, g.uvm, g.nrm, g.pos, g.mat = [base + k * plane for k in range(5)]
        g.width, g.height, g.pitch = W, H, pitch
        return g

    sc = glib._lib.scene_struct(__import__("paper_2306_05051_b200.synth", fromlist=["x"]).SceneParams())
    G = (m.glint_gbuffer * 2)(frame(0x10000000), frame(0x20000000))
    S = (m.glint_scene * 2)(sc, sc)
    Q = (C.c_int64 * 2)(pitch, pitch)
    fake_ctx = C.c_void_p(0x1000)               # validation never dereferences it

    def run(o0, o1):
        P = (C.c_void_p * 2)(o0, o1)
        return L.glint_eval_batch(fake_ctx, 2, G, S, P, Q, None)

    out = 0x30000000
    assert run(out, 0x10000000 + 2 * plane) == m.GLINT_EALIAS          # over frame 0's nrm plane
    assert run(out, 0x20000000 + 4 * plane + 16 * 5) == m.GLINT_EALIAS  # inside frame 1's mat plane
    assert run(out, out) == m.GLINT_EALIAS                              # two outputs overlap
    assert run(out, out + plane - 16) == m.GLINT_EALIAS                 # overlap by one float4
    assert run(0x20000000 - plane + 16, out) == m.GLINT_EALIAS          # last float4 reaches frame 1's duv
    assert run(out, out + 4 * 3) == m.GLINT_EALIGN                      # misaligned second output
    rc = run(out, out + plane)                                          # adjacent: valid, then needs the device
    if not torch.cuda.is_available():
        assert rc == m.GLINT_ECUDA or rc == m.GLINT_EDEVICE
    # frame-level validation still applies, and n_frames = 0 is a no-op
    bad = (m.glint_scene * 2)(sc, sc)
    bad[1].ndf_kind = 7
    P = (C.c_void_p * 2)(out, out + plane)
    assert L.glint_eval_batch(fake_ctx, 2, G, bad, P, Q, None) == m.GLINT_EINVAL
    assert L.glint_eval_batch(fake_ctx, 0, None, None, None, None, None) == m.GLINT_OK
    assert L.glint_eval_batch(None, 2, G, S, P, Q, None) == m.GLINT_EINVAL
    assert L.glint_eval_batch(fake_ctx, -1, G, S, P, Q, None) == m.GLINT_EINVAL


@pytest.mark.skipif(__import__("torch").cuda.is_available(),
                    reason="fake, never dereferenced addresses are safe only where the device check fails "
                           "(a passing call would dereference the fake context)")
def test_batch_alias_rule_against_brute_force(glib):
    """The output-overlap rule of glint_eval_batch (include/glint.h) against a
    brute-force pixel-set intersection over random pitched regions (fake,
    never dereferenced addresses; no GPU): exact when the two regions share a
    pitch (or one is a single row that fits the other's pitch), and never
    missing a real overlap otherwise (conservative)."""
    import random
    import torch
    L = glib.lib()
    m = glib._lib
    sc = m.scene_struct(__import__("paper_2306_05051_b200.synth", fromlist=["x"]).SceneParams())
    S2 = (m.glint_scene * 2)(sc, sc)
    fake = C.c_void_p(0x1000)
    rng = random.Random(1)
    for _ in range(6000):
        P1, P2 = rng.choice([(8, 8), (8, 8), (6, 8), (8, 5)])
        w1, h1, w2, h2 = rng.randint(1, P1), rng.randint(1, 5), rng.randint(1, P2), rng.randint(1, 5)
        base = 0x100000
        o1, o2 = base + 16 * rng.randint(0, 60), base + 16 * rng.randint(0, 60)
        px1 = {o1 // 16 + r * P1 + c for r in range(h1) for c in range(w1)}
        px2 = {o2 // 16 + r * P2 + c for r in range(h2) for c in range(w2)}
        truth = bool(px1 & px2)
        g0, g1 = m.glint_gbuffer(), m.glint_gbuffer()
        g0.duv = g0.uvm = g0.nrm = g0.pos = g0.mat = 0x40000000
        g1.duv = g1.uvm = g1.nrm = g1.pos = g1.mat = 0x50000000
        g0.width, g0.height, g0.pitch = w1, h1, w1
        g1.width, g1.height, g1.pitch = w2, h2, w2
        G = (m.glint_gbuffer * 2)(g0, g1)
        rc = L.glint_eval_batch(fake, 2, G, S2, (C.c_void_p * 2)(o1, o2), (C.c_int64 * 2)(P1, P2), None)
        refused = rc == m.GLINT_EALIAS
        if not torch.cuda.is_available():
            assert refused or rc in (m.GLINT_ECUDA, m.GLINT_EDEVICE)
        exact = P1 == P2 or (h1 == 1 and w1 <= P2) or (h2 == 1 and w2 <= P1)
        if exact:
            assert refused == truth, (P1, P2, w1, h1, w2, h2, o1 - base, o2 - base)
        else:
            assert refused or not truth, (P1, P2, w1, h1, w2, h2, o1 - base, o2 - base)


@pytest.mark.skipif(__import__("torch").cuda.is_available(),
                    reason="fake, never dereferenced addresses are safe only where the device check fails")
def test_tile_origins_in_one_output_alias_rule_without_gpu(glib):
    """Row bands of one frame written into ONE full-frame output through their
    tile origins (glint.h x0, y0; SURVEY 8e sharding): disjoint bands pass the
    batch's alias rule, overlapping bands are refused, a negative origin is
    invalid and an origin past 2^40 float4 is refused as too large -- all
    before the context or device is touched."""
    import torch
    L = glib.lib()
    m = glib._lib
    W, Hb, pitch = 64, 8, 64
    plane = pitch * Hb * 16
    sc = m.scene_struct(__import__("paper_2306_05051_b200.synth", fromlist=["x"]).SceneParams())
    fake = C.c_void_p(0x1000)

    def band(base, y0, x0=0):
        g = m.glint_gbuffer()
        g.duv, g.uvm, g.nrm, g.pos, g.mat = [base + k * plane for k in range(5)]
        g.width, g.height, g.pitch, g.x0, g.y0 = W, Hb, pitch, x0, y0
        return g

    out = 0x70000000
    S = (m.glint_scene * 2)(sc, sc)
    Q = (C.c_int64 * 2)(W, W)
    P = (C.c_void_p * 2)(out, out)                   # the same full-frame output for both bands

    def run(g0, g1):
        return L.glint_eval_batch(fake, 2, (m.glint_gbuffer * 2)(g0, g1), S, P, Q, None)

    rc = run(band(0x10000000, 0), band(0x20000000, Hb))            # rows 0-7 and 8-15
    assert rc in (m.GLINT_ECUDA, m.GLINT_EDEVICE)
    assert run(band(0x10000000, 0), band(0x20000000, Hb - 1)) == m.GLINT_EALIAS   # one shared row
    assert run(band(0x10000000, 0), band(0x20000000, 3)) == m.GLINT_EALIAS
    assert run(band(0x10000000, 0, x0=-1), band(0x20000000, Hb)) == m.GLINT_EINVAL
    G = (m.glint_gbuffer * 2)(band(0x10000000, 0), band(0x20000000, 64))
    Qbig = (C.c_int64 * 2)(W, 2 ** 34)                                  # (64 + 8) rows x 2^34 >= 2^40
    assert L.glint_eval_batch(fake, 2, G, S, P, Qbig, None) == m.GLINT_ELIMIT
