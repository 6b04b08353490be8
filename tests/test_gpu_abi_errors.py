"""Error behaviour of the C ABI on a GPU (include/glint.h): every documented
GLINT_E* condition is reported before anything is launched, the output is left
untouched, and a valid call right after still succeeds."""
import ctypes as C

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import _lib, build, synth
    build.build()
    ctx = pkg.Context(0)
    fr = synth.c2(35, window=(600, 632, 0, 64), device="cuda")
    yield pkg, _lib, ctx, fr
    ctx.close()


def _call(_lib, ctx, g, sc, out, dbg=None, out_pitch=None):
    if out_pitch is None:
        out_pitch = max(out.stride(0) // 4, g.width) if out is not None else 0
    return _lib.lib().glint_eval(ctx.handle, C.byref(g), C.byref(sc), out.data_ptr() if out is not None else None,
                                 out_pitch, dbg, None)


def test_error_codes(env):
    pkg, L, ctx, fr = env
    out = torch.full((32, 64, 4), 7.0, device="cuda")
    g, sc = L._gbuffer_struct(fr.gbuf), L.scene_struct(fr.scene)
    assert _call(L, ctx, g, sc, out, out_pitch=64) == L.GLINT_OK
    torch.cuda.synchronize()
    ref = out.clone()
    out.fill_(7.0)
    cases = []
    bad = L._gbuffer_struct(fr.gbuf); bad.duv += 4; cases.append(("misaligned plane", bad, sc, L.GLINT_EALIGN))
    bad = L._gbuffer_struct(fr.gbuf); bad.pitch = 63; cases.append(("pitch < width", bad, sc, L.GLINT_EALIGN))
    bad = L._gbuffer_struct(fr.gbuf); bad.width, bad.height, bad.pitch = 65536, 32768, 65536
    cases.append(("2^31 pixels", bad, sc, L.GLINT_ELIMIT))
    bad = L._gbuffer_struct(fr.gbuf); bad.width = -1; cases.append(("negative width", bad, sc, L.GLINT_EINVAL))
    bad = L._gbuffer_struct(fr.gbuf); bad.mat = 0; cases.append(("null plane", bad, sc, L.GLINT_EINVAL))
    for field, val in (("eval_mode", 4), ("eval_mode", -1), ("max_ratio_level", 0), ("max_ratio_level", 9),
                       ("n_lights", 17), ("ndf_kind", 2), ("view_kind", 2)):
        s2 = L.scene_struct(fr.scene); setattr(s2, field, val); cases.append((f"{field}={val}", g, s2, L.GLINT_EINVAL))
    s2 = L.scene_struct(fr.scene); s2.beta = 0.0; cases.append(("beta = 0", g, s2, L.GLINT_EINVAL))
    s2 = L.scene_struct(fr.scene); s2.beta = float("nan"); cases.append(("beta = nan", g, s2, L.GLINT_EINVAL))
    for name, gg, ss, want in cases:
        assert _call(L, ctx, gg, ss, out) == want, name
    assert _call(L, ctx, g, sc, out, out_pitch=63) == L.GLINT_EALIGN                # output pitch < width
    assert _call(L, ctx, g, sc, None, out_pitch=64) == L.GLINT_EINVAL            # null output
    bad_out = torch.empty(32 * 64 * 4 + 1, device="cuda")[1:]                       # misaligned output
    assert L.lib().glint_eval(ctx.handle, C.byref(g), C.byref(sc), bad_out.data_ptr(), 64, None, None) == L.GLINT_EALIGN
    s2 = L.scene_struct(fr.scene); s2.eval_mode = 3                                  # debug records: mode 0 only
    dbg = torch.empty(32 * 64 * L.DEBUG_REC_BYTES, dtype=torch.uint8, device="cuda")
    assert _call(L, ctx, g, s2, out, C.c_void_p(dbg.data_ptr())) == L.GLINT_EINVAL
    torch.cuda.synchronize()
    assert torch.all(out == 7.0)                                                    # untouched
    assert _call(L, ctx, g, sc, out, out_pitch=64) == L.GLINT_OK                    # still usable
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int32), ref.view(torch.int32))
