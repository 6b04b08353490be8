"""glint_eval_batch (include/glint.h): independent frames in one call, their
launches chained with programmatic dependent launch. Every frame must equal
glint_eval's result bit for bit (itself parity-tested against the oracle), and
small batches are also compared with the oracle directly; outputs that alias
inputs or each other are refused before anything launches; work after the
batch on the stream sees every frame complete; the batch captures into a CUDA
graph."""
import numpy as np
import pytest
import torch

from test_gpu_parity import compare_radiance

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import build
    build.build()
    c = pkg.Context(0)
    yield c
    c.close()


def _same(a, b):
    return torch.equal(a.contiguous().view(torch.int32), b.contiguous().view(torch.int32))


def test_batch_matches_oracle_small_mixed(ctx):
    """Ragged sizes, 0/1/3/16 lights, every eval mode, an empty frame and a
    pitched view in one batch; each frame vs the oracle (radiance 1e-4,
    flags exact) and vs glint_eval (bit-identical)."""
    import oracle
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import synth
    gbs, scs = [], []
    for seed, shape, nl in ((11, (67, 13), 3), (12, (1, 1), 16), (13, (40, 129), 1), (14, (5, 300), 0),
                            (15, (33, 33), 2)):
        gbs.append(synth.random_gbuffer(*shape, seed=seed))
        scs.append(synth.random_scene(seed, n_lights=nl))
    scs[2].draws = 64
    scs[4].method = "zk"
    fr = synth.c2(35, window=(600, 664, 0, 200))
    gbs.append(fr.gbuf)
    scs.append(fr.scene)
    gbs.append(synth.GBuffer(*[p[:0] for p in fr.gbuf.planes()]))        # empty
    scs.append(fr.scene)
    dev = [g.to("cuda") for g in gbs]
    wide = dev[5]
    dev[5] = synth.GBuffer(*[p[:, 10:150] for p in wide.planes()])        # pitched view
    outs = pkg.glint_eval_batch(ctx, dev, scs)
    torch.cuda.synchronize()
    assert outs[6].numel() == 0
    for f in range(6):
        ref = pkg.glint_eval(ctx, dev[f], scs[f])
        torch.cuda.synchronize()
        assert _same(outs[f], ref), f"frame {f}: batch != glint_eval"
        host = gbs[f] if f != 5 else gbs[5].crop(0, 64, 10, 150)
        rgb_o, fl_o, _ = oracle.eval(host, scs[f])
        compare_radiance(outs[f], rgb_o, fl_o, f"batch frame {f}")


def test_batch_full_c2_step_bit_identical(ctx):
    """The bench's C2 step (10 full 1080p elevations) as one batch, repeated:
    bit-identical to 10 glint_eval launches, every time (tiles of consecutive
    frames overlap in time; their scheduler slots and outputs are separate)."""
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import synth
    frames = synth.c2_frames(device="cuda")
    refs = [pkg.glint_eval(ctx, fr.gbuf, fr.scene).clone() for fr in frames]
    outs = [torch.empty_like(r) for r in refs]
    for _ in range(3):
        for o in outs:
            o.fill_(float("nan"))
        pkg.glint_eval_batch(ctx, [fr.gbuf for fr in frames], [fr.scene for fr in frames], outs=outs)
        torch.cuda.synchronize()
        for f, (o, r) in enumerate(zip(outs, refs)):
            assert _same(o, r), f"elevation frame {f}"
    # the bench's launch configuration against the oracle directly: 800
    # sampled pixels of every frame, recomputed one by one on the CPU
    import oracle
    g = torch.Generator().manual_seed(7)
    for f, (fr, o) in enumerate(zip(frames, outs)):
        idx = torch.randint(0, fr.gbuf.height * fr.gbuf.width, (800,), generator=g)
        rgb_o, fl_o, _ = oracle.eval(fr.gbuf.take(idx).to("cpu"), fr.scene)
        compare_radiance(o.reshape(-1, 4)[idx.to(o.device)], rgb_o, fl_o, f"batch C2 frame {f}")


def test_batch_completion_is_ordered_before_later_stream_work(ctx):
    """Work enqueued on the stream right after the batch must see every frame
    complete. A slow full frame first, short frames after it (so the chained
    launches finish before the first one could): a device-side copy of all
    outputs issued immediately after the batch must equal the references."""
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import synth
    big = synth.c4(1, device="cuda")                         # 3840x2160, 16 lights
    small = [synth.c2(e, window=(500, 532, 0, 1920), device="cuda") for e in (15, 45, 75)]
    frames = [big] + small
    refs = [pkg.glint_eval(ctx, fr.gbuf, fr.scene).clone() for fr in frames]
    outs = [torch.empty_like(r) for r in refs]
    s = torch.cuda.current_stream()
    for _ in range(3):
        for o in outs:
            o.fill_(float("nan"))
        pkg.glint_eval_batch(ctx, [fr.gbuf for fr in frames], [fr.scene for fr in frames], outs=outs, stream=s)
        snap = [o.clone() for o in outs]                     # same stream, no host sync in between
        torch.cuda.synchronize()
        for f, (o, r) in enumerate(zip(snap, refs)):
            assert _same(o, r), f"frame {f} incomplete when the next stream op ran"


def test_batch_rejects_aliasing_outputs(ctx):
    """An output overlapping any frame's input plane, or another output, is
    refused with GLINT_EALIAS before anything launches."""
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import synth
    from paper_2306_05051_b200._lib import GLINT_EALIAS, GlintError
    frs = [synth.c2(e, window=(500, 532, 0, 256), device="cuda") for e in (15, 45)]
    gbs, scs = [fr.gbuf for fr in frs], [fr.scene for fr in frs]
    n0 = ctx.launch_count()
    o0 = torch.empty(32, 256, 4, device="cuda")
    cases = {
        "output over another frame's input": [o0, gbs[0].mat],
        "output over its own input": [gbs[0].duv, torch.empty(32, 256, 4, device="cuda")],
        "two outputs overlap": [o0, o0],
    }
    big = torch.empty(64, 256, 4, device="cuda")
    cases["outputs overlap by one row"] = [big[:32], big[31:63]]
    for what, outs in cases.items():
        with pytest.raises(GlintError) as ei:
            pkg.glint_eval_batch(ctx, gbs, scs, outs=outs)
        assert ei.value.code == GLINT_EALIAS, what
    assert ctx.launch_count() == n0
    # adjacent, non-overlapping outputs are fine
    pkg.glint_eval_batch(ctx, gbs, scs, outs=[big[:32], big[32:]])
    torch.cuda.synchronize()
    for f in range(2):
        assert _same(big[32 * f:32 * (f + 1)], pkg.glint_eval(ctx, gbs[f], scs[f]))
    assert pkg.glint_eval_batch(ctx, [], []) == []


def test_batch_graph_capture_and_replay(ctx):
    """A batch captured into a CUDA graph (programmatic edges between its
    launches) replays bit-identically."""
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import synth
    frames = [synth.c2(e, window=(300, 556, 0, 1920), device="cuda") for e in (25, 45, 65)]
    gbs, scs = [fr.gbuf for fr in frames], [fr.scene for fr in frames]
    refs = [pkg.glint_eval(ctx, g, s).clone() for g, s in zip(gbs, scs)]
    outs = [torch.empty_like(r) for r in refs]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        pkg.glint_eval_batch(ctx, gbs, scs, outs=outs, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        pkg.glint_eval_batch(ctx, gbs, scs, outs=outs, stream=torch.cuda.current_stream())
    for _ in range(3):
        for o in outs:
            o.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        for o, r in zip(outs, refs):
            assert _same(o, r)


def test_batch_launch_count_and_stats(ctx):
    """One launch per non-empty frame (bench's gpu_launches evidence)."""
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import synth
    frs = [synth.c2(e, window=(500, 532, 0, 256), device="cuda") for e in (15, 45, 75)]
    gbs = [fr.gbuf for fr in frs] + [synth.GBuffer(*[p[:0] for p in frs[0].gbuf.planes()])]
    scs = [fr.scene for fr in frs] + [frs[0].scene]
    n0 = ctx.launch_count()
    outs = pkg.glint_eval_batch(ctx, gbs, scs)
    torch.cuda.synchronize()
    assert ctx.launch_count() - n0 == 3
    assert all(np.isfinite(o[..., :3].cpu().numpy()).all() for o in outs[:3])


def test_batches_on_concurrent_streams(ctx):
    """Two batches in flight at once on two streams (their chains interleave
    on the SMs; every launch has its own scheduler slot): each frame still
    equals its glint_eval reference bit for bit."""
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import synth
    fa = [synth.c2(e, window=(200, 456, 0, 1920), device="cuda") for e in (15, 35, 55)]
    fb = [synth.c2(e, window=(600, 856, 0, 1920), device="cuda") for e in (25, 45, 65, 85)]
    refs = {id(fr): pkg.glint_eval(ctx, fr.gbuf, fr.scene).clone() for fr in fa + fb}
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        oa = [torch.full_like(refs[id(fr)], float("nan")) for fr in fa]
        ob = [torch.full_like(refs[id(fr)], float("nan")) for fr in fb]
        sa.wait_stream(torch.cuda.current_stream())
        sb.wait_stream(torch.cuda.current_stream())
        pkg.glint_eval_batch(ctx, [f.gbuf for f in fa], [f.scene for f in fa], outs=oa, stream=sa)
        pkg.glint_eval_batch(ctx, [f.gbuf for f in fb], [f.scene for f in fb], outs=ob, stream=sb)
        torch.cuda.synchronize()
        for fr, o in list(zip(fa, oa)) + list(zip(fb, ob)):
            assert _same(o, refs[id(fr)])


def test_host_batch_matches_per_frame_host_entry(ctx):
    """glint_eval_host_batch (one copy/compute pipeline across frames) equals
    glint_eval_host frame by frame, bit for bit: frames of different widths
    (the chunk stage is sized for the largest), one larger than a 1M-pixel
    chunk (several chunks per frame), a pitched host view, an empty frame."""
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import synth
    frs = [synth.c2(25), synth.c2(65, window=(300, 420, 0, 700)), synth.c2(45, window=(500, 501, 0, 1920))]
    gbs = [fr.gbuf.pin() for fr in frs]
    wide = synth.c2(85, window=(600, 664, 0, 400)).gbuf.pin()
    gbs.append(synth.GBuffer(*[p[:, 30:330] for p in wide.planes()]))       # pitched host view
    gbs.append(synth.GBuffer(*[p[:0] for p in wide.planes()]))              # empty
    scs = [fr.scene for fr in frs] + [frs[0].scene, frs[0].scene]
    outs = pkg.glint_eval_host_batch(ctx, gbs, scs)
    assert outs[4].numel() == 0
    for f in range(4):
        ref = pkg.glint_eval_host(ctx, gbs[f], scs[f])
        assert _same(outs[f], ref), f"frame {f}"
    dev = pkg.glint_eval(ctx, gbs[0].to("cuda"), scs[0])
    torch.cuda.synchronize()
    assert _same(outs[0], dev.cpu())


def test_host_batch_rejects_aliasing(ctx):
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import synth
    from paper_2306_05051_b200._lib import GLINT_EALIAS, GlintError
    frs = [synth.c2(e, window=(500, 532, 0, 256)) for e in (15, 45)]
    gbs = [fr.gbuf.pin() for fr in frs]
    with pytest.raises(GlintError) as ei:
        pkg.glint_eval_host_batch(ctx, gbs, [fr.scene for fr in frs], outs=[torch.empty(32, 256, 4), gbs[0].nrm])
    assert ei.value.code == GLINT_EALIAS


def test_batches_write_pitched_outputs(ctx):
    """Pitched outputs (out_pitch > width): two frames written side by side
    as column views of one wide buffer (interleaved rows, no common pixel)
    are accepted (the alias rule is exact for equal pitches), overlapping
    column views are refused, pitched views into separate buffers leave their
    padding untouched; all bit-identical to glint_eval; device and host batch
    entries."""
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import synth
    from paper_2306_05051_b200._lib import GLINT_EALIAS, GlintError
    frs = [synth.c2(e, window=(400, 464, 0, 300), device="cuda") for e in (25, 55)]
    gbs, scs = [fr.gbuf for fr in frs], [fr.scene for fr in frs]
    refs = [pkg.glint_eval(ctx, g, s) for g, s in zip(gbs, scs)]
    wide = torch.full((64, 600, 4), 7.0, device="cuda")
    # side-by-side column views of one buffer: disjoint pixels -> accepted
    outs = pkg.glint_eval_batch(ctx, gbs, scs, outs=[wide[:, :300], wide[:, 300:]])
    torch.cuda.synchronize()
    assert _same(wide[:, :300], refs[0]) and _same(wide[:, 300:], refs[1])
    # overlapping column views (columns 250..299 shared) -> refused
    with pytest.raises(GlintError) as ei:
        pkg.glint_eval_batch(ctx, gbs, scs, outs=[wide[:, :300], wide[:, 250:550]])
    assert ei.value.code == GLINT_EALIAS
    # pitched views into two separate wide buffers: accepted
    w0 = torch.full((64, 400, 4), 7.0, device="cuda")
    w1 = torch.full((64, 400, 4), 7.0, device="cuda")
    outs = pkg.glint_eval_batch(ctx, gbs, scs, outs=[w0[:, 50:350], w1[:, 100:400]])
    torch.cuda.synchronize()
    for o, r in zip(outs, refs):
        assert _same(o, r)
    assert torch.all(w0[:, :50] == 7.0) and torch.all(w0[:, 350:] == 7.0) and torch.all(w1[:, :100] == 7.0)
    # host entry with pitched host outputs
    h0 = torch.full((64, 400, 4), 7.0).pin_memory()
    h1 = torch.full((64, 400, 4), 7.0).pin_memory()
    hin = [fr.gbuf.to("cpu").pin() for fr in frs]
    houts = pkg.glint_eval_host_batch(ctx, hin, scs, outs=[h0[:, 50:350], h1[:, 100:400]])
    for o, r in zip(houts, refs):
        assert _same(o, r.cpu())
    assert torch.all(h0[:, :50] == 7.0) and torch.all(h1[:, :100] == 7.0)


def test_host_batch_mixed_eval_modes(ctx):
    """One host batch mixing the method (48 draws), its 64/160-draw ablations
    and the Zirr-style baseline: each chunk's launch takes its own frame's
    mode; every frame equals its glint_eval bit for bit."""
    import copy
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import synth
    base = synth.c2(45, window=(400, 528, 0, 960))
    frames = []
    for draws, method in ((48, "ours"), (160, "ours"), (48, "zk"), (64, "ours"), (48, "ours")):
        sc = copy.deepcopy(base.scene)
        sc.draws, sc.method = draws, method
        frames.append(sc)
    hin = base.gbuf.pin()
    outs = pkg.glint_eval_host_batch(ctx, [hin] * len(frames), frames)
    dev = base.gbuf.to("cuda")
    for sc, o in zip(frames, outs):
        assert _same(o, pkg.glint_eval(ctx, dev, sc).cpu()), (sc.draws, sc.method)
