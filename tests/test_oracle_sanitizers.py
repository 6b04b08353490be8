"""The CPU oracle under AddressSanitizer + UndefinedBehaviorSanitizer (VERDICT
r1, section 5 aux items): a driver built with -fsanitize=address,undefined
and -fno-sanitize-recover runs the oracle on stress, edge-case and workload
inputs in every eval mode; it must exit cleanly (any out-of-bounds access,
signed overflow, bad shift or misaligned load aborts it) and reproduce the
uninstrumented build's output bit for bit."""
import os
import shutil
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


@pytest.fixture(scope="module")
def driver(tmp_path_factory):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    out = str(tmp_path_factory.mktemp("asan") / "oracle_asan")
    cmd = ["gcc", "-O1", "-g", "-std=c11", "-D_GNU_SOURCE", "-ffp-contract=off", "-fno-fast-math",
           "-fno-tree-vectorize", "-fsanitize=address,undefined", "-fno-sanitize-recover=all",
           "-fno-omit-frame-pointer", "-o", out, os.path.join(HERE, "oracle_asan_main.c"),
           os.path.join(ROOT, "oracle", "glint_oracle.c"), "-lm"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        pytest.skip("sanitizer runtime unavailable: " + r.stderr[-300:])
    return out


def _run(driver, tmp_path, gb, scene):
    import oracle
    planes = oracle._planes(gb)
    n = planes[0].shape[0]
    sc = oracle.scene_struct(scene)
    inp, outp = str(tmp_path / "in.bin"), str(tmp_path / "out.bin")
    with open(inp, "wb") as f:
        f.write(np.int64(n).tobytes())
        f.write(bytes(sc))
        for p in planes:
            f.write(np.ascontiguousarray(p, np.float32).tobytes())
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=1", UBSAN_OPTIONS="print_stacktrace=1")
    r = subprocess.run([driver, inp, outp], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "runtime error" not in r.stderr and "ERROR: AddressSanitizer" not in r.stderr, r.stderr[-3000:]
    raw = open(outp, "rb").read()
    rgb = np.frombuffer(raw[:24 * n], np.float64).reshape(n, 3)
    fl = np.frombuffer(raw[24 * n:28 * n], np.uint32)
    rec = None
    if sc.eval_mode == 0 and sc.n_lights:
        rec = np.frombuffer(raw[28 * n:], oracle.REC_DTYPE).reshape(n, sc.n_lights)
    return rgb, fl, rec


def test_oracle_is_clean_under_asan_ubsan(driver, tmp_path):
    import oracle
    from paper_2306_05051_b200 import synth
    cases = [(synth.random_gbuffer(13, 17, seed=3), synth.random_scene(3, n_lights=3)),
             (synth.random_gbuffer(7, 9, seed=5), synth.random_scene(5, n_lights=16, ndf="beckmann")),
             (synth.c1("ggx", "az90").gbuf, synth.c1("ggx", "az90").scene),
             (synth.c2(5, window=(400, 416, 900, 964)).gbuf, synth.c2(5).scene)]
    # extreme inputs (R-27b, R-30b, R-37): huge / tiny / non-finite components
    gb = synth.random_gbuffer(8, 12, seed=9)
    rng = np.random.default_rng(9)
    planes = [p.clone() for p in gb.planes()]
    for i in range(8 * 12):
        k, c = int(rng.integers(0, 5)), int(rng.integers(0, 4))
        if k == 1 and c >= 2:
            c = 0
        planes[k].view(-1, 4)[i, c] = float(rng.choice([0.0, -0.0, 1e-40, 3e38, -1e38, float("nan"), float("inf")]))
    cases.append((synth.GBuffer(*planes), synth.random_scene(9, n_lights=2)))
    for gb, sc in cases:
        for method, draws in (("ours", 48), ("ours", 64), ("ours", 160), ("zk", 48)):
            sc.method, sc.draws = method, draws
            rgb, fl, rec = _run(driver, tmp_path, gb, sc)
            rgb_o, fl_o, rec_o = oracle.eval(gb, sc, debug=(method, draws) == ("ours", 48))
            assert np.array_equal(fl, fl_o)
            assert np.array_equal(rgb.view(np.uint64), rgb_o.view(np.uint64)) or \
                np.array_equal(np.isnan(rgb), np.isnan(rgb_o)) and np.allclose(rgb, rgb_o, rtol=0, atol=0, equal_nan=True)
            if rec is not None:
                assert np.array_equal(rec.view(np.uint8), rec_o.view(np.uint8))
        sc.method, sc.draws = "ours", 48
