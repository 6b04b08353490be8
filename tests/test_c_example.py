"""The C ABI from plain C (examples/glint_c_example.c): compiled with gcc
against include/glint.h and libglint.so (no Python, no torch on the path),
run on the GPU; its radiance must equal the Python binding's for the same
C1 inputs. The compile step runs on CPU too (the ABI header is C-clean)."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _compile(out):
    from paper_2306_05051_b200 import build
    build.build()
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include", os.path.join(ROOT, "examples", "glint_c_example.c"),
           "-L", os.path.join(ROOT, "paper_2306_05051_b200"), "-lglint", "-L", "/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{os.path.join(ROOT, 'paper_2306_05051_b200')}", "-Wl,-rpath,/usr/local/cuda/lib64", "-lm",
           "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_c_example_compiles(tmp_path):
    _compile(str(tmp_path / "glint_c_example"))


@pytest.mark.gpu
def test_c_example_runs_and_matches_python(tmp_path):
    import torch
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import synth
    exe = str(tmp_path / "glint_c_example")
    _compile(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    m = re.search(r"glinting pixels (\d+) of 4096, radiance sum ([0-9.e+-]+), host entry identical 1, "
                  r"batch identical 1, aliased batch refused 1, bands identical 1, active pairs 4096", r.stdout)
    assert m, r.stdout
    fr = synth.c1("ggx", "mirror")
    ctx = pkg.Context(0)
    out = pkg.glint_eval(ctx, fr.gbuf.to("cuda"), fr.scene).cpu().numpy().reshape(-1, 4)
    ctx.close()
    assert int(m.group(1)) == int((out[:, 0] > 0).sum())
    assert abs(float(m.group(2)) - float(out[:, :3].astype(np.float64).sum())) <= 1e-6 * abs(float(m.group(2)))
