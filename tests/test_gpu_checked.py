"""A checked build (-DGLINT_CHECKED: device asserts on every computed index,
the stand-in for compute-sanitizer, which this pool does not offer) runs the
TMA ring, pitched views, debug records, all eval modes, the host pipeline and
the two batch entries (chained launches, cross-frame host pipeline)
on representative inputs without tripping an assert, and gives exactly the
production library's bits."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_matches_production(tmp_path):
    from paper_2306_05051_b200 import build
    build.build()
    checked = build.build(force=True, out=os.path.join(ROOT, "paper_2306_05051_b200", "libglint_checked.so"),
                          defines=("GLINT_CHECKED",))
    runs = {}
    for name, lib in (("prod", build.LIB), ("checked", checked)):
        out = str(tmp_path / f"{name}.npz")
        env = dict(os.environ, GLINT_LIB=lib, PYTHONPATH=ROOT)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "checked_run.py"), out], env=env,
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0 and "checked run ok" in r.stdout, (name, r.stdout[-2000:], r.stderr[-4000:])
        runs[name] = np.load(out)
    a, b = runs["prod"], runs["checked"]
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32)), k
