"""Dev: print the inputs of pixels where the kernel and the oracle disagree on
the finite-extremes fuzz buffer of tests/test_gpu_parity.py."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
import paper_2306_05051_b200 as pkg
from paper_2306_05051_b200 import synth
sys.path.insert(0, "tests")
from test_gpu_parity import _fuzz_gbuffer
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
gb = _fuzz_gbuffer(32, 48, seed, [0.0, -0.0, 1e-40, -1e-40, 1e38, -1e38, 1e-30, 3.0e38])
sc = synth.random_scene(seed, n_lights=3)
ctx = pkg.Context(0)
out = pkg.glint_eval(ctx, gb.to("cuda"), sc).reshape(-1, 4).cpu().numpy()
o2, rec = pkg.glint_eval(ctx, gb.to("cuda"), sc, debug=True)
rgb_o, fl_o, rec_o = oracle.eval(gb, sc, debug=True)
err = np.abs(out[:, :3] - rgb_o)
bad = ~(err <= 1e-4 * np.abs(rgb_o) + 1e-30)
for i in np.argwhere(bad.any(1))[:, 0][:6]:
    print("pixel", i, "gpu", out[i], "oracle", rgb_o[i], fl_o[i])
    for name, p in zip(("duv", "uvm", "nrm", "pos", "mat"), gb.planes()):
        print("  ", name, p.view(-1, 4)[i].tolist())
    for l in range(3):
        a, b = rec[i, l], rec_o[i, l]
        print("   light", l, "C gpu/orc", a["C"], b["C"], "Dp", a["Dp"], b["Dp"], "p", a["p"], b["p"], "active", a["light_active"])
