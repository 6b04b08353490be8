"""Dev: production vs DEBUG instantiation vs oracle for the fuzz buffer, per light."""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle
import paper_2306_05051_b200 as pkg
from paper_2306_05051_b200 import synth
from test_gpu_parity import _fuzz_gbuffer
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
gb = _fuzz_gbuffer(32, 48, seed, [0.0, -0.0, 1e-40, -1e-40, 1e38, -1e38, 1e-30, 3.0e38],
                   [0.0, -0.0, 1e-40, -1e-40, 2.0 ** 60, -(2.0 ** 60), 1e-30, 1e9])
sc = synth.random_scene(seed, n_lights=3)
ctx = pkg.Context(0)
gd = gb.to("cuda")
prod = pkg.glint_eval(ctx, gd, sc).reshape(-1, 4).cpu().numpy()
dbg, rec = pkg.glint_eval(ctx, gd, sc, debug=True)
dbg = dbg.reshape(-1, 4).cpu().numpy()
rgb_o, fl_o, rec_o = oracle.eval(gb, sc, debug=True)
bad = np.argwhere(~(np.abs(prod[:, :3] - rgb_o) <= 1e-4 * np.abs(rgb_o) + 1e-30).all(1))[:, 0]
print("bad pixels", bad)
for i in bad[:4]:
    print(i, "prod", prod[i, :3], "dbg", dbg[i, :3], "orc", rgb_o[i])
    for l in range(3):
        sc1 = synth.SceneParams(**{**sc.__dict__}); sc1.lights = [sc.lights[l]]
        p1 = pkg.glint_eval(ctx, gd, sc1).reshape(-1, 4).cpu().numpy()[i, :3]
        o1 = oracle.eval(gb.take(torch.tensor([i])), sc1)[0][0]
        print("   light", l, "prod", p1, "orc", o1)
    # neighbours in the same warp: flags and activity
    w0 = (i // 32) * 32
    print("   warp flags", fl_o[w0:w0 + 32])
