"""Dev: per-light diagnosis of the scene-fuzz radiance mismatch."""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle
import paper_2306_05051_b200 as pkg
from paper_2306_05051_b200 import synth
import test_gpu_parity as T
seed = int(sys.argv[1])
# rebuild the scene exactly as the test does
src = open("tests/test_gpu_parity.py").read()
body = src.split("def test_fuzz_scene_parameters(ctx, seed):")[1].split("    import oracle\n")[0]
body = "\n".join(l[4:] for l in body.split("\n") if not l.strip().startswith('"""') and "tolerance where" not in l
                 and "8, max ratio" not in l and "1e36, directional" not in l and "(fp32 overflow" not in l)
ns = {"np": np, "synth": synth, "seed": seed}
exec(body, ns)
gb, sc = ns["gb"], ns["sc"]
ctx = pkg.Context(0)
prod = pkg.glint_eval(ctx, gb.to("cuda"), sc).reshape(-1, 4).cpu().numpy()
rgb_o, fl_o, rec_o = oracle.eval(gb, sc, debug=True)
mask = T.well_conditioned(gb, sc)
bad = np.argwhere(~(np.abs(prod[:, :3] - rgb_o) <= 1e-4 * np.abs(rgb_o) + 1e-30).all(1) & mask)[:, 0]
print("bad", bad, "beta", sc.beta, "K", sc.max_ratio_level, sc.ndf)
for i in bad[:3]:
    print(i, prod[i, :3], rgb_o[i], [p.view(-1, 4)[i].tolist() for p in gb.planes()])
    for l, lt in enumerate(sc.lights):
        sc1 = synth.SceneParams(**{**sc.__dict__}); sc1.lights = [lt]
        p1 = pkg.glint_eval(ctx, gb.to("cuda"), sc1).reshape(-1, 4).cpu().numpy()[i, :3]
        o1 = oracle.eval(gb.take(torch.tensor([i])), sc1, debug=True)
        print("  light", l, lt.kind, "I", lt.intensity[0], "prod", p1, "orc", o1[0][0], "C", o1[2][0, 0]["C"], "p", o1[2][0, 0]["p"])
