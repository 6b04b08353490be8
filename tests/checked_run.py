"""Subprocess body of tests/test_gpu_checked.py: evaluates a fixed set of
inputs with the library named by GLINT_LIB and saves the outputs (npz)."""
import sys

import numpy as np
import torch

import paper_2306_05051_b200 as pkg
from paper_2306_05051_b200 import synth


def cases():
    out = [("c1", synth.c1("ggx", "mirror")), ("c1b", synth.c1("beckmann", "az90"))]
    for e in (5, 25, 65, 90):
        out.append((f"c2_{e}", synth.c2(e, window=(380, 508, 0, 1920))))
    out.append(("c3", synth.c3(window=(900, 1028, 1700, 1956))))
    out.append(("c4", synth.c4(3, window=(1000, 1064, 1800, 1928))))
    out.append(("rand", synth.Frame("rand", synth.random_gbuffer(67, 129, seed=5), synth.random_scene(5, n_lights=6))))
    return out


def main(path):
    ctx = pkg.Context(0)
    res = {}
    for name, fr in cases():
        gd = fr.gbuf.to("cuda")
        for d, m in ((48, "ours"), (64, "ours"), (160, "ours"), (48, "zk")):
            fr.scene.draws, fr.scene.method = d, m
            res[f"{name}_{m}{d}"] = pkg.glint_eval(ctx, gd, fr.scene).cpu().numpy()
        fr.scene.draws, fr.scene.method = 48, "ours"
        view = synth.GBuffer(*[p[:, 1:] for p in gd.planes()])           # pitched: no TMA
        res[f"{name}_pitched"] = pkg.glint_eval(ctx, view, fr.scene).cpu().numpy()
        _, rec = pkg.glint_eval(ctx, gd, fr.scene, debug=True)
        res[f"{name}_count"] = np.ascontiguousarray(rec["count"])
        res[f"{name}_host"] = pkg.glint_eval_host(ctx, fr.gbuf.pin(), fr.scene).numpy()
    # the batch entries: all cases chained in one glint_eval_batch (PDL
    # launches), and through one glint_eval_host_batch pipeline
    frs = cases()
    outs = pkg.glint_eval_batch(ctx, [fr.gbuf.to("cuda") for _, fr in frs], [fr.scene for _, fr in frs])
    for (name, _), o in zip(frs, outs):
        res[f"{name}_batch"] = o.cpu().numpy()
    houts = pkg.glint_eval_host_batch(ctx, [fr.gbuf.pin() for _, fr in frs], [fr.scene for _, fr in frs])
    for (name, _), o in zip(frs, houts):
        res[f"{name}_hostbatch"] = o.numpy()
    torch.cuda.synchronize()
    ctx.close()
    np.savez(path, **res)
    print("checked run ok", len(res))


if __name__ == "__main__":
    main(sys.argv[1])
