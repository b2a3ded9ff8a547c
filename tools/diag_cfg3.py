"""Diagnostic: cfg3 full step, per-generation statistics of the rows."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import scenes  # noqa: E402
from paper_2506_14097_b200 import relcp as R  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
for max_iter in (3000, 100000):
    sc = scenes.cfg3(n=n)
    ctx = R.Context(dynamics=sc["dynamics"], dt=sc["dt"], box=list(sc["box"]), lcp_tol=1e-8, lcp_max_iter=max_iter,
                    max_recursions=3)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(12 * n)
    rep = ctx.step(bodies, cs)
    m = cs.count
    out = dict(max_iter=max_iter, rep={k: rep[k] for k in ("recursions", "status", "n_c", "iterations", "residuals",
                                                           "max_overlap", "margin", "n_pairs")})
    gen = cs.gen[:m]
    for g in range(rep["recursions"] + 1):
        sel = gen == g
        out[f"gen{g}"] = dict(rows=int(sel.sum()), nz_max=float(cs.n[2, :m][sel].abs().max()) if sel.any() else 0,
                              phi_min=float(cs.phi[:m][sel].min()) if sel.any() else 0,
                              lam_max=float(cs.lam[:m][sel].max()) if sel.any() else 0)
    out["pos_z_max"] = float(bodies.pos[:, 2].abs().max())
    out["disp_max"] = float((bodies.pos - torch.as_tensor(sc["pos"], device="cuda")).norm(dim=1).max())
    print(json.dumps(out), flush=True)
