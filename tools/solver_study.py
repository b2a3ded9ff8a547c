"""LCP solver study: BB projected gradient vs
APGD with adaptive restart, iterations to tol 1e-8 per LCP of one ReLCP step
(cfg1, cfg2 recipe, cfg5 recipe) and for the cfg4 network.  JSON lines."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import scenes  # noqa: E402
from paper_2506_14097_b200 import relcp as R  # noqa: E402

cases = [("cfg1", lambda: scenes.cfg1(), 4), ("cfg2-20k", lambda: scenes.cfg2(), 4),
         ("cfg5-200k", lambda: scenes.cfg5(n=200_000), 2), ("cfg5", lambda: scenes.cfg5(), 2),
         ("cfg4", lambda: scenes.cfg4(), 0)]
sel = sys.argv[1:]
for name, mk, rec in cases:
    if sel and name not in sel:
        continue
    sc = mk()
    for solver in (0, 1, 2):
        ctx = R.Context(dynamics=sc["dynamics"], dt=sc["dt"], box=list(sc["box"]), lcp_tol=1e-8,
                        lcp_max_iter=30000, max_recursions=rec, solver=solver)
        bodies = R.BodyState.from_scene(sc)
        cs = R.ConstraintStore(12 * sc["n"] + 1024)
        torch.cuda.synchronize()
        t = time.time()
        if name == "cfg4":
            net = sc["network"]
            ctx.load_constraints(bodies, cs, net["ia"], net["ib"], net["n"], net["ra"], net["rb"], net["phi"])
            rep = ctx.solve_lcp(bodies, cs)
            out = dict(iterations=[rep["iterations"]], residuals=[rep["residual"]], n_c=[cs.count])
        else:
            rep = ctx.step(bodies, cs)
            out = {k: rep[k] for k in ("iterations", "residuals", "n_c", "recursions", "max_overlap")}
        torch.cuda.synchronize()
        out.update(config=name, solver=["BB", "APGD", "APGD_FUSED"][solver], seconds=time.time() - t)
        print(json.dumps(out), flush=True)
