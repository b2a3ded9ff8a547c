"""Probe: overdamped GPU relaxation of the cfg5 recipe (drivers.relax), then
one inertial ReLCP step from the relaxed state with fresh N(0,1) velocities.

    python tools/relax_probe.py [n] [relax_max_rec] [relax_lcp_max_iter]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import scenes  # noqa: E402
from paper_2506_14097_b200 import drivers, relcp as R  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
rec = int(sys.argv[2]) if len(sys.argv) > 2 else 50
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 20000
sc = scenes.cfg5(n=n)
t0 = time.perf_counter()


def cb(k, b, cs, rep):
    torch.cuda.synchronize()
    print(json.dumps(dict(step=k, t=time.perf_counter() - t0, rec=rep["recursions"], status=rep["status"],
                          n_c=rep["n_c"], iters=rep["iterations"], res=rep["residuals"],
                          max_overlap=rep["max_overlap"])), flush=True)


pos, quat, reps = drivers.relax(sc, max_recursions=rec, lcp_max_iter=cap, callback=cb)
print("relax_s", time.perf_counter() - t0, flush=True)
rng = np.random.Generator(np.random.PCG64(55))
vel = rng.standard_normal((n, 6))
s2 = dict(sc)
s2.update(pos=pos.cpu().numpy(), quat=quat.cpu().numpy(), vel=vel)
for solver in (0, 2):
    ctx = R.Context(dynamics=0, dt=1e-3, box=list(sc["box"]), cutoff=0.1, eps_ncp=1e-5, lcp_tol=1e-8,
                    lcp_max_iter=200000, max_recursions=50, solver=solver)
    for rep_i in range(2):
        bodies = R.BodyState.from_scene(s2)
        cs = R.ConstraintStore(16 * n + 1024)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        rep = ctx.step(bodies, cs)
        torch.cuda.synchronize()
        print(json.dumps(dict(solver=solver, wall_s=time.perf_counter() - t1, **{k: rep[k] for k in (
            "recursions", "status", "n_c", "iterations", "residuals", "max_overlap", "ms_generate", "ms_solve",
            "ms_check", "snsd_nonconv", "n_pairs")})), flush=True)
