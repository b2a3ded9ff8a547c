"""Full-size multi-step runs: the cfg2 compaction
(20,000 ellipsoids, phi 0.40 -> 0.55) and the cfg3 growth (200,000 planar
ellipsoids), one JSON line per step: N_C per recursion, LCP iterations, max
overlap after the step, status, wall time.  Solver: fused APGD (robust on
augmented LCPs).

    python tools/run_drivers.py [cfg2_steps] [cfg3_steps] [colony_steps]

The colony run: 2^17 spherocylinders growing
l_dot = l and dividing at 2 l_0 (drivers.colony, R22, R28), dt = 1e-3 (at
1e-2 the first step's trial configuration drives rows of rods, compressed by
the start-of-step growth, through each other: intersecting centrelines are
undefined, R22).
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import scenes  # noqa: E402
from paper_2506_14097_b200 import drivers as D  # noqa: E402

n2 = int(sys.argv[1]) if len(sys.argv) > 1 else 200
n3 = int(sys.argv[2]) if len(sys.argv) > 2 else 10
n4 = int(sys.argv[3]) if len(sys.argv) > 3 else 0
kw = dict(lcp_tol=1e-8, lcp_max_iter=20000, max_recursions=20, solver=2)
t_last = [time.time()]


def log(name):
    def cb(k, bodies, cs, rep):
        torch.cuda.synchronize()
        t = time.time()
        print(json.dumps(dict(run=name, step=k, n_c=rep["n_c"], iterations=rep["iterations"],
                              recursions=rep["recursions"], status=rep["status"], max_overlap=rep["max_overlap"],
                              phi=rep.get("phi"), box=rep.get("box"), n_bodies=rep.get("n_bodies"),
                              divisions=rep.get("divisions"), seconds=t - t_last[0])), flush=True)
        t_last[0] = t
    return cb


if n2 > 0:
    D.compaction(scenes.cfg2(), steps=200, phi_end=0.55, stop_after=n2, callback=log("cfg2"), **kw)
if n3 > 0:
    t_last[0] = time.time()
    D.growth(scenes.cfg3(), steps=n3, callback=log("cfg3"), **kw)
if n4 > 0:
    t_last[0] = time.time()
    D.colony(scenes.colony_rods(dt=1e-3), steps=n4, callback=log("colony"), **kw)
