"""The paper's colony experiment, scaled by the
generation count: one spherocylinder (b = 0.5, tip-to-tip l_0 = 2) grows
l_dot = l and divides at 2 l_0 (drivers.colony, R22, R28) for `gens`
doublings (the paper: 17, 131,072 cells).  One JSON line per step with the
body count, divisions, rows, recursions, max overlap and wall time.

    python tools/colony_run.py [gens] [dt]
"""
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_14097_b200 import drivers as D  # noqa: E402

gens = int(sys.argv[1]) if len(sys.argv) > 1 else 12
dt = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-2
r, l0 = 0.25, 2.0
sc = dict(name="colony-1", n=1, pos=np.zeros((1, 3)), quat=np.array([[1.0, 0, 0, 0]]),
          axes=np.array([[0.5 * l0 - r, r, r]]), shape=np.ones(1, np.int32), vel=np.zeros((1, 6)),
          inv_mass=np.ones(1), inv_inertia=np.ones((1, 3)), kinematic=np.zeros(1, np.int32), box=np.zeros(3),
          dt=dt, dynamics=1, xi=1.0, cutoff=0.1, eps_ncp=1e-5, lcp_tol=1e-8)
steps = int(math.ceil(gens * math.log(2.0) / dt)) + 2
t = [time.time()]


def cb(k, bodies, cs, rep):
    torch.cuda.synchronize()
    now = time.time()
    print(json.dumps(dict(run="colony", step=k, n_bodies=rep["n_bodies"], divisions=rep["divisions"],
                          n_c=rep["n_c"][-1], recursions=rep["recursions"], status=rep["status"],
                          lcp_iters=sum(rep["iterations"]), max_overlap=rep["max_overlap"],
                          seconds=now - t[0])), flush=True)
    t[0] = now


D.colony(sc, steps=steps, l0=l0, callback=cb, lcp_max_iter=20000, max_recursions=50)
