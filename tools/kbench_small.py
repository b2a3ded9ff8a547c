"""Small-store LCP iteration micro-bench / ncu target: cfg2 (20k bodies) or
cfg3 (200k) A_0, a capped BB solve.  python tools/kbench_small.py [cfg2|cfg3] [iters]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import scenes  # noqa: E402
from paper_2506_14097_b200 import relcp as R  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
sc = scenes.cfg2() if name == "cfg2" else scenes.cfg3()
ctx = R.Context(dynamics=sc["dynamics"], dt=sc["dt"], box=list(sc["box"]), cutoff=sc["cutoff"], lcp_max_iter=iters,
                lcp_tol=1e-30)
bodies = R.BodyState.from_scene(sc)
cs = R.ConstraintStore(8 * sc["n"])
ctx.generate_contacts(bodies, cs)
ctx.set_timing(True)
for rep in range(2):
    ctx.reset_stats()
    r = ctx.solve_lcp(bodies, cs)
    st = ctx.stats()
    it, sp = max(1, st["iter_timed"]), max(1, st["split_timed"])
    print(f"{name} N={sc['n']} N_C={cs.count} iters {r['iterations']} iter {1e3 * st['iter_ms'] / it:.2f} us "
          f"(first batch: K6 {1e3 * st['scatter_ms'] / sp:.2f} us, K7 {1e3 * st['gather_ms'] / sp:.2f} us)", flush=True)
