"""Small-store LCP iteration micro-bench / ncu target: cfg2 (20k bodies) or
cfg3 (200k) or cfg1 (512) A_0, a capped BB solve.
    RELCP_CLUSTER=0|1 python tools/kbench_small.py [cfg1|cfg2|cfg3] [iters]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import scenes  # noqa: E402
from paper_2506_14097_b200 import relcp as R  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
sc = {"cfg1": scenes.cfg1, "cfg2": scenes.cfg2, "cfg3": scenes.cfg3}[name]()
ctx = R.Context(dynamics=sc["dynamics"], dt=sc["dt"], box=list(sc["box"]), cutoff=sc["cutoff"], lcp_max_iter=iters,
                lcp_tol=1e-30, cluster=int(os.environ.get("RELCP_CLUSTER", "1")),
                k6_bpw=int(os.environ.get("RELCP_K6_BPW", "0")))
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
          f"(first batch: K6 {1e3 * st['scatter_ms'] / sp:.2f} us, K7 {1e3 * st['gather_ms'] / sp:.2f} us) "
          f"cluster_solves {st['cluster_solves']} resid {r['residual']:.3e}", flush=True)
