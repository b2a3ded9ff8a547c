"""Same-box A/B of relcp_step's internal body order on cfg5-relaxed:
lattice-ordered and relabelled input, reorder off / on.
    python tools/reorder_ab.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from gen import scenes  # noqa: E402
from paper_2506_14097_b200 import drivers, relcp as R  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
lit = scenes.cfg5()
pos, quat, _ = bench.relax_cfg5(lit, R, drivers)
base = scenes.with_state(lit, pos, quat, 55, "cfg5-relaxed")
cs = R.ConstraintStore(8 * lit["n"] + 4 * 1024 * 1024)
for name, sc in (("lattice", base), ("relabelled", scenes.relabelled(base, 99))):
    bodies = R.BodyState.from_scene(sc)
    init = {k: getattr(bodies, k).clone() for k in ("pos", "quat", "vel")}
    for ro in (R.REORDER_OFF, R.REORDER_AUTO, R.REORDER_ON, R.REORDER_OFF, R.REORDER_AUTO, R.REORDER_ON):
        ctx = R.Context(dynamics=sc["dynamics"], dt=sc["dt"], box=list(sc["box"]), cutoff=sc["cutoff"],
                        eps_ncp=sc["eps_ncp"], lcp_tol=1e-8, lcp_max_iter=200000, max_recursions=50, reorder=ro)
        ms, st, reps, _ = bench.time_steps(ctx, bodies, init, cs, steps, 3, None)
        it, roof = bench.roofline_of(st, reps, sc["n"], 6530.3, ms)
        print(f"{name:10s} reorder={ro} {it / (ms / 1e3):7.1f} it/s  step {ms / steps:7.2f} ms  iter "
              f"{roof['iter_ms'] * 1e3:6.1f} us (K6 {roof['scatter_ms'] * 1e3:6.1f}, K7 {roof['gather_ms'] * 1e3:6.1f})"
              f"  frac {roof['frac']:.3f}  iters {reps[-1]['iterations']}", flush=True)
        ctx.close()
