"""BB iterations and step time vs the power-iteration count (alpha_0 = 1/L,
R1) on cfg5-relaxed and cfg2.   python tools/power_ab.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from gen import scenes  # noqa: E402
from paper_2506_14097_b200 import drivers, relcp as R  # noqa: E402

lit = scenes.cfg5()
pos, quat, _ = bench.relax_cfg5(lit, R, drivers)
sc = scenes.with_state(lit, pos, quat, 55, "cfg5-relaxed")
cs = R.ConstraintStore(8 * lit["n"] + 4 * 1024 * 1024)
bodies = R.BodyState.from_scene(sc)
init = {k: getattr(bodies, k).clone() for k in ("pos", "quat", "vel")}
for pw in (20, 8, 4, 2, 20):
    ctx = R.Context(dynamics=sc["dynamics"], dt=sc["dt"], box=list(sc["box"]), cutoff=sc["cutoff"],
                    eps_ncp=sc["eps_ncp"], lcp_tol=1e-8, lcp_max_iter=200000, max_recursions=50, power_iters=pw)
    ms, st, reps, _ = bench.time_steps(ctx, bodies, init, cs, 3, 3, None)
    it = sum(sum(r["iterations"]) for r in reps)
    r = reps[-1]
    print(f"cfg5-relaxed power_iters={pw:2d}: {it / (ms / 1e3):7.1f} it/s  step {ms / 3:7.2f} ms  iters {r['iterations']} "
          f"solve {r['ms_solve']:.1f} ms  status {r['status']}", flush=True)
    ctx.close()
sc2 = scenes.cfg2()
b2 = R.BodyState.from_scene(sc2)
for pw in (20, 8, 4, 2):
    ctx = R.Context(dynamics=sc2["dynamics"], dt=sc2["dt"], box=list(sc2["box"]), cutoff=sc2["cutoff"],
                    eps_ncp=sc2["eps_ncp"], lcp_tol=1e-8, lcp_max_iter=30000, power_iters=pw)
    cs2 = R.ConstraintStore(8 * sc2["n"])
    ctx.generate_contacts(b2, cs2)
    rep = ctx.solve_lcp(b2, cs2)
    print(f"cfg2 A_0 power_iters={pw:2d}: {rep['iterations']} iterations, residual {rep['residual']:.2e}", flush=True)
    ctx.close()
