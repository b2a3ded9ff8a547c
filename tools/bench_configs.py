"""Per-config measurements (BASELINE configs 1-5 at full size) on one B200.

For each config: the ReLCP step (cfg1, cfg2, cfg3, cfg5; cfg4 is a given
network: load + LCP solve), the Delassus apply and the fused LCP iteration
timed with CUDA events, algorithmic GB/s (176 N_C + 152 N per apply,
216 N_C + 152 N per iteration).  One JSON line per config.

    python tools/bench_configs.py [cfg1 cfg2 ...]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import scenes  # noqa: E402
from paper_2506_14097_b200 import relcp as R  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0) \
    if os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")) else 6650.0


def ev():
    return torch.cuda.Event(enable_timing=True)


def time_apply(ctx, bodies, cs, n, reps=20):
    ctx.prepare_operator(bodies, cs)
    nc = cs.count
    x = torch.rand(max(nc, 1), dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        ctx.delassus_apply(bodies, cs, x, y)
    a, b = ev(), ev()
    a.record()
    for _ in range(reps):
        ctx.delassus_apply(bodies, cs, x, y)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    byt = 176.0 * nc + 152.0 * n
    return dict(n_c=nc, ms=ms, GBps=byt / ms / 1e6, frac_measured=byt / ms / 1e6 / PEAK)


def run(name):
    t0 = time.time()
    if name == "cfg1":
        sc = scenes.cfg1()
    elif name == "cfg2":
        sc = scenes.cfg2()
    elif name == "cfg3":
        sc = scenes.cfg3()
    elif name == "cfg4":
        sc = scenes.cfg4()
    elif name == "cfg4-6M":
        sc = scenes.cfg4(c_fixed=3)
    else:
        sc = scenes.cfg5()
    gen_s = time.time() - t0
    n = sc["n"]
    ctx = R.Context(dynamics=sc["dynamics"], dt=sc["dt"], box=list(sc["box"]), cutoff=sc["cutoff"],
                    eps_ncp=sc["eps_ncp"], lcp_tol=1e-8, lcp_max_iter=3000, max_recursions=2 if name == "cfg5" else 50,
                    layout=int(os.environ.get("RELCP_LAYOUT", "2")))
    bodies = R.BodyState.from_scene(sc)
    init = {k: getattr(bodies, k).clone() for k in ("pos", "quat", "vel")}
    out = dict(config=name, n_bodies=n, gen_s=gen_s, layout=int(os.environ.get("RELCP_LAYOUT", "2")))
    if name.startswith("cfg4"):
        net = sc["network"]
        cs = R.ConstraintStore(len(net["ia"]) + 16)
        ctx.load_constraints(bodies, cs, net["ia"], net["ib"], net["n"], net["ra"], net["rb"], net["phi"])
        ctx.set_params(lcp_max_iter=20000)
        ctx.set_timing(True)
        ctx.reset_stats()
        a, b = ev(), ev()
        a.record()
        rep = ctx.solve_lcp(bodies, cs)
        b.record()
        torch.cuda.synchronize()
        st = ctx.stats()
        ms = a.elapsed_time(b)
        it = st["iter_timed"]
        it_ms = st["iter_ms"] / max(1, it)
        nc = cs.count
        out.update(n_c=nc, lcp=dict(iterations=rep["iterations"], residual=rep["residual"],
                                    converged=rep["converged"], solve_ms=ms,
                                    it_per_s=rep["iterations"] / (ms / 1e3)),
                   iteration=dict(ms=it_ms, GBps=(216.0 * nc + 152.0 * n) / it_ms / 1e6,
                                  frac_measured=(216.0 * nc + 152.0 * n) / it_ms / 1e6 / PEAK))
        out["apply"] = time_apply(ctx, bodies, cs, n)
        return out
    cs = R.ConstraintStore(12 * n + 1024)
    rep = ctx.step(bodies, cs)  # warm-up
    for k, v in init.items():
        getattr(bodies, k).copy_(v)
    # step time without per-iteration events (LCP batches replayed as CUDA graphs)
    a, b = ev(), ev()
    a.record()
    ctx.step(bodies, cs)
    b.record()
    torch.cuda.synchronize()
    out["step_ms_graphs"] = a.elapsed_time(b)
    for k, v in init.items():
        getattr(bodies, k).copy_(v)
    ctx.reset_stats()
    ctx.set_timing(True)
    a, b = ev(), ev()
    a.record()
    rep = ctx.step(bodies, cs)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    st = ctx.stats()
    iters = sum(rep["iterations"])
    it_bytes = sum(i * (216.0 * c + 152.0 * n) for c, i in zip(rep["n_c"], rep["iterations"]))
    # bytes per iteration averaged over the step / time per timed iteration
    it_ms = st["iter_ms"] / max(1, st["iter_timed"]) * iters
    out.update(step_ms=ms, recursions=rep["recursions"], status=rep["status"], n_c=rep["n_c"],
               lcp_iters=rep["iterations"], residuals=rep["residuals"], max_overlap=rep["max_overlap"],
               n_pairs=rep["n_pairs"], ms_generate=rep["ms_generate"], ms_solve=rep["ms_solve"],
               ms_check=rep["ms_check"], it_per_s_step=iters / (ms / 1e3),
               iteration=dict(ms=st["iter_ms"] / max(1, st["iter_timed"]),
                              GBps=it_bytes / it_ms / 1e6 if it_ms > 0 else None,
                              frac_measured=it_bytes / it_ms / 1e6 / PEAK if it_ms > 0 else None),
               gpu_launches=st["launches"])
    for k, v in init.items():
        getattr(bodies, k).copy_(v)
    out["apply"] = time_apply(ctx, bodies, cs, n)  # on the step's final store, W at C^k
    return out


if __name__ == "__main__":
    names = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]
    for nm in names:
        print(json.dumps(run(nm)), flush=True)
