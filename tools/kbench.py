"""Kernel micro-bench / ncu target: cfg5 A_0 at N bodies; a few Delassus
applies then a capped LCP solve.  python tools/kbench.py [N] [iters] [final|relaxed]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import scenes  # noqa: E402
from paper_2506_14097_b200 import relcp as R  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
sc = scenes.cfg5(n=n)
if len(sys.argv) > 3 and sys.argv[3] == "relaxed":
    # the bench headline's store: cfg5 relaxed by the library (drivers.relax), A_0 at that state
    from paper_2506_14097_b200 import drivers  # noqa: E402
    pos, quat, _ = drivers.relax(sc, max_recursions=0, lcp_max_iter=20000, max_steps=60)
    sc = scenes.with_state(sc, pos.cpu().numpy(), quat.cpu().numpy(), 55, "cfg5-relaxed")
ctx = R.Context(dynamics=sc["dynamics"], dt=sc["dt"], box=list(sc["box"]), lcp_max_iter=iters, lcp_tol=1e-30,
                solver=int(os.environ.get("RELCP_SOLVER", "0")),
                layout=int(os.environ.get("RELCP_LAYOUT", "2")),
                k6_pipe=int(os.environ.get("RELCP_K6PIPE", "0")),
                k6_bpw=int(os.environ.get("RELCP_K6_BPW", "0")))  # 20 power iterations: APGD steps 1/(1.1 L)
bodies = R.BodyState.from_scene(sc)
cs = R.ConstraintStore(8 * n)
ctx.generate_contacts(bodies, cs)
torch.cuda.synchronize()
t = time.time()
ctx.generate_contacts(bodies, cs)
print(f"generate_contacts {1e3 * (time.time() - t):.1f} ms (pairs {ctx.get_pairs()[0].numel()}, rows {cs.count})",
      flush=True)
if len(sys.argv) > 3 and sys.argv[3] == "final":
    # the step's final (largest, augmented) store; W at the step's C^k
    init = {k: getattr(bodies, k).clone() for k in ("pos", "quat", "vel")}
    ctx.set_params(max_recursions=2, lcp_max_iter=3000, lcp_tol=1e-8)
    ctx.step(bodies, cs)
    for k, v in init.items():
        getattr(bodies, k).copy_(v)
    ctx.set_params(lcp_max_iter=iters, lcp_tol=1e-30)
    cs.lam.zero_()
ctx.prepare_operator(bodies, cs)
nc = cs.count
x = torch.rand(nc, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    ctx.delassus_apply(bodies, cs, x, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
prof_apply = os.environ.get("KBENCH_PROFILE_APPLY") == "1"  # ncu --profile-from-start off: only these applies
if prof_apply:
    torch.cuda.profiler.start()
e0.record()
for _ in range(20):
    ctx.delassus_apply(bodies, cs, x, y)
e1.record()
torch.cuda.synchronize()
if prof_apply:
    torch.cuda.profiler.stop()
ms = e0.elapsed_time(e1) / 20
print(f"N={n} N_C={nc} apply {ms:.4f} ms  alg {(176 * nc + 152 * n) / ms / 1e6:.0f} GB/s", flush=True)
ctx.set_timing(True)
prof = os.environ.get("KBENCH_PROFILE_SOLVE") == "1"  # ncu --profile-from-start off: only this solve
if prof:
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
t = time.time()
rep = ctx.solve_lcp(bodies, cs)
if prof:
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
st = ctx.stats()
it, sp = max(1, st["iter_timed"]), max(1, st["split_timed"])
print(f"solve {rep['iterations']} it in {time.time() - t:.3f}s; scatter {st['scatter_ms'] / sp:.4f} ms "
      f"gather {st['gather_ms'] / sp:.4f} ms (first batch); iter {st['iter_ms'] / it:.4f} ms over {it}; iter alg "
      f"{(216 * nc + 152 * n) / (st['iter_ms'] / it) / 1e6:.0f} GB/s; K6 alg "
      f"{(96 * nc + 104 * n) / (st['scatter_ms'] / sp) / 1e6:.0f} GB/s; layout {st['op_layout']} "
      f"jds_solves {st['jds_solves']} resid {rep['residual']:.3e}", flush=True)
