"""Quick GPU probe: generate / solve / full step at a given config size."""
import sys, time, json
import numpy as np
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from gen import scenes
from paper_2506_14097_b200 import relcp as R

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
t0 = time.time()
sc = scenes.cfg5(n=n)
print("gen", time.time() - t0, flush=True)
ctx = R.Context(dynamics=sc["dynamics"], dt=sc["dt"], box=list(sc["box"]), lcp_max_iter=int(sys.argv[2]) if len(sys.argv) > 2 else 20000, max_recursions=int(sys.argv[3]) if len(sys.argv) > 3 else 2)
bodies = R.BodyState.from_scene(sc)
cs = R.ConstraintStore(24 * n)
torch.cuda.synchronize()
t = time.time(); n0, rc = ctx.generate_contacts(bodies, cs); torch.cuda.synchronize()
print("generate", time.time() - t, "n0", n0, "pairs", ctx.get_pairs()[0].numel(), "rc", rc, flush=True)
x = torch.rand(cs.count, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
ctx.prepare_operator(bodies, cs)
for _ in range(3): ctx.delassus_apply(bodies, cs, x, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): ctx.delassus_apply(bodies, cs, x, y)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
nc = cs.count
print("apply ms", ms, "alg GB/s", (176 * nc + 152 * n) / ms / 1e6, flush=True)
t = time.time(); rep = ctx.solve_lcp(bodies, cs); torch.cuda.synchronize()
dt = time.time() - t
print("solve", dt, rep, "it/s", rep["iterations"] / dt, flush=True)
bodies = R.BodyState.from_scene(sc)
t = time.time(); rep = ctx.step(bodies, cs); torch.cuda.synchronize()
print("step", time.time() - t, json.dumps(rep), flush=True)
