"""Host-time breakdown of one cfg5 bench step by phase (debug build with
-DRELCP_PHASE_TIMING: every mark synchronises, so the phases add up to a
slightly slower step than bench.py's).  Build here (no GPU needed):
    python tools/phases.py --build
then on the B200:
    RELCP_LIB=paper_2506_14097_b200/lib/librelcp_phases.so python tools/phases.py [N] [relaxed]
("relaxed": the bench headline's cfg5-relaxed state and parameters)
Prints the phase marks of the last of three steps, then a summary per phase."""
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2506_14097_b200", "lib",
                   "librelcp_phases.so")

if "--build" in sys.argv:
    from paper_2506_14097_b200 import build
    print(build.build(defines=("RELCP_PHASE_TIMING",), out=OUT))
    sys.exit(0)

import torch  # noqa: E402

from gen import scenes  # noqa: E402
from paper_2506_14097_b200 import relcp as R  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
sc = scenes.cfg5(n=n)
relaxed = len(sys.argv) > 2 and sys.argv[2] == "relaxed"
if relaxed:
    from paper_2506_14097_b200 import drivers  # noqa: E402
    import numpy as np  # noqa: E402
    pos, quat, _ = drivers.relax(sc, max_recursions=0, lcp_max_iter=20000, max_steps=60)
    sc = scenes.with_state(sc, pos.cpu().numpy(), quat.cpu().numpy(), 55, "cfg5-relaxed")
ctx = R.Context(dynamics=sc["dynamics"], dt=sc["dt"], box=list(sc["box"]), cutoff=sc["cutoff"], eps_ncp=sc["eps_ncp"],
                max_recursions=50 if relaxed else 2, lcp_max_iter=200000 if relaxed else 3000,
                lcp_tol=1e-8)  # bench.py's parameters (headline / literal line)
bodies = R.BodyState.from_scene(sc)
cs = R.ConstraintStore(8 * n)
init = {k: getattr(bodies, k).clone() for k in ("pos", "quat", "vel")}
log = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "phases.log")
for k in range(3):
    for key, v in init.items():
        getattr(bodies, key).copy_(v)
    cs.count = 0
    torch.cuda.synchronize()
    if k == 2:
        sys.stderr.flush()
        fd = os.open(log, os.O_WRONLY | os.O_CREAT | os.O_TRUNC)
        saved = os.dup(2)
        os.dup2(fd, 2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep = ctx.step(bodies, cs)
    e1.record()
    torch.cuda.synchronize()
    if k == 2:
        os.dup2(saved, 2)
        os.close(fd)
    print(f"step {k}: {e0.elapsed_time(e1):.1f} ms, iterations {rep['iterations']}", flush=True)
tot = {}
for line in open(log):
    m = re.match(r"\[phase\] (\S+)\s+([0-9.]+) ms", line)
    if m:
        tot[m.group(1)] = tot.get(m.group(1), 0.0) + float(m.group(2))
print(open(log).read())
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k:24s} {v:9.2f} ms")
