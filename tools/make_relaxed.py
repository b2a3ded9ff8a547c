"""Write tests/golden/cfg1_relaxed.txt: the overlap-free companion of BASELINE
cfg1 (SURVEY.md §8(d) "cfg1-relaxed").

The literal cfg1 start overlaps (about 215 of its ~420 near pairs, min Phi
about -0.5).  The paper's theory assumes an overlap-free start (P:L869,
P:L881), so the Cor. 4 pin (small dt -> zero augmentations) needs
a relaxed state.  This script makes it with the ORACLE only: overdamped ReLCP
steps (Algorithm 1, overdamped form P:L512-522, local drag
P:L928-944) with zero velocity and no external force, until a full candidate
scan at the accepted state finds min Phi >= -eps_NCP.  It calls only
`oracle/` and `gen/`; nothing here comes from the CUDA path.

    python tools/make_relaxed.py            # writes the fixture
    python tools/make_relaxed.py --check    # regenerate and compare bitwise
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from gen import scenes  # noqa: E402
from oracle import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "cfg1_relaxed.txt")


def min_phi(sc) -> float:
    """min Phi over every pair the broadphase finds within the cutoff."""
    rad = oracle.bounding_radius(sc["axes"])
    pi, pj = oracle.broadphase(sc["pos"], rad, sc["box"], sc["cutoff"])
    phi, *_ = oracle.snsd(sc["pos"], sc["quat"], sc["axes"], sc["box"], pi, pj)
    return float(np.min(phi)) if len(phi) else np.inf


def relax(sc, dt: float = 1e-2, max_steps: int = 20):
    s = dict(sc)
    s.update(dynamics=scenes.OVERDAMPED, dt=dt, vel=np.zeros_like(sc["vel"]))
    for k in range(max_steps):
        r = oracle.relcp_step(s, max_recursions=50, lcp_tol=1e-10)
        s["pos"], s["quat"] = r["pos"], r["quat"]
        m = min_phi(s)
        print(f"step {k}: recursions {r['recursions']} n_c {r['n_c']} min Phi {m:.3e}", flush=True)
        if m >= -s["eps_ncp"]:
            return s["pos"], s["quat"], k + 1, m
    raise RuntimeError("relaxation did not reach min Phi >= -eps_NCP")


def render(seed: int = 1) -> str:
    sc = scenes.cfg1(seed)
    pos, quat, steps, m = relax(sc)
    body = "".join(" ".join(f"{v:.17g}" for v in (*p, *q)) + "\n" for p, q in zip(pos, quat))
    head = (f"# cfg1-relaxed (SURVEY.md §8(d)): gen.scenes.cfg1(seed={seed}) relaxed by the oracle's overdamped\n"
            f"# ReLCP steps (Algorithm 1, P:L526-548; overdamped P:L512-522; drag P:L928-944), dt 1e-2,\n"
            f"# zero velocity, until min Phi >= -eps_NCP over the candidate scan (P:L645-648).\n"
            f"# Written by tools/make_relaxed.py (oracle only).  steps {steps}, min Phi {m:.6e}\n"
            f"# sha256(body) {hashlib.sha256(body.encode()).hexdigest()}\n"
            f"# columns: px py pz qs qx qy qz (one line per body, body order of cfg1)\n")
    return head + body


if __name__ == "__main__":
    text = render()
    if "--check" in sys.argv:
        same = open(OUT).read() == text
        print("fixture reproduced bitwise" if same else "fixture DIFFERS")
        sys.exit(0 if same else 1)
    with open(OUT, "w") as f:
        f.write(text)
    print(OUT)
