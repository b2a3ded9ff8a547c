"""Write tests/golden/cfg3_full_sample.txt: the ORACLE's LCP-SNSD step of the
full-size BASELINE cfg3 colony (200,000 planar ellipsoids, ~431k A_0 rows),
sampled.

Algorithm 1 lines 1-4 (overdamped form P:L512-522, local drag
P:L928-944): A_0 from the oracle's own broadphase + SNSD at C^k (R5), the LCP
0 <= g = Phi~_0 + A_0 gamma _|_ gamma >= 0 solved by orc_bbpgd to r <= 1e-12,
C_1 = C^k + dt G^k (W D gamma) -- oracle.relcp_step(..., snsd_only=True), the
paper's LCP-SNSD update.  A full copy is not stored: the file holds
sha256 of the (ia, ib) list, N_C, and a seeded sample of 20,000 rows (ia, ib,
lambda, g, Phi) and 5,000 bodies (C_1 position and quaternion), plus the
maxima of |lambda| and |g| over ALL rows.  Calls only gen/ and oracle/.

    python tools/make_cfg3_sample.py          # ~10 min on one core
"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from gen import scenes  # noqa: E402
from oracle import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "cfg3_full_sample.txt")
TOL = 1e-12


def main():
    sc = scenes.cfg3()
    t0 = time.time()
    r = oracle.relcp_step(sc, lcp_tol=TOL, max_recursions=0, snsd_only=True, lcp_max_iter=2_000_000)
    secs = time.time() - t0
    if not all(r["converged"]):
        raise RuntimeError(f"oracle did not converge: {r['residuals']}")
    c = r["constraints"]
    ia, ib = c["ia"].astype(np.int32), c["ib"].astype(np.int32)
    o = np.lexsort((ib, ia))
    ia, ib, lam, g, phi = ia[o], ib[o], c["lam"][o], r["g_hist"][0][o], c["phi"][o]
    rng = np.random.Generator(np.random.PCG64(303))
    rows = np.sort(rng.choice(len(ia), 20000, replace=False))
    bods = np.sort(rng.choice(sc["n"], 5000, replace=False))
    pos, quat = r["pos"], r["quat"]
    lines = [
        "# cfg3 (BASELINE configs[2], gen.scenes.cfg3(seed=3), 200,000 planar ellipsoids): the ORACLE's",
        f"# LCP-SNSD step (oracle.relcp_step snsd_only, orc_bbpgd tol {TOL:g}): iterations {r['iterations'][0]}, "
        f"residual {r['residuals'][0]:.3e}, {secs:.0f} s",
        "# Algorithm 1 lines 1-4 (P:L526-536), overdamped (P:L512-522), drag (P:L928-944), LCP-SNSD (P:L908).",
        "# Written by tools/make_cfg3_sample.py (oracle only).  Rows sorted by (ia, ib) (R18).",
        f"# n_rows {len(ia)} n_bodies {sc['n']}",
        f"# max_abs lam {np.max(np.abs(lam)):.17g} g {np.max(np.abs(g)):.17g}",
        f"# rows_sha256 {hashlib.sha256(ia.tobytes() + ib.tobytes()).hexdigest()}",
        "# R <row> <ia> <ib> <lambda> <g> <phi>   |   B <body> <x y z> <qs qx qy qz> (C_1, wrapped)",
    ]
    lines += [f"R {i} {ia[i]} {ib[i]} {lam[i]:.17g} {g[i]:.17g} {phi[i]:.17g}" for i in rows]
    lines += [f"B {b} " + " ".join(f"{v:.17g}" for v in (*pos[b], *quat[b])) for b in bods]
    with open(OUT, "w") as f:
        f.write("\n".join(lines) + "\n")
    print(OUT, r["iterations"], r["residuals"], secs)


if __name__ == "__main__":
    main()
