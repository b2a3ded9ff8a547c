"""Write tests/golden/cfg4_full_sample.txt: the ORACLE's solution of the
full-size BASELINE cfg4 network LCP (1000 x 1000 rings, ~4.0M rows), sampled.

The cfg4 LCP (0 <= g = A lambda + q _|_ lambda >= 0, A = dt^2 D^T M^-1 D,
Lemma 3; rows t = r x n P:L1413; q = Phi_0 + dt D^T U^k,
P:L557-561) is solved by oracle.network_lcp (orc_bbpgd, serial C, long-double
dots) to r <= 1e-12 (both sides solve to 1e-12: with 1-3 rows per link A
is ill-conditioned and r <= 1e-10 leaves lambda determined only to ~1e-6, R19).  A full copy of lambda (32 MB) is not stored: the file
holds a seeded sample of 20,000 rows (lambda, g) and 5,000 bodies (U = W D
lambda, unique by Lemma 5), plus max|lambda|, max|g|, max|U| over
ALL rows / bodies.  This script calls only gen/ and oracle/; nothing here
comes from the CUDA path.

    python tools/make_cfg4_sample.py [tol] [out]   # writes the fixture (tens of minutes, one core)
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

OUT = os.path.join(ROOT, "tests", "golden", "cfg4_full_sample.txt")
TOL = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-12
if len(sys.argv) > 2:
    OUT = sys.argv[2]


def main():
    sc = scenes.cfg4()
    t0 = time.time()
    x, g, info, W, rw = oracle.network_lcp(sc, tol=TOL)
    secs = time.time() - t0
    if not info["converged"]:
        raise RuntimeError(f"oracle did not converge: {info}")
    _, U = oracle.wrench(W, rw["ia"], rw["ib"], rw["n"], rw["ta"], rw["tb"], x)
    rng = np.random.Generator(np.random.PCG64(404))
    rows = np.sort(rng.choice(len(x), 20000, replace=False))
    bods = np.sort(rng.choice(sc["n"], 5000, replace=False))
    lines = [
        "# cfg4 (BASELINE configs[3], gen.scenes.cfg4(seed=4), 1000 x 1000 rings) solved by the ORACLE",
        f"# oracle.network_lcp (orc_bbpgd, serial, tol {TOL:g}): iterations {info['iterations']}, "
        f"residual {info['residual']:.3e}, {secs:.0f} s",
        "# Lemma 3 (P:L280-299); rows t = r x n (P:L1413); q = Phi_0 + dt D^T U^k (P:L557-561);",
        "# U = W D lambda unique (Lemma 5, P:L333-373).  Written by tools/make_cfg4_sample.py (oracle only).",
        f"# n_rows {len(x)} n_bodies {sc['n']} active_fraction {float(np.mean(x > 0)):.6f}",
        f"# max_abs lam {np.max(np.abs(x)):.17g} g {np.max(np.abs(g)):.17g} U {np.max(np.abs(U)):.17g}",
        f"# rows_sha256 {hashlib.sha256(rw['ia'].tobytes() + rw['ib'].tobytes()).hexdigest()}",
        "# R <row> <lambda> <g>   |   B <body> <U0..U5>",
    ]
    lines += [f"R {i} {x[i]:.17g} {g[i]:.17g}" for i in rows]
    lines += [f"B {b} " + " ".join(f"{v:.17g}" for v in U[b]) for b in bods]
    with open(OUT, "w") as f:
        f.write("\n".join(lines) + "\n")
    print(OUT, info, secs)


if __name__ == "__main__":
    main()
