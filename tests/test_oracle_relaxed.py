"""cfg1-relaxed: the overlap-free companion of cfg1 and the
small-timestep reduction it exists to pin.

The paper's reduction corollary (proof P:L1910-1935): from an
overlap-free C^k, the maximum overlap left by the recursion-0 (classical SNSD
LCP) update, eta_1(dt), tends to 0 as dt -> 0, so below some dt_red no row is
appended and ReLCP equals the single-constraint SNSD LCP.  The paper observes
exactly this at its smallest timestep.  With the LCP enforcing the
linearised gaps, the overlap left is the second-order remainder of that
linearisation (Taylor), so eta_1 falls roughly as dt^2.
"""
import importlib.util
import os

import numpy as np
import pytest

from gen import scenes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _make_relaxed():
    spec = importlib.util.spec_from_file_location("make_relaxed", os.path.join(ROOT, "tools", "make_relaxed.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_fixture_is_the_oracle_relaxation():
    """tests/golden/cfg1_relaxed.txt is what tools/make_relaxed.py (oracle only)
    writes: regenerate and compare the text bitwise."""
    mk = _make_relaxed()
    assert open(mk.OUT).read() == mk.render()


def test_relaxed_start_is_overlap_free(orc):
    """Every candidate pair of the stored state has Phi >= -eps_NCP (the
    stopping rule's acceptance), by a full oracle SNSD scan."""
    sc = scenes.cfg1_relaxed()
    rad = orc.bounding_radius(sc["axes"])
    pi, pj = orc.broadphase(sc["pos"], rad, sc["box"], sc["cutoff"])
    phi, *_ = orc.snsd(sc["pos"], sc["quat"], sc["axes"], sc["box"], pi, pj)
    assert len(phi) > 400
    assert np.min(phi) >= -sc["eps_ncp"]
    # the literal cfg1 start is deeply overlapping (SURVEY ambiguity #18)
    raw = scenes.cfg1()
    phi0, *_ = orc.snsd(raw["pos"], raw["quat"], raw["axes"], raw["box"], *orc.broadphase(
        raw["pos"], orc.bounding_radius(raw["axes"]), raw["box"], raw["cutoff"]))
    assert np.min(phi0) < -0.1


def test_reduction_small_dt_no_augmentation(orc):
    """at cfg1's dt = 1e-3 (and 1e-4) the recursion-0 update
    already meets the stopping rule: zero augmentations, and eta_1 shrinks
    with dt (by ~dt^2: measured 1.45e-6 -> 1.2e-8)."""
    eta = {}
    for dt in (1e-3, 1e-4):
        r = orc.relcp_step(scenes.cfg1_relaxed(dt=dt), lcp_tol=1e-10)
        assert r["recursions"] == 0 and r["status"] == 0
        assert r["max_overlap"] <= 1e-5
        eta[dt] = r["max_overlap"]
    assert eta[1e-4] < eta[1e-3] / 30.0


@pytest.mark.slow
def test_bigdt_augments_and_terminates(orc):
    """cfg1-bigdt: the relaxed start at dt = 0.1 leaves the
    small-dt regime; the recursion appends rows and still terminates with
    every pair at Phi >= -eps_NCP (Cor. P:L879-888)."""
    r = orc.relcp_step(scenes.cfg1_relaxed(dt=0.1), lcp_tol=1e-10)
    assert r["recursions"] >= 1 and r["status"] == 0
    assert r["max_overlap"] <= 1e-5
    assert r["n_c"] == sorted(r["n_c"]) and r["n_c"][-1] > r["n_c"][0]
