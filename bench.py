"""Benchmark of the B200 ReLCP hot path (arXiv 2506.14097) -- driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json metric config, configs[4]): cfg5 = 2,000,000
ellipsoids (1.0, 0.6, 0.4), periodic cube at phi = 0.55, uniform random
orientations, u, w ~ N(0,1), dt = 1e-3, inertial, fp64, seeded synthetic
(gen/scenes.py).  One timed step = one full ReLCP time step through the C ABI
(relcp_step: broadphase + SNSD generation of A_0, LCP solves, trial
configurations, SNSD check + augmentation) from the same initial state.  The
literal cfg5 start overlaps deeply (Phi_0 down to -0.5), so the recursion
does not settle quickly: the step is capped at `--max-recursions` (2: N_C
grows 5.3M -> 8.5M -> 11.4M, BASELINE's "~10M after augmentation") and each
LCP at `--lcp-max-iter` BB iterations; both caps are in `config`.

metric  = LCP iterations/s: BB projected-gradient iterations executed in the
          K steps / device time of the K steps (whole step, generation and
          checks included), summed over ranks / max over ranks.
roofline: the fused LCP iteration (K6 scatter + K7 gather), algorithmic bytes
          216 N_C + 152 N per iteration / its CUDA-event time.
N > 1: independent replicas (seed 5 + rank), no data-path collective
(DESIGN.md "replicas only").

--impl reference: the CPU oracle (oracle/, test infrastructure) timed on the
host on a bounded sample of the same recipe, scaled to the 2M workload by the
body-count ratio (iteration cost is linear in N_C ~ N).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from gen import scenes  # noqa: E402

METRIC = "LCP iterations/s (fp64, 2M ellipsoids, 1 B200)"
UNIT = "iterations/s"
N_FULL = 2_000_000


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_FULL)
    ap.add_argument("--max-recursions", type=int, default=2)
    ap.add_argument("--lcp-max-iter", type=int, default=3000)
    ap.add_argument("--sample-n", type=int, default=1000, help="oracle sample size (bodies)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-apply", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------- oracle leg
def oracle_sample(args, steps=1):
    """Time the CPU oracle's ReLCP step on a bounded cfg5-recipe sample."""
    from oracle import oracle as O
    O.build()
    sc = scenes.cfg5(n=args.sample_n)
    iters = 0
    t = 0.0
    rows = []
    for _ in range(steps):
        t0 = time.perf_counter()
        r = O.relcp_step(sc, max_recursions=args.max_recursions, lcp_tol=1e-8, lcp_max_iter=args.lcp_max_iter)
        t += time.perf_counter() - t0
        iters += sum(r["iterations"])
        rows = r["n_c"]
    raw = iters / t
    scaled = raw * args.sample_n / args.n
    return dict(value=scaled, raw_it_per_s=raw, seconds=t, iterations=iters, n_c=rows)


def run_reference(args, rank, world):
    if rank != 0:
        return
    for _ in range(max(0, args.warmup)):
        oracle_sample(args, 1)
    r = oracle_sample(args, max(1, args.steps))
    sample = (f"oracle relcp_step on the cfg5 recipe at {args.sample_n} bodies (seed 5), "
              f"max_recursions={args.max_recursions}, lcp_max_iter={args.lcp_max_iter}, tol 1e-8; "
              f"it/s scaled by {args.sample_n}/{args.n} bodies")
    line = dict(impl="reference", metric=METRIC, value=r["value"], unit=UNIT, n_gpus=world, steps=args.steps,
                warmup=args.warmup, ms_per_step=1e3 * r["seconds"] / max(1, args.steps), higher_is_better=True,
                scaling="weak", vs_baseline=None, dtype="f64", data="synthetic",
                config=dict(workload=f"cfg5 sample ({args.sample_n} bodies) of the 2M-ellipsoid ReLCP step",
                            n_bodies=args.sample_n, max_recursions=args.max_recursions,
                            lcp_max_iter=args.lcp_max_iter),
                cpu_baseline=dict(value=r["value"], unit=UNIT, cores=1, kind="oracle", sample=sample,
                                  raw_it_per_s=r["raw_it_per_s"]),
                e2e=dict(value=r["value"], unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- clocks
class Clocks:
    def __init__(self, idx):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={idx}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["nvidia-smi unavailable"])
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [ln.split(",") for ln in open(self.f.name).read().strip().splitlines() if ln.count(",") >= 8]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].strip() in ("Active", "1")})
        return dict(sm_mhz=statistics.median(sm) if sm else None, sm_max_mhz=max(mx) if mx else None,
                    reasons=reasons, samples=len(rows))


# ---------------------------------------------------------------- ours
def combine_ranks(ms, iters, dist, device):
    """Whole-job aggregate over replicas: the MAX device time over ranks and
    the SUM of the iterations every rank executed (value = sum / max)."""
    if not dist:
        return ms, float(iters)
    import torch
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    it_t = torch.tensor([float(iters)], dtype=torch.float64, device=device)
    dist.all_reduce(it_t, op=dist.ReduceOp.SUM)
    return float(t.item()), float(it_t.item())


def iter_bytes(n_c, iters, n):
    return sum(it * (216.0 * c + 152.0 * n) for c, it in zip(n_c, iters))


def run_ours(args, rank, world, dist):
    import torch
    from paper_2506_14097_b200 import relcp as R

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    seed = 5 + rank
    sc = scenes.cfg5(seed=seed, n=args.n)
    ctx = R.Context(dynamics=sc["dynamics"], dt=sc["dt"], box=list(sc["box"]), cutoff=sc["cutoff"],
                    eps_ncp=sc["eps_ncp"], lcp_tol=1e-8, lcp_max_iter=args.lcp_max_iter,
                    max_recursions=args.max_recursions)
    bodies = R.BodyState.from_scene(sc)
    init = {k: getattr(bodies, k).clone() for k in ("pos", "quat", "vel")}
    cap = 8 * args.n + 4 * 1024 * 1024
    cs = R.ConstraintStore(cap)

    def restore():
        for k, v in init.items():
            getattr(bodies, k).copy_(v)

    reports = []

    def one_step():
        restore()
        rep = ctx.step(bodies, cs)
        reports.append(rep)
        return rep

    for _ in range(max(3, args.warmup)):
        one_step()
    reports.clear()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ctx.reset_stats()
    ctx.set_timing(True)
    clocks = Clocks(dev.index) if rank == 0 else None
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof = os.environ.get("RELCP_PROFILE_TIMED") == "1"  # ncu --profile-from-start off: timed region only
    if prof:
        torch.cuda.profiler.start()
    e0.record()
    for _ in range(args.steps):
        one_step()
    e1.record()
    torch.cuda.synchronize()
    if prof:
        torch.cuda.profiler.stop()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop() if clocks else None
    ctx.set_timing(False)
    stats = ctx.stats()
    iters = sum(sum(r["iterations"]) for r in reports)
    assert iters == stats["lcp_iterations"], (iters, stats)
    nbytes = sum(iter_bytes(r["n_c"], r["iterations"], args.n) for r in reports)
    # timed iterations: each solve's first batch (events around K6 / K7) and its
    # complete CUDA-graph batches (events around the graph launch); the few
    # iterations of a solve's last, partly executed batch are left out
    it_timed = max(1, stats["iter_timed"])
    it_ms = stats["iter_ms"] * iters / it_timed  # extrapolated to every iteration of the step
    ms_max, iters_all = combine_ranks(ms, iters, dist, dev)
    value = iters_all / (ms_max / 1e3)

    peaks = {}
    pk_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk_path):
        peaks = json.load(open(pk_path))
    peak = peaks.get("hbm_gbs")
    peak_src = "measured" if peak else "fallback"
    peak = peak or 6650.0
    achieved = (nbytes / iters) / (stats["iter_ms"] / it_timed / 1e3) / 1e9 if stats["iter_ms"] > 0 else None
    # DRAM traffic per iteration from the committed ncu --set full capture (K6 + K7)
    traffic = traffic_ratio = traffic_nc = None
    tr_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tr_path):
        tr = json.load(open(tr_path))
        traffic, traffic_ratio, traffic_nc = tr["dram_bytes_per_iteration"], tr["ratio"], tr["n_c"]

    # Delassus apply GB/s at A_0 and at the final (largest) store
    apply = {}
    if not args.no_apply:
        for label in ("final", "A0"):
            restore()
            if label == "final":
                ctx.step(bodies, cs)
                restore()
            else:
                ctx.generate_contacts(bodies, cs)
            ctx.prepare_operator(bodies, cs)
            nc = cs.count
            x = torch.rand(nc, dtype=torch.float64, device=dev)
            y = torch.empty_like(x)
            for _ in range(5):
                ctx.delassus_apply(bodies, cs, x, y)
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 30
            a0.record()
            for _ in range(reps):
                ctx.delassus_apply(bodies, cs, x, y)
            a1.record()
            torch.cuda.synchronize()
            ams = a0.elapsed_time(a1) / reps
            ab = 176.0 * nc + 152.0 * args.n
            apply[label] = dict(n_c=nc, ms=ams, alg_bytes=ab, GBps=ab / (ams / 1e3) / 1e9,
                                frac=ab / (ams / 1e3) / 1e9 / peak)

    # end to end through the public API with host buffers (pinned), copies timed
    e2e = None
    if not args.no_e2e:
        fields_in = ("pos", "quat", "vel", "axes", "inv_mass", "inv_inertia")
        host_in = {k: getattr(bodies, k).cpu().pin_memory() for k in fields_in}
        for k in ("pos", "quat", "vel"):
            host_in[k].copy_(init[k].cpu())
        host_out = {k: torch.empty_like(host_in[k]).pin_memory() for k in ("pos", "quat", "vel")}
        h2d = sum(v.numel() * v.element_size() for v in host_in.values())
        d2h = sum(v.numel() * v.element_size() for v in host_out.values())
        reports.clear()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            for k in fields_in:
                getattr(bodies, k).copy_(host_in[k], non_blocking=True)
            reports.append(ctx.step(bodies, cs))
            for k in ("pos", "quat", "vel"):
                host_out[k].copy_(getattr(bodies, k), non_blocking=True)
        f1.record()
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1)
        eit = sum(sum(r["iterations"]) for r in reports)
        e2e = dict(value=eit / (ems / 1e3) * (world if dist else 1), unit=UNIT, h2d_bytes_per_step=int(h2d),
                   d2h_bytes_per_step=int(d2h), ms_per_step=ems / args.steps)

    if rank != 0:
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        r = oracle_sample(args, 1)
        cpu = dict(value=r["value"], unit=UNIT, cores=1, kind="oracle",
                   sample=(f"oracle relcp_step, cfg5 recipe at {args.sample_n} bodies, same caps, tol 1e-8; "
                           f"{r['iterations']} iterations in {r['seconds']:.1f} s = {r['raw_it_per_s']:.1f} it/s "
                           f"at N_C {r['n_c']}, scaled by {args.sample_n}/{args.n}"),
                   raw_it_per_s=r["raw_it_per_s"])
    last = reports[-1] if reports else {}
    line = dict(
        metric=METRIC, value=value, unit=UNIT, n_gpus=world, steps=args.steps, warmup=max(3, args.warmup),
        ms_per_step=ms_max / args.steps, higher_is_better=True, scaling="weak", vs_baseline=None, dtype="f64",
        data="synthetic",
        config=dict(workload="cfg5: 2M ellipsoids (1.0,0.6,0.4), periodic phi=0.55, dt=1e-3, inertial; one "
                             "ReLCP step (generate + LCP solves + check/augment)",
                    n_bodies=args.n, max_recursions=args.max_recursions, lcp_max_iter=args.lcp_max_iter,
                    lcp_tol=1e-8, parallelism=f"replicas{world}", l2="inputs larger than L2 (GB working set)",
                    n_c=last.get("n_c"), lcp_iters=last.get("iterations"), n_pairs=last.get("n_pairs")),
        roofline=dict(bound="hbm", kernel="LCP iteration (K6 scatter + K7 gather)", achieved=achieved, peak=peak,
                      unit="GB/s", frac=(achieved / peak) if achieved else None, traffic=traffic,
                      traffic_n_c=traffic_nc, traffic_over_algorithmic=traffic_ratio,
                      peak_source=peak_src, frac_of_8TBps=(achieved / 8000.0) if achieved else None,
                      iter_ms=stats["iter_ms"] / it_timed, iters_timed=stats["iter_timed"],
                      scatter_ms=stats["scatter_ms"] / max(1, stats["split_timed"]),
                      gather_ms=stats["gather_ms"] / max(1, stats["split_timed"]),
                      split_timed=stats["split_timed"], share_of_step=it_ms / ms),
        delassus_apply=apply,
        cpu_baseline=cpu, e2e=e2e, gpu_launches=stats["launches"], clocks=clk,
        step_report={k: last.get(k) for k in ("recursions", "status", "residuals", "max_overlap", "ms_generate",
                                              "ms_solve", "ms_check", "snsd_nonconv")},
    )
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        tdist.init_process_group("nccl")
        dist = tdist
    try:
        run_ours(args, rank, world, dist)
    finally:
        if dist:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
