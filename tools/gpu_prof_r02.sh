# round-2 evidence: power-iteration A/B on the headline, ncu --set full of K6 / K7 (BB) and the apply
# kernels on the relaxed headline store (N_C = 7.39M), CSR layout (the cfg5 AUTO choice)
mkdir -p gpurun_out
for p in 20 6 3; do
  timeout 900 python bench.py --power-iters $p --no-cpu-baseline --no-e2e --no-apply --no-literal --no-relabel > gpurun_out/bench_pi$p.json 2> gpurun_out/bench_pi$p.err; echo "power $p rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/bench_pi$p.json').read().strip().splitlines()[-1]); r=d['roofline']; s=d['step_report']
print($p, round(d['value'],1), round(d['ms_per_step'],2), s['iterations'], s['ms_generate'], s['ms_solve'], s['ms_check'], round(r['frac'],4), d['complete_step'])"
done
KBENCH_PROFILE_SOLVE=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_scatter|k_lcp_iter" -s 40 -c 4 -o gpurun_out/prof_iter_r02 python tools/kbench.py 2000000 200 relaxed > gpurun_out/ncu_iter.log 2>&1; echo ncu_iter=$?
KBENCH_PROFILE_APPLY=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_scatter|k_gather" -s 4 -c 4 -o gpurun_out/prof_apply_r02 python tools/kbench.py 2000000 20 relaxed > gpurun_out/ncu_apply.log 2>&1; echo ncu_apply=$?
