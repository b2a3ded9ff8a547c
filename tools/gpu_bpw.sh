# k6_bpw: bitwise test, small-store A/B (auto vs 32), ncu durations of the cfg2 iteration kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "bodies_per_warp or k6_pipe or apply_parity or lcp_solve_parity_cfg1" > gpurun_out/bpw_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/bpw_tests.log
for rep in 1 2; do
for bpw in 0 32 16; do
  RELCP_K6_BPW=$bpw timeout 300 python tools/kbench_small.py cfg2 2000 2>&1 | tail -1 | sed "s/^/bpw$bpw /"
done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/cfg2_launches.csv python tools/kbench_small.py cfg2 100 > gpurun_out/cfg2_ncu.log 2>&1; echo ncu_rc=$?
python - <<'PY'
import csv, collections
rows = list(csv.reader(l for l in open('gpurun_out/cfg2_launches.csv') if l.startswith('"')))
h = rows[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
d = collections.defaultdict(list)
for r in rows[1:]:
    v = float(r[vi].replace(',', '')); v = v / 1000 if r[ui] == 'nsecond' else v
    d[r[ki][:60]].append(v)
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    v2 = sorted(v); print(f"{len(v):5d} median {v2[len(v2)//2]:8.2f} us  {k}")
PY
