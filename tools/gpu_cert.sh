# SNSD curvature certificate: the new test + SNSD / step parity, then the headline bench and a phase breakdown
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout=400 -k "snsd or step or generate or broadphase" > gpurun_out/pytest_cert.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_cert.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-apply --no-literal --no-relabel > gpurun_out/bench_cert.json 2> gpurun_out/bench_cert.err; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_cert.json').read().strip().splitlines()[-1]); r=d['roofline']; s=d['step_report']
print(round(d['value'],1), round(d['ms_per_step'],2), s['iterations'], s['ms_generate'], s['ms_solve'], s['ms_check'], round(r['frac'],4), d['complete_step'], s['max_overlap'])"
RELCP_LIB=paper_2506_14097_b200/lib/librelcp_phases.so timeout 600 python tools/phases.py 2000000 relaxed > gpurun_out/phases_relaxed_cert.txt 2>&1; grep -E "^(snsd|solve|bp)" gpurun_out/phases_relaxed_cert.txt | tail -8
