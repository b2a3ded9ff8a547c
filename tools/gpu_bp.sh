mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x --timeout=600 -k "broadphase or generate or step or subbox" > gpurun_out/pytest_bp.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_bp.log
RELCP_LIB=paper_2506_14097_b200/lib/librelcp_phases.so timeout 600 python tools/phases.py 2000000 relaxed > gpurun_out/phases_relaxed_bp.txt 2>&1; grep -E "^(snsd|solve|bp)" gpurun_out/phases_relaxed_bp.txt | head -8
timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-apply --no-relabel > gpurun_out/bench_bp.json 2> gpurun_out/bench_bp.err; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_bp.json').read().strip().splitlines()[-1]); r=d['roofline']; s=d['step_report']
print(round(d['value'],1), round(d['ms_per_step'],2), s['iterations'], round(s['ms_generate'],2), round(s['ms_solve'],2), round(s['ms_check'],2), round(r['frac'],4), round(r['iter_ms']*1e3,1), d['clocks']['sm_mhz'], d['complete_step'])
l=d['literal_cfg5']; print('literal', round(l['value'],1), l['ms_per_step'], l['step_report']['ms_generate'], l['step_report']['ms_check'])"
