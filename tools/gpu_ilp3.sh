mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q --timeout=600 -x > gpurun_out/pytest_ilp3.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_ilp3.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); r=d['roofline']
print(d['value'], d['ms_per_step'], d['config']['lcp_iters'], round(r['frac'],4), r['scatter_ms'], r['gather_ms'], d['clocks'], d['complete_step'], d['e2e']['value'])"
timeout 1500 python tools/bench_configs.py cfg1 cfg2 cfg3 cfg4 cfg4-6M cfg5 > gpurun_out/r02_configs.jsonl 2> gpurun_out/cfgs.err; echo cfgs_rc=$?
