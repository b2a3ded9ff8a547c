# round-2 GPU pass: every GPU test, smoke, the full bench, per-config records
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout=600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
rm -f gpurun_out/r02_configs.jsonl
timeout 1500 python tools/bench_configs.py cfg1 cfg2 cfg3 cfg4 cfg4-6M cfg5 > gpurun_out/r02_configs.jsonl 2> gpurun_out/cfgs.err; echo cfgs_rc=$?
