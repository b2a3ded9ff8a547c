# round-2 evidence pass: every GPU test, smoke, the full bench, per-config records,
# the ncu launch list of one timed headline step (kernel shares)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout=600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 1500 python tools/bench_configs.py cfg1 cfg2 cfg3 cfg4 cfg4-6M cfg5 > gpurun_out/r02_configs.jsonl 2> gpurun_out/cfgs.err; echo cfgs_rc=$?
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-apply --no-cpu-baseline --no-literal --no-relabel"
export RELCP_PROFILE_TIMED=1
timeout 400 $CMD > gpurun_out/plain.json 2> gpurun_out/plain.err && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
unset RELCP_PROFILE_TIMED
python tools/launch_share.py gpurun_out/launches.csv > gpurun_out/launch_share.txt 2>&1; head -20 gpurun_out/launch_share.txt
