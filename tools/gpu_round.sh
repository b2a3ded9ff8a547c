# One GPU round: GPU tests, smoke, bench, ncu launch list of one timed step,
# ncu --set full of the LCP-iteration kernels.  Run under gpurun.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout=400 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-apply --no-cpu-baseline"
export RELCP_PROFILE_TIMED=1
timeout 400 $CMD > gpurun_out/plain.json 2> gpurun_out/plain.err && \
timeout 3300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
unset RELCP_PROFILE_TIMED
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_lcp_iter" -s 100 -c 4 -o gpurun_out/prof_iter python tools/kbench.py 2000000 200 > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_snsd" -c 3 -o gpurun_out/prof_snsd python tools/kbench.py 2000000 20 > gpurun_out/ncu_snsd.log 2>&1; echo ncu3_rc=$?
