mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dd.py tests/test_gpu_fullsize.py -m gpu -q --timeout=600 -rA > gpurun_out/pytest_dd.log 2>&1; echo pytest_rc=$?
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-apply --no-cpu-baseline --no-literal"
export RELCP_PROFILE_TIMED=1
timeout 400 $CMD > gpurun_out/plain.json 2> gpurun_out/plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
unset RELCP_PROFILE_TIMED
timeout 300 python tools/kbench.py 2000000 200 relaxed > gpurun_out/kbench_relaxed.log 2>&1; echo kb_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_lcp_iter|k_gather" -s 100 -c 6 -o gpurun_out/prof_relaxed python tools/kbench.py 2000000 200 relaxed > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
