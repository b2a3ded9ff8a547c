mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout=400 -k "k6_pipe" > gpurun_out/pytest_pipe.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_pipe.log
for mode in a0 relaxed; do for p in 0 1; do
  RELCP_K6PIPE=$p timeout 300 python tools/kbench.py 2000000 200 $mode > gpurun_out/kbp_${mode}_$p.log 2>&1; echo "$mode pipe=$p rc=$?"
  grep -h "apply\|solve" gpurun_out/kbp_${mode}_$p.log | sed 's/(first batch).*K6/K6/'
done; done
