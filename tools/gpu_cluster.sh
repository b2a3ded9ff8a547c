# single-cluster BB loop: micro-bench cfg1 / cfg2 (cluster on / off), then the GPU parity file
mkdir -p gpurun_out
for cfg in cfg1 cfg2; do for c in 0 1; do
  RELCP_CLUSTER=$c timeout 300 python tools/kbench_small.py $cfg 4000 > gpurun_out/ks_${cfg}_$c.log 2>&1; echo "$cfg cluster=$c rc=$?"; tail -2 gpurun_out/ks_${cfg}_$c.log
done; done
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout=400 > gpurun_out/pytest_parity.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_parity.log
