# single-cluster BB loop A/B (fences, cluster size) on cfg1 / cfg2, then the parity file twice
mkdir -p gpurun_out
for cfg in cfg1 cfg2; do
  for lib in paper_2506_14097_b200/lib/librelcp.so "$@"; do
    tag=$(basename $lib .so)
    RELCP_LIB=$lib timeout 300 python tools/kbench_small.py $cfg 4000 > gpurun_out/ks_${cfg}_$tag.log 2>&1; echo "$cfg $tag rc=$?"; tail -1 gpurun_out/ks_${cfg}_$tag.log
  done
done
for r in 1 2; do
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout=400 > gpurun_out/pytest_parity_$r.log 2>&1; echo pytest_rc=$?
tail -1 gpurun_out/pytest_parity_$r.log
done
