# programmatic dependent launch A/B: small / mid / cfg5 stores, then the LCP / step parity tests
mkdir -p gpurun_out
for lib in paper_2506_14097_b200/lib/librelcp.so paper_2506_14097_b200/lib/variants/librelcp_nopdl.so; do
  tag=$(basename $lib .so)
  for cfg in cfg2 cfg3; do
    RELCP_CLUSTER=0 RELCP_LIB=$lib timeout 300 python tools/kbench_small.py $cfg 3000 > gpurun_out/pdl_${cfg}_$tag.log 2>&1; echo "$cfg $tag rc=$?"; tail -1 gpurun_out/pdl_${cfg}_$tag.log
  done
  RELCP_LIB=$lib timeout 300 python tools/kbench.py 2000000 200 relaxed > gpurun_out/pdl_cfg5_$tag.log 2>&1; echo "cfg5 $tag rc=$?"; grep solve gpurun_out/pdl_cfg5_$tag.log | sed 's/(first batch).*iter /iter /'
done
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout=400 -k "lcp or step or timing or cfg4" > gpurun_out/pytest_pdl.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_pdl.log
