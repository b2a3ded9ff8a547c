# JDS K6 bring-up: GPU parity tests of the new layout, then kbench A/B (CSR vs JDS, register budgets)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout=400 -k "layout or jds" > gpurun_out/pytest_jds.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_jds.log
for mode in a0 relaxed; do
  RELCP_LAYOUT=0 timeout 300 python tools/kbench.py 2000000 200 $mode > gpurun_out/kb_${mode}_csr.log 2>&1; echo "$mode csr rc=$?"
  grep -h "apply\|solve" gpurun_out/kb_${mode}_csr.log
  for lib in paper_2506_14097_b200/lib/librelcp.so paper_2506_14097_b200/lib/variants/librelcp_t128.so paper_2506_14097_b200/lib/variants/librelcp_m6.so; do
    tag=$(basename $lib .so)
    RELCP_LIB=$lib timeout 300 python tools/kbench.py 2000000 200 $mode > gpurun_out/kb_${mode}_${tag}.log 2>&1; echo "$mode $tag rc=$?"
    grep -h "apply\|solve" gpurun_out/kb_${mode}_${tag}.log
  done
done
