# new K7 default (ILP 1 x 3 blocks): parity files, then the apply-gather ILP A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dd.py tests/test_gpu_edge.py -m gpu -q -x > gpurun_out/k7new_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/k7new_tests.log
for rep in 1 2; do for mode in a0 relaxed; do for lib in paper_2506_14097_b200/lib/librelcp.so "$@"; do
  tag=$(basename $lib .so)
  RELCP_LAYOUT=0 RELCP_LIB=$lib timeout 300 python tools/kbench.py 2000000 200 $mode > gpurun_out/kb_${mode}_${tag}.log 2>&1
  echo "$mode $tag $(grep -h 'apply' gpurun_out/kb_${mode}_${tag}.log | sed 's/.*apply/apply/') $(grep -h solve gpurun_out/kb_${mode}_${tag}.log | sed 's/.*scatter/scatter/; s/(first batch).*//')"
done; done; done
