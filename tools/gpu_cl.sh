# K6 component-lane sums (K6_CL): bitwise/parity subset on each variant lib, then kbench A/B
mkdir -p gpurun_out
for lib in "$@"; do
  tag=$(basename $lib .so)
  RELCP_LIB=$lib timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "bodies_per_warp or apply_parity or lcp_solve_parity or hubs" > gpurun_out/cl_tests_$tag.log 2>&1; echo "$tag tests_rc=$?"; tail -1 gpurun_out/cl_tests_$tag.log
done
for rep in 1 2; do
for mode in a0 relaxed; do
  for lib in paper_2506_14097_b200/lib/librelcp.so "$@"; do
    tag=$(basename $lib .so)
    RELCP_LAYOUT=0 RELCP_LIB=$lib timeout 300 python tools/kbench.py 2000000 200 $mode > gpurun_out/kb_${mode}_${tag}.log 2>&1; echo "$mode $tag rc=$?"
    grep -h "apply\|solve" gpurun_out/kb_${mode}_${tag}.log | sed 's/(first batch).*K6/K6/'
  done
done
done
