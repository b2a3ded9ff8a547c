# K6 A/B: libs given as args (default lib first); kbench on cfg5 A_0 and the relaxed store
mkdir -p gpurun_out
for mode in a0 relaxed; do
  for lib in "$@"; do
    tag=$(basename $lib .so)
    RELCP_LIB=$lib timeout 300 python tools/kbench.py 2000000 200 $mode > gpurun_out/kb_${mode}_${tag}.log 2>&1; echo "$mode $tag rc=$?"
    grep -h "apply\|solve" gpurun_out/kb_${mode}_${tag}.log
  done
done
