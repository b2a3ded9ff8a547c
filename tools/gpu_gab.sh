# apply-gather variants (K7') on cfg5 A_0 / relaxed
mkdir -p gpurun_out
for lib in "$@"; do
  tag=$(basename $lib .so)
  for mode in a0 relaxed; do
    RELCP_LIB=$lib timeout 300 python tools/kbench.py 2000000 20 $mode > gpurun_out/g_${mode}_$tag.log 2>&1; echo "$mode $tag rc=$?"; grep apply gpurun_out/g_${mode}_$tag.log
  done
done
