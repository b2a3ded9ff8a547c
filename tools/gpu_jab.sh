mkdir -p gpurun_out
for lib in "$@"; do
  tag=$(basename $lib .so)
  RELCP_LIB=$lib timeout 300 python tools/kbench_small.py cfg3 3000 > gpurun_out/j_cfg3_$tag.log 2>&1; echo "cfg3 $tag rc=$?"; tail -1 gpurun_out/j_cfg3_$tag.log
done
