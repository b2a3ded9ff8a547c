# K7 variants on the mid-size (cfg3) and cfg5 stores
mkdir -p gpurun_out
for lib in "$@"; do
  tag=$(basename $lib .so)
  RELCP_LIB=$lib timeout 300 python tools/kbench_small.py cfg3 3000 > gpurun_out/k7_cfg3_$tag.log 2>&1; echo "cfg3 $tag rc=$?"; tail -1 gpurun_out/k7_cfg3_$tag.log
  RELCP_LIB=$lib timeout 300 python tools/kbench.py 2000000 200 relaxed > gpurun_out/k7_cfg5_$tag.log 2>&1; echo "cfg5 $tag rc=$?"; grep solve gpurun_out/k7_cfg5_$tag.log | sed 's/iter alg.*//'
done
