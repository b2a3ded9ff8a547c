# K6 bodies-per-warp A/B (K6_GB_SMALL variants given as arguments): small stores + cfg5 A_0, twice, interleaved
mkdir -p gpurun_out
for rep in 1 2; do
for lib in paper_2506_14097_b200/lib/librelcp.so "$@"; do
  tag=$(basename $lib .so)
  RELCP_LIB=$lib timeout 300 python tools/kbench_small.py cfg2 2000 2>&1 | tail -1 | sed "s/^/$tag /"
  RELCP_LIB=$lib timeout 300 python tools/kbench_small.py cfg3 1000 2>&1 | tail -1 | sed "s/^/$tag /"
  RELCP_LIB=$lib timeout 300 python tools/kbench.py 2000000 200 2>&1 | grep solve | sed "s/^/$tag /"
done
done
