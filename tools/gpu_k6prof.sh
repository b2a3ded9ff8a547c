# ncu --set full of K6 (BB mode) on the relaxed store for each lib given
mkdir -p gpurun_out
for lib in "$@"; do
  tag=$(basename $lib .so)
  RELCP_LIB=$lib timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_lcp_iter" -s 60 -c 3 -o gpurun_out/prof_$tag python tools/kbench.py 2000000 200 relaxed > gpurun_out/ncu_$tag.log 2>&1; echo "$tag ncu_rc=$?"
done
