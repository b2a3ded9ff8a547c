mkdir -p gpurun_out
MODE=${1:-a0}
CMD="python tools/kbench.py 2000000 200 $MODE"
timeout 300 $CMD > gpurun_out/kbench_$MODE.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_lcp_iter|k_gather" -s 60 -c 4 -o gpurun_out/prof_k_$MODE $CMD > gpurun_out/ncu_k_$MODE.log 2>&1; echo ncu_rc=$?
