mkdir -p gpurun_out
for rep in 1 2; do
for f in paper_2506_14097_b200/lib/librelcp.so paper_2506_14097_b200/lib/variants/*.so; do
  echo "== $f"; RELCP_LIB=$f timeout 120 python tools/kbench.py 2000000 300 ${1:-} 2>&1 | tail -2
done
done > gpurun_out/sweep.log 2>&1
