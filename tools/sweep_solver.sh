mkdir -p gpurun_out
for s in 0 2 0 2; do
  echo "== solver $s"; RELCP_SOLVER=$s timeout 120 python tools/kbench.py 2000000 300 ${1:-} 2>&1 | grep solve
done
