# small-store iteration A/B: persistent variants vs the two-kernel path
for lib in "$@"; do
  tag=$(basename $lib .so)
  RELCP_LIB=$lib timeout 300 python tools/kbench_small.py cfg2 2000 2>&1 | tail -1 | sed "s/^/$tag /"
  RELCP_LIB=$lib timeout 300 python tools/kbench_small.py cfg3 1000 2>&1 | tail -1 | sed "s/^/$tag /"
done
RELCP_PBB_MAX_ROWS=0 timeout 300 python tools/kbench_small.py cfg2 2000 2>&1 | tail -1 | sed "s/^/two-kernel /"
RELCP_PBB_MAX_ROWS=0 timeout 300 python tools/kbench_small.py cfg3 1000 2>&1 | tail -1 | sed "s/^/two-kernel /"
