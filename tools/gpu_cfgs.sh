# per-config records on both operator layouts -> gpurun_out/r02_configs.jsonl
mkdir -p gpurun_out
for lay in 0 1; do
  RELCP_LAYOUT=$lay timeout 900 python tools/bench_configs.py "$@" >> gpurun_out/r02_configs.jsonl 2> gpurun_out/cfgs_$lay.err; echo "layout $lay rc=$?"
done
