# K7 block shape / ILP A/B: kbench on cfg5 A_0 and the relaxed store, cfg3 iteration (bench_configs) per library
mkdir -p gpurun_out
for rep in 1 2; do
for mode in a0 relaxed; do
  for lib in paper_2506_14097_b200/lib/librelcp.so "$@"; do
    tag=$(basename $lib .so)
    RELCP_LAYOUT=0 RELCP_LIB=$lib timeout 300 python tools/kbench.py 2000000 200 $mode > gpurun_out/kb_${mode}_${tag}.log 2>&1
    echo "$mode $tag $(grep -h solve gpurun_out/kb_${mode}_${tag}.log | sed 's/.*scatter/scatter/; s/(first batch).*//')"
  done
done
done
for lib in paper_2506_14097_b200/lib/librelcp.so "$@"; do
  tag=$(basename $lib .so)
  RELCP_LIB=$lib timeout 600 python tools/bench_configs.py cfg3 cfg2 > gpurun_out/cfg3_${tag}.jsonl 2> gpurun_out/cfg3_${tag}.err
  python - "$tag" gpurun_out/cfg3_${tag}.jsonl <<'PY'
import json, sys
for l in open(sys.argv[2]):
    d = json.loads(l)
    print(sys.argv[1], d.get('config'), {k: (round(v, 4) if isinstance(v, float) else v) for k, v in d.items() if 'iter' in k and not isinstance(v, (list, dict))})
PY
done
