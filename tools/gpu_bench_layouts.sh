# headline bench on both operator layouts (headline line only)
mkdir -p gpurun_out
for lay in 0 1 0 1; do
  timeout 900 python bench.py --layout $lay --no-cpu-baseline --no-e2e --no-apply --no-literal --no-relabel > gpurun_out/bench_lay$lay.json 2> gpurun_out/bench_lay$lay.err; echo "layout $lay rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/bench_lay$lay.json').read().strip().splitlines()[-1]); r=d['roofline']
print(d['config']['operator_layout'], round(d['value'],1), round(d['ms_per_step'],2), d['config']['lcp_iters'], round(r['frac'],4), round(r['iter_ms']*1e3,1), round(r['scatter_ms']*1e3,1), round(r['gather_ms']*1e3,1), d['clocks']['sm_mhz'])"
done
