"""DRAM bytes per LCP iteration (K6 + K7) and per Delassus apply (K6 mode 0 +
gather) from `ncu --set full` raw CSV exports, against the algorithmic bytes
(216 N_C + 152 N per iteration, 176 N_C + 152 N per apply).

    python tools/ncu_traffic.py ITER_RAW.csv [APPLY_RAW.csv] [--nc N_C --n N --store NAME] > profiles/ncu_traffic.json

Round 2 (the headline's store): profiles/r02_prof_iter_relaxed_raw.csv,
profiles/r02_prof_apply_relaxed_raw.csv, --nc 7393149 --n 2000000 --store
"cfg5-relaxed A_0" (tools/kbench.py 2000000 200 relaxed, CSR layout).
"""
import csv
import json
import sys

UNIT_B = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
UNIT_US = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
NC, N, STORE = 5304369, 2000000, "cfg5 A_0"  # defaults: tools/kbench.py 2000000
args = []
i = 1
while i < len(sys.argv):
    if sys.argv[i] == "--nc":
        NC = int(sys.argv[i + 1]); i += 2
    elif sys.argv[i] == "--n":
        N = int(sys.argv[i + 1]); i += 2
    elif sys.argv[i] == "--store":
        STORE = sys.argv[i + 1]; i += 2
    else:
        args.append(sys.argv[i]); i += 1


def kernels(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    ki, ti = h.index("Kernel Name"), h.index("gpu__time_duration.sum")
    rd, wr = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    out = {}
    for r in rows[2:]:
        name = r[ki].split("(")[0].replace("void ", "")
        b = float(r[rd]) * UNIT_B[units[rd]] + float(r[wr]) * UNIT_B[units[wr]]
        us = float(r[ti]) * UNIT_US[units[ti]]
        out.setdefault(name, []).append((b, us))
    return {k: (sum(b for b, _ in v) / len(v), sum(u for _, u in v) / len(v)) for k, v in out.items()}


def pick(ks, prefix):
    hits = [v for k, v in ks.items() if k.startswith(prefix)]
    assert len(hits) == 1, (prefix, list(ks))
    return hits[0]


it = kernels(args[0])
k6, k7 = pick(it, "k_scatter<1"), pick(it, "k_lcp_iter")
res = dict(source=f"ncu --set full, tools/kbench.py ({STORE} store): {args[0]}", n_c=NC, n=N,
           k6_dram_bytes=k6[0], k7_dram_bytes=k7[0], dram_bytes_per_iteration=k6[0] + k7[0],
           alg_bytes_per_iteration=216 * NC + 152 * N, k6_us=k6[1], k7_us=k7[1])
res["ratio"] = res["dram_bytes_per_iteration"] / res["alg_bytes_per_iteration"]
if len(args) > 1:
    ap = kernels(args[1])
    s0, ga = pick(ap, "k_scatter<0"), pick(ap, "k_gather")
    res.update(apply_source=args[1], apply_dram_bytes=s0[0] + ga[0], apply_alg_bytes=176 * NC + 152 * N,
               apply_scatter_us=s0[1], apply_gather_us=ga[1])
    res["apply_ratio"] = res["apply_dram_bytes"] / res["apply_alg_bytes"]
print(json.dumps(res, indent=1))
