# K6 A/B on cfg5 A_0 and the relaxed store: CSR layout, then each library given as an argument (JDS AUTO)
mkdir -p gpurun_out
for mode in a0 relaxed; do
  RELCP_LAYOUT=0 timeout 300 python tools/kbench.py 2000000 200 $mode > gpurun_out/kb_${mode}_csr.log 2>&1; echo "$mode csr rc=$?"
  grep -h "solve" gpurun_out/kb_${mode}_csr.log | sed 's/(first batch).*K6/K6/'
  for lib in "$@"; do
    tag=$(basename $lib .so)
    RELCP_LIB=$lib timeout 300 python tools/kbench.py 2000000 200 $mode > gpurun_out/kb_${mode}_${tag}.log 2>&1; echo "$mode $tag rc=$?"
    grep -h "solve" gpurun_out/kb_${mode}_${tag}.log | sed 's/(first batch).*K6/K6/'
  done
done
