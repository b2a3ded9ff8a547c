# SNSD register-budget variants: generation time on cfg5 A_0 (literal) and the relaxed state
mkdir -p gpurun_out
for lib in "$@"; do
  tag=$(basename $lib .so)
  for mode in a0 relaxed; do
    RELCP_LIB=$lib timeout 300 python tools/kbench.py 2000000 5 $mode > gpurun_out/s_${mode}_$tag.log 2>&1; echo "$mode $tag rc=$?"; grep generate gpurun_out/s_${mode}_$tag.log
  done
done
