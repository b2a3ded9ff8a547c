# last evidence pass of round 2 (K7 at 1 row x 3 blocks): gpu_final.sh, then ncu --set full of K6 / K7 (BB)
# and the apply kernels on the headline store, exported to CSV
bash tools/gpu_final.sh
KBENCH_PROFILE_SOLVE=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_scatter|k_lcp_iter" -s 40 -c 4 -o gpurun_out/prof_iter_r02g python tools/kbench.py 2000000 200 relaxed > gpurun_out/ncu_iter.log 2>&1; echo ncu_iter=$?
KBENCH_PROFILE_APPLY=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_scatter|k_gather" -s 4 -c 4 -o gpurun_out/prof_apply_r02g python tools/kbench.py 2000000 20 relaxed > gpurun_out/ncu_apply.log 2>&1; echo ncu_apply=$?
for n in iter apply; do
  ncu -i gpurun_out/prof_${n}_r02g.ncu-rep --page raw --csv > gpurun_out/r02_prof_${n}_relaxed_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_${n}_r02g.ncu-rep --page details --csv > gpurun_out/r02_prof_${n}_relaxed_details.csv 2>/dev/null
done
ls -la gpurun_out/*.csv
