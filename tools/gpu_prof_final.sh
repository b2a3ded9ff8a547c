# final round-2 profiles: ncu --set full of K6 / K7 (BB) and the apply kernels on the headline store,
# and the launch list of one timed headline step
mkdir -p gpurun_out
KBENCH_PROFILE_SOLVE=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_scatter|k_lcp_iter" -s 40 -c 4 -o gpurun_out/prof_iter_r02f python tools/kbench.py 2000000 200 relaxed > gpurun_out/ncu_iter.log 2>&1; echo ncu_iter=$?
KBENCH_PROFILE_APPLY=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_scatter|k_gather" -s 4 -c 4 -o gpurun_out/prof_apply_r02f python tools/kbench.py 2000000 20 relaxed > gpurun_out/ncu_apply.log 2>&1; echo ncu_apply=$?
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-apply --no-cpu-baseline --no-literal --no-relabel"
export RELCP_PROFILE_TIMED=1
timeout 400 $CMD > gpurun_out/plain.json 2> gpurun_out/plain.err && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
unset RELCP_PROFILE_TIMED
python tools/launch_share.py gpurun_out/launches.csv > gpurun_out/launch_share.txt 2>&1; head -12 gpurun_out/launch_share.txt
