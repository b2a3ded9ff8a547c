mkdir -p gpurun_out
timeout 1500 python tools/relax_probe.py 2000000 50 20000 > gpurun_out/relax_2m.log 2>&1; echo relax_rc=$?
