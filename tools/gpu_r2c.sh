mkdir -p gpurun_out
timeout 900 python tools/relax_probe.py 2000000 0 20000 > gpurun_out/relax_2m_r0.log 2>&1; echo relax0_rc=$?
timeout 600 python tools/relax_probe.py 2000000 2 3000 > gpurun_out/relax_2m_r2.log 2>&1; echo relax2_rc=$?
