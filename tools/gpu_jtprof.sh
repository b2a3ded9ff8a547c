# JDS K6: full parity file, then an ncu --set full capture of the tiled JDS scatter and the CSR scatter
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q --timeout=400 > gpurun_out/pytest_parity.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_parity.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_scatter_jt" -s 20 -c 2 -o gpurun_out/prof_jt python tools/kbench.py 2000000 100 > gpurun_out/ncu_jt.log 2>&1; echo ncu_jt=$?
RELCP_LAYOUT=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_scatter" -s 20 -c 2 -o gpurun_out/prof_csr python tools/kbench.py 2000000 100 > gpurun_out/ncu_csr.log 2>&1; echo ncu_csr=$?
