mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dd.py -q --timeout=600 > gpurun_out/pytest_jds2.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_jds2.log
