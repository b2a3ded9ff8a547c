mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dd.py tests/test_gpu_fullsize.py -q --timeout=600 -k "step" > gpurun_out/pytest_ddstep.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_ddstep.log
