# new K6 default (9 blocks x 4 warps, 56 regs for the 32-body kernel): parity files, then A/B against 8 / 10 blocks, JDS at 9
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dd.py tests/test_gpu_edge.py -m gpu -q -x > gpurun_out/k6new_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/k6new_tests.log
bash tools/gpu_k7shape.sh "$@"
