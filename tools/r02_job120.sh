mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_black.py tests/test_gpu_tail.py -m gpu -x -q -p no:cacheprovider > gpurun_out/j120_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/j120_pytest.log
