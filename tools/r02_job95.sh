mkdir -p gpurun_out
J=j95
timeout 1500 python -m pytest tests/test_gpu_minitail.py -m gpu -x -q -p no:cacheprovider > gpurun_out/${J}_mini.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_mini.log
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_gpu_minitail.py > gpurun_out/${J}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_pytest.log
