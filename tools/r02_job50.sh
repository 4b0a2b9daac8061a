mkdir -p gpurun_out
J=j50
timeout 300 python tests/legk_worker.py default > gpurun_out/${J}_default.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_default.log
TMG_LEGK_NMIN=16 timeout 300 python tests/legk_worker.py small > gpurun_out/${J}_small.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_small.log
TMG_LEGK_NMIN=16 TMG_LEGK_K0=9 timeout 300 python tests/legk_worker.py small > gpurun_out/${J}_small9.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_small9.log
timeout 300 python tests/legk_worker.py split > gpurun_out/${J}_split.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_split.log
timeout 900 python -m pytest tests/test_sharded.py -q -p no:cacheprovider -m gpu -k "partial" > gpurun_out/${J}_sharded.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_sharded.log
timeout 300 python tools/legk_time.py > gpurun_out/${J}_time1.log 2>&1
