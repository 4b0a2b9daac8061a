mkdir -p gpurun_out
J=j119
timeout 900 python tools/dbg_black.py > gpurun_out/${J}_dbg.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${J}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_pytest.log
timeout 900 python bench.py > gpurun_out/${J}_bench_config3.json 2> gpurun_out/${J}_bench_config3.err
