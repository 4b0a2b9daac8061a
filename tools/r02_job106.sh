mkdir -p gpurun_out
J=j106
timeout 1500 python -m pytest tests/test_gpu_transfers.py tests/test_gpu_hybrid.py tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_tail.py tests/test_gpu_minitail.py -m gpu -x -q -p no:cacheprovider > gpurun_out/${J}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_pytest.log
for c in config1 config2 config3; do
  timeout 900 python bench.py --config $c --no-cpu > gpurun_out/${J}_bench_$c.json 2> gpurun_out/${J}_bench_$c.err
done
