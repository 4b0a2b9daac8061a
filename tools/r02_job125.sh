mkdir -p gpurun_out
J=j125
timeout 1200 python -m pytest tests/test_gpu_black.py tests/test_gpu_golden.py -m gpu -x -q -p no:cacheprovider > gpurun_out/${J}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_pytest.log
for c in config1 config2 config3 config3_v11; do
  x=""; if [ $c = config3_v11 ]; then x="--nu 1"; fi
  timeout 900 python bench.py --config ${c%_v11} $x > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err
done
