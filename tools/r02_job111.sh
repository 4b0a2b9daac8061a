mkdir -p gpurun_out
J=j111
timeout 1500 python -m pytest tests/test_gpu_minitail.py tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -x -q -p no:cacheprovider > gpurun_out/${J}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_pytest.log
run() { echo "== $1 | $2" >> gpurun_out/${J}.log; env $2 timeout 300 python bench.py --config $1 --no-cpu 2>gpurun_out/${J}_err.log | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d.get('kernels_per_cycle'), d['solve']['ms'], d['solve']['cycles'], d['solve']['final_rel_defect'])" >> gpurun_out/${J}.log 2>&1; }
for c in config1 config2 config1; do
  run $c "TMG_MINI=1"
done
