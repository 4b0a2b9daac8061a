mkdir -p gpurun_out
J=j114
for v in main rcp3leg main rcp3leg; do
  if [ $v = main ]; then L=paper_2110_08389_b200/libtmg_b200.so; else L=paper_2110_08389_b200/libtmg_b200_$v.so; fi
  echo "== $v" >> gpurun_out/${J}.log
  TMG_LIB_PATH=$L timeout 300 python tools/legk_time.py >> gpurun_out/${J}.log 2>&1
done
run() { echo "== $1 | $2" >> gpurun_out/${J}.log; env $2 timeout 300 python bench.py --config $1 --no-cpu --no-solve 2>gpurun_out/${J}_err.log | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d.get('kernels_per_cycle'))" >> gpurun_out/${J}.log 2>&1; }
for v in main rcp3mini main rcp3mini; do
  if [ $v = main ]; then L=paper_2110_08389_b200/libtmg_b200.so; else L=paper_2110_08389_b200/libtmg_b200_$v.so; fi
  run config1 "TMG_LIB_PATH=$L"
done
echo "== pytest legk with rcp3leg" >> gpurun_out/${J}.log
TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_rcp3leg.so timeout 900 python -m pytest tests/test_gpu_legk.py tests/test_gpu_golden.py -m gpu -x -q -p no:cacheprovider >> gpurun_out/${J}.log 2>&1
