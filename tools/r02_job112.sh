mkdir -p gpurun_out
J=j112
run() { echo "== $1 | $2" >> gpurun_out/${J}.log; env $2 timeout 300 python bench.py --config $1 --no-cpu --no-solve 2>gpurun_out/${J}_err.log | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d.get('kernels_per_cycle'))" >> gpurun_out/${J}.log 2>&1; }
for v in main mt384 mt640 mt768 main mt640; do
  if [ $v = main ]; then L=paper_2110_08389_b200/libtmg_b200.so; else L=paper_2110_08389_b200/libtmg_b200_$v.so; fi
  run config1 "TMG_LIB_PATH=$L"
done
