mkdir -p gpurun_out
J=j90
for v in nobpf main nobpf main; do
  if [ $v = main ]; then L=paper_2110_08389_b200/libtmg_b200.so; else L=paper_2110_08389_b200/libtmg_b200_$v.so; fi
  echo "== $v" >> gpurun_out/${J}_ab.log
  TMG_LIB_PATH=$L timeout 300 python tools/legk_time.py >> gpurun_out/${J}_ab.log 2>&1
done
echo "== pytest legk" >> gpurun_out/${J}_ab.log
timeout 900 python -m pytest tests/test_gpu_legk.py tests/test_tridiag.py -m gpu -x -q -p no:cacheprovider >> gpurun_out/${J}_ab.log 2>&1
