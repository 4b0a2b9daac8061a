mkdir -p gpurun_out
J=j60
timeout 600 python -m pytest tests/test_gpu_transfers.py -q -p no:cacheprovider -x > gpurun_out/${J}_tr.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_tr.log
timeout 900 python -m pytest tests/test_sharded.py -q -p no:cacheprovider -m gpu -k "partial" > gpurun_out/${J}_sharded.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_sharded.log
for v in v2 v3 v2 v3; do
  if [ $v = v2 ]; then export TMG_RESTRICT=v2; else unset TMG_RESTRICT; fi
  echo "== $v" >> gpurun_out/${J}_time.log
  timeout 300 python tools/transfer_time.py --tag $v >> gpurun_out/${J}_time.log 2>&1
  timeout 300 python tools/legk_time.py >> gpurun_out/${J}_time.log 2>&1
done
unset TMG_RESTRICT
timeout 300 python tests/legk_worker.py default > gpurun_out/${J}_default.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_default.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum --clock-control none -k regex:restrict -c 12 --csv python tools/transfer_time.py > gpurun_out/${J}_ncu.csv 2>&1
