mkdir -p gpurun_out
J=j62
timeout 600 python -m pytest tests/test_gpu_transfers.py -q -p no:cacheprovider -x > gpurun_out/${J}_tr.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_tr.log
for v in v2 v3; do
  if [ $v = v2 ]; then export TMG_RESTRICT=v2; else unset TMG_RESTRICT; fi
  echo "== $v" >> gpurun_out/${J}_time.log
  timeout 300 python tools/transfer_time.py --tag $v >> gpurun_out/${J}_time.log 2>&1
  timeout 300 python tools/legk_time.py >> gpurun_out/${J}_time.log 2>&1
done
unset TMG_RESTRICT
ncu --set full --import-source on --clock-control none -k regex:restrict3 -c 1 -o gpurun_out/${J}_r3 python tools/transfer_time.py > gpurun_out/${J}_ncu.log 2>&1
