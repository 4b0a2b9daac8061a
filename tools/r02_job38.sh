mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_transfers.py -q -x -p no:cacheprovider > gpurun_out/j38_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/j38_pytest.log
for v in v2 default v2 default; do echo "== $v" >> gpurun_out/j38_time.log; TMG_RESTRICT=$v timeout 300 python tools/legk_time.py >> gpurun_out/j38_time.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/j38_launches.csv python tools/vcycle_once.py > gpurun_out/j38_ncu.log 2>&1
