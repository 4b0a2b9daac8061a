# final verification of round 2 (after the shared-memory coarse tail)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/verify_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/verify_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/verify_smoke.log 2>&1
bash tools/r02_benchall.sh
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_vcycle_launches.csv python tools/vcycle_once.py > gpurun_out/r02_vcycle_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_vcycle_c1_launches.csv python tools/vcycle_once.py config1 > gpurun_out/r02_vcycle_c1_ncu.log 2>&1
