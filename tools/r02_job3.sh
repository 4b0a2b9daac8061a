# round 2, job 3: leg-kernel parity (each under its own timeout) and A/B timing
mkdir -p gpurun_out
timeout 300 python tests/legk_worker.py default > gpurun_out/j3_default.log 2>&1; echo "rc=$?" >> gpurun_out/j3_default.log
TMG_LEGK_NMIN=16 TMG_LEGK_K0=3 timeout 300 python tests/legk_worker.py small > gpurun_out/j3_small.log 2>&1; echo "rc=$?" >> gpurun_out/j3_small.log
timeout 300 python tests/legk_worker.py split > gpurun_out/j3_split.log 2>&1; echo "rc=$?" >> gpurun_out/j3_split.log
timeout 300 python tools/legk_time.py > gpurun_out/j3_time1.log 2>&1
TMG_LEGK=0 timeout 300 python tools/legk_time.py > gpurun_out/j3_time0.log 2>&1
