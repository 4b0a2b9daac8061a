set -x
timeout 900 python -m pytest tests/test_3d_wire.py -m gpu -x -q 2>&1 | tail -3
python tools/cube_time.py 1024 wireframe
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/w1025_launches7.csv python tools/cube_sweep_once.py 1024 wireframe 1 > gpurun_out/ncu_w.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:wblock_kernel -s 6 -c 1 -o gpurun_out/wblock_w1025 python tools/cube_sweep_once.py 1024 wireframe 1 > gpurun_out/ncu_full_w.log 2>&1
