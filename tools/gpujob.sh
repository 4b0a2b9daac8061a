set -x
timeout 900 python -m pytest tests/test_3d.py tests/test_3d_wire.py tests/test_sharded_3d.py -m gpu -x -q 2>&1 | tail -2
python tools/cube_time.py 1024 wireframe
python tools/cube_time.py 512 wireframe
python bench.py --config config5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/w1025_session.csv python tools/cube_sweep_once.py 1024 wireframe 1 session > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:wblock_kernel -s 14 -c 1 -o gpurun_out/wblock_hyb_w1025 python tools/cube_sweep_once.py 1024 wireframe 1 session > gpurun_out/ncu_full_w.log 2>&1
