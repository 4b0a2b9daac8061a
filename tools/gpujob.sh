set -x
python bench.py --config config5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:wblock_kernel -s 12 -c 1 -o gpurun_out/wblock_hyb_w1025 python tools/cube_sweep_once.py 1024 wireframe 1 session > gpurun_out/ncu_full_w.log 2>&1
ls -la gpurun_out/
