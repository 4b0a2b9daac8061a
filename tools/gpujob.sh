set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --config config4 --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --config config5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python bench.py --config config1 --steps 20 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python bench.py --config config2 --steps 20 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/t257_sweep3.csv python tools/cube_sweep_once.py 256 tweed 1 session > /dev/null 2>&1
