python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke10.log 2>&1
python bench.py > gpurun_out/b10_c3.json 2> gpurun_out/b10_c3.err
python bench.py --config config1 > gpurun_out/b10_c1.json 2>&1
python bench.py --config config2 > gpurun_out/b10_c2.json 2>&1
python bench.py --config config4 --steps 10 --warmup 3 > gpurun_out/b10_c4.json 2>&1
python bench.py --config config5 --steps 3 --warmup 3 > gpurun_out/b10_c5.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/cycle_norm10.csv python tools/profile_session.py --cycles 1 --sweeps 0 > /dev/null 2>&1
