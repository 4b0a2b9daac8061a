# round 2: every BASELINE configuration through bench.py (ours), config 3
# V(1,1) too, and the reference arm of config 3
mkdir -p gpurun_out
for c in config1 config2 config3 config4 config5; do
  timeout 900 python bench.py --config $c > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err
done
timeout 900 python bench.py --config config3 --nu 1 --no-cpu > gpurun_out/r02_bench_config3_v11.json 2> gpurun_out/r02_bench_config3_v11.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err
