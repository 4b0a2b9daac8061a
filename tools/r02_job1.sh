# round 2, job 1: full GPU suite with the new parity tests, smoke, both bench
# arms on config 3, compute-sanitizer memcheck on the small-grid workload
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/j1_gpu.txt 2>&1
free -g >> gpurun_out/j1_gpu.txt; nproc >> gpurun_out/j1_gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/j1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j1_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j1_smoke.log 2>&1
python bench.py > gpurun_out/j1_bench.json 2> gpurun_out/j1_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/j1_bench_ref.json 2> gpurun_out/j1_bench_ref.err
timeout 1500 compute-sanitizer --tool memcheck --target-processes all --leak-check no --log-file gpurun_out/j1_memcheck.%p.log python tools/sanitize_run.py all > gpurun_out/j1_memcheck_out.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/j1_memcheck_out.log
timeout 1200 compute-sanitizer --tool synccheck --target-processes all --log-file gpurun_out/j1_synccheck.%p.log python tools/sanitize_run.py all > gpurun_out/j1_synccheck_out.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/j1_synccheck_out.log
timeout 1500 compute-sanitizer --tool racecheck --target-processes all --log-file gpurun_out/j1_racecheck.%p.log python tools/sanitize_run.py all > gpurun_out/j1_racecheck_out.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/j1_racecheck_out.log
