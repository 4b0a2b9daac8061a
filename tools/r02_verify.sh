# HEAD verification: GPU test suite, smoke, default bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/verify_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/verify_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/verify_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/verify_bench.json 2> gpurun_out/verify_bench.err
timeout 300 python bench.py --config config1 --no-cpu > gpurun_out/verify_bench_c1.json 2> gpurun_out/verify_bench_c1.err
