mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/j8_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j8_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j8_smoke.log 2>&1
python bench.py > gpurun_out/j8_bench.json 2> gpurun_out/j8_bench.err
