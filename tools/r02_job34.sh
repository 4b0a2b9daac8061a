mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j34_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j34_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j34_smoke.log 2>&1
python bench.py > gpurun_out/j34_bench.json 2> gpurun_out/j34_bench.err
bash tools/r02_check.sh
