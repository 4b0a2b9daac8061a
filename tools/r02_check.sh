# bounds-checked library (make check) over the small-grid workload, the leg
# kernel's tiny / default / split cases and the GPU parity suites
mkdir -p gpurun_out
export TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_check.so
O=gpurun_out/boundscheck.log
echo "library: $TMG_LIB_PATH" > $O
nvidia-smi --query-gpu=name,driver_version --format=csv,noheader >> $O
for args in "all" ; do
  echo "== sanitize_run.py $args" >> $O
  timeout 900 python tools/sanitize_run.py $args >> $O 2>&1; echo "rc=$?" >> $O
done
echo "== sanitize_run.py 2d with the leg kernel on every tweed level (TMG_LEGK_NMIN=16, K0=3)" >> $O
TMG_LEGK_NMIN=16 TMG_LEGK_K0=3 timeout 900 python tools/sanitize_run.py 2d >> $O 2>&1; echo "rc=$?" >> $O
for w in default split; do
  echo "== legk_worker $w" >> $O
  timeout 600 python tests/legk_worker.py $w >> $O 2>&1; echo "rc=$?" >> $O
done
echo "== legk_worker small (NMIN=16, K0=3)" >> $O
TMG_LEGK_NMIN=16 TMG_LEGK_K0=3 timeout 600 python tests/legk_worker.py small >> $O 2>&1; echo "rc=$?" >> $O
echo "== pytest gpu parity / hybrid / golden / plans (checked library)" >> $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hybrid.py tests/test_gpu_golden.py tests/test_gpu_plans.py -q -p no:cacheprovider >> $O 2>&1; echo "rc=$?" >> $O
echo "== minitail_worker (shared-memory coarse tail, checked library)" >> $O
timeout 900 python tests/minitail_worker.py >> $O 2>&1; echo "rc=$?" >> $O
echo "== minitail_worker TMG_MINI_UNIT=128" >> $O
TMG_MINI_UNIT=128 timeout 900 python tests/minitail_worker.py >> $O 2>&1; echo "rc=$?" >> $O
