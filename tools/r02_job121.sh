mkdir -p gpurun_out
J=j121
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${J}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_pytest.log
for v in 0 1 0 1; do
  echo "== restrict black-zero $v" >> gpurun_out/${J}.log
  TMG_RESTRICT_BLACK=$v timeout 300 python tools/legk_time.py >> gpurun_out/${J}.log 2>&1
done
for c in config1 config3; do for v in 0 1; do
  echo "== $c black-zero $v" >> gpurun_out/${J}.log
  TMG_RESTRICT_BLACK=$v timeout 600 python bench.py --config $c --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['solve']['ms'], d['solve']['cycles'], d['solve']['final_rel_defect'], d['solve'].get('asymptotic_ratio'))" >> gpurun_out/${J}.log 2>&1
done; done
