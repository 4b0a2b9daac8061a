mkdir -p gpurun_out
J=j91
run() { echo "== $1 | $2" >> gpurun_out/${J}.log; env $2 timeout 300 python bench.py --config $1 --no-cpu --no-solve 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d.get('kernels_per_cycle'))" >> gpurun_out/${J}.log 2>&1; }
for c in config1 config2; do
  run $c "TMG_TAIL=0"
  run $c "TMG_TAIL=1"
  for n in 8 16 32 64; do
    run $c "TMG_TAIL=1 TMG_TAIL_NMAX=$n"
    run $c "TMG_TAIL=1 TMG_TAIL_NMAX=$n TMG_TAIL_CTAS=1"
    run $c "TMG_TAIL=1 TMG_TAIL_NMAX=$n TMG_TAIL_CTAS=4"
  done
done
