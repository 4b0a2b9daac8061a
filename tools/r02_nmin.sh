mkdir -p gpurun_out
for nm in 512 256 128 64 32; do
  echo "== NMIN $nm" >> gpurun_out/j35.log
  TMG_LEGK_NMIN=$nm timeout 300 python tools/legk_time.py >> gpurun_out/j35.log 2>&1
  TMG_LEGK_NMIN=$nm timeout 300 python tools/legk_time.py config2 >> gpurun_out/j35.log 2>&1
  TMG_LEGK_NMIN=$nm timeout 300 python tools/legk_time.py config1 >> gpurun_out/j35.log 2>&1
done
