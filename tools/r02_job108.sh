mkdir -p gpurun_out
J=j108
for n in 512 1024 2048 256; do
  echo "== NMIN $n" >> gpurun_out/${J}.log
  TMG_LEGK_NMIN=$n timeout 300 python tools/legk_time.py >> gpurun_out/${J}.log 2>&1
done
