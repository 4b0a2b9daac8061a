mkdir -p gpurun_out
J=j107
for v in main hb6; do
  if [ $v = main ]; then L=paper_2110_08389_b200/libtmg_b200.so; else L=paper_2110_08389_b200/libtmg_b200_$v.so; fi
  TMG_LIB_PATH=$L timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${J}_$v.csv python tools/cube_cycle_once.py 1024 wireframe > gpurun_out/${J}_$v.log 2>&1
done
