# A/B: legk_time.py under each library variant given as arguments
mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v" >> gpurun_out/${J}_ab.log
  TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_$v.so timeout 300 python tools/legk_time.py >> gpurun_out/${J}_ab.log 2>&1
done
