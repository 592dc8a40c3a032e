# ncu full capture of one k_tail launch (warm caches, dense warp sampling)
OUT=${1:-gpurun_out/tailncu}; mkdir -p $OUT
timeout 600 ncu --set full --warp-sampling-interval 0 --clock-control none --cache-control none --import-source on \
  --kernel-name-base demangled -k "regex:k_tail" -s 20 -c 1 -o $OUT/prof_tail python tools/one_solve.py > $OUT/ncu_tail.log 2>&1
echo "tail rc=$?" >> $OUT/status.txt
