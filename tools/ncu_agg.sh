# ncu full capture of the level-0 cooperative aggregation kernel (one C2 setup)
OUT=${1:-gpurun_out/aggncu}; mkdir -p $OUT
timeout 900 ncu --set full --warp-sampling-interval 2 --clock-control none --import-source on \
  --kernel-name-base demangled -k "regex:k_aggregate_coop" -c 1 -o $OUT/prof_agg python tools/one_solve.py > $OUT/ncu_agg.log 2>&1
echo "agg rc=$?" >> $OUT/status.txt
