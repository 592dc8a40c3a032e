# ncu captures of the level-4 (deepest) solve kernels of one C2 solve:
# full sections, warm caches, dense stall sampling.  Usage: bash tools/ncu_l4.sh [outdir]
OUT=${1:-gpurun_out/l4}; mkdir -p $OUT
for spec in "k_dir_update:0:dir" "k_csr_group<.*EpiResidSum:0:rsum" "k_csr_group<.*SrcUp.*EpiSweepBeta:0:sbeta"; do
  IFS=: read pat skip tag <<< "$spec"
  timeout 600 ncu --set full --warp-sampling-interval 0 --clock-control none --cache-control none --import-source on \
    --kernel-name-base demangled -k "regex:$pat" -s $skip -c 1 -o $OUT/prof_$tag python tools/one_solve.py > $OUT/ncu_$tag.log 2>&1
  echo "$tag rc=$?" >> $OUT/status.txt
done
