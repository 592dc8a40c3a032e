#!/bin/bash
# One gpurun session: smoke, GPU parity tests, bench, ncu launch list + one full capture.
# Usage (from the repo root, on the GPU box): bash tools/gpu_round.sh [tag] [stages]
TAG=${1:-r1}
STAGES=${2:-"smoke tests bench ncu"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu | head -20 >> $OUT/nproc.txt
for st in $STAGES; do
  case $st in
    smoke) timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/status.txt ;;
    tests) timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "tests rc=$?" >> $OUT/status.txt ;;
    testsk) timeout 1500 python -m pytest tests -q -m gpu --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "tests rc=$?" >> $OUT/status.txt ;;
    bench) timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status.txt ;;
    benchref) timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "benchref rc=$?" >> $OUT/status.txt ;;
    ncu) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
           python tools/one_solve.py > $OUT/ncu_launches.log 2>&1; echo "ncu rc=$?" >> $OUT/status.txt ;;
    ncufull)
      # level-0 hot kernels of iteration 1 (TMA tile kernels): residual (first
      # SrcVec/EpiResid TMA launch), post-sweep (2nd EpiSweepBeta TMA launch:
      # the level-1 FCG step 2 precedes it), NPCG direction SpMV
      for spec in "k_csr_tma<.*SrcVec.*EpiResid:0:resid" "k_csr_tma<.*SrcVec.*EpiSweepBeta:1:sweep" "k_csr_tma<.*EpiDirNpcg:0:dir"; do
        IFS=: read pat skip tag <<< "$spec"
        timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
          -k "regex:$pat" -s $skip -c 1 -o $OUT/prof_$tag python tools/one_solve.py > $OUT/ncu_full_$tag.log 2>&1
        echo "ncufull $tag rc=$?" >> $OUT/status.txt
      done ;;
  esac
done
