#!/bin/bash
# Round-2 final evidence run (one gpurun session, from the repo root on the
# GPU box): smoke, every GPU test, bench (ours + reference arm), the ncu launch
# list of one C2 setup + solve, ncu --set full of the level-0 kernels at C2
# and of the 27-point direction kernel at C4, the configs lines and the
# partitioned workloads at N = 1.   Usage: bash tools/gpu_r2final.sh [tag] [stages]
TAG=${1:-r2final}
STAGES=${2:-"smoke tests bench benchref ncu ncufull ncuc4 configs part"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt
for st in $STAGES; do
  case $st in
    smoke) timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/status.txt ;;
    tests) timeout 2400 python -m pytest tests -q -m gpu --durations=20 > $OUT/pytest_gpu.log 2>&1; echo "tests rc=$?" >> $OUT/status.txt ;;
    bench) timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status.txt ;;
    benchref) timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "benchref rc=$?" >> $OUT/status.txt ;;
    ncu) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
           python tools/one_solve.py > $OUT/ncu_launches.log 2>&1; echo "ncu rc=$?" >> $OUT/status.txt ;;
    ncufull) timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
           -k "regex:k_csr_tma_rows" --launch-skip 30 -c 3 -o $OUT/l0_c2 python tools/one_solve.py > $OUT/ncufull.log 2>&1
           echo "ncufull rc=$?" >> $OUT/status.txt ;;
    ncuc4) ONE_SOLVE_N=256 ONE_SOLVE_STENCIL=27 timeout 1200 ncu --set full --clock-control none --import-source on \
           --kernel-name-base demangled -k "regex:k_ell<.*Epi" -c 3 -o $OUT/l0_c4 python tools/one_solve.py \
           > $OUT/ncuc4.log 2>&1; echo "ncuc4 rc=$?" >> $OUT/status.txt ;;
    configs) timeout 1500 python tools/configs_bench.py C1 C3 C4 C5 > $OUT/configs.jsonl 2> $OUT/configs.err; echo "configs rc=$?" >> $OUT/status.txt ;;
    part) for w in c2slab c4 c5; do timeout 900 python bench.py --workload $w > $OUT/part_$w.json 2> $OUT/part_$w.err; echo "part $w rc=$?" >> $OUT/status.txt; done ;;
  esac
done
