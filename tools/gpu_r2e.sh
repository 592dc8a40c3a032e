mkdir -p gpurun_out/r2e
timeout 300 python tools/timeline.py 128 gpurun_out/r2e/timeline.json > gpurun_out/r2e/timeline.txt 2>&1
UAAMG_TAIL_PROF=1 timeout 300 python tools/one_solve.py > gpurun_out/r2e/tailprof.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2e/bench.json 2> gpurun_out/r2e/bench.err
UAAMG_NO_DIR_CLUSTER=1 timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2e/bench_nocl.json 2> gpurun_out/r2e/bench_nocl.err
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r2e/tests.txt 2>&1
