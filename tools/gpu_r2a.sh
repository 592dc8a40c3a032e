mkdir -p gpurun_out/r2a
bash tools/l0_sweep.sh >/dev/null 2>&1 || true
timeout 300 tools/bin/l0_sweep 7 > gpurun_out/r2a/l0_sweep7.txt 2>&1
timeout 300 tools/bin/l0_sweep 27 > gpurun_out/r2a/l0_sweep27.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py -x -q --durations=10 > gpurun_out/r2a/tests.txt 2>&1
timeout 300 python tools/timeline.py 128 gpurun_out/r2a/timeline.json > gpurun_out/r2a/timeline.txt 2>&1
for w in c2slab c4 c5; do timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/r2a/$w.json 2> gpurun_out/r2a/$w.err; done
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err
