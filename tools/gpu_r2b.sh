mkdir -p gpurun_out/r2b
bash tools/l0_sweep.sh >/dev/null 2>&1 || true
timeout 300 tools/bin/l0_sweep 7 > gpurun_out/r2b/l0_sweep7.txt 2>&1
timeout 300 tools/bin/l0_sweep 27 > gpurun_out/r2b/l0_sweep27.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_fullsize.py -x -q -k "not c3 and not c5_sharded" --durations=5 > gpurun_out/r2b/tests.txt 2>&1
timeout 300 python tools/e2e_io.py > gpurun_out/r2b/e2e_io.txt 2>&1
timeout 900 python tools/configs_bench.py C1 C4 C3 C5 > gpurun_out/r2b/configs.jsonl 2> gpurun_out/r2b/configs.err
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2b/bench.json 2> gpurun_out/r2b/bench.err
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 > gpurun_out/r2b/c4.json 2> gpurun_out/r2b/c4.err
