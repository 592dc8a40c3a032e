mkdir -p gpurun_out/dist
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q --durations=8 > gpurun_out/dist/sharded.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/dist/dist.txt 2>&1
