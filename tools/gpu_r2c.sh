mkdir -p gpurun_out/r2c
timeout 600 python -m pytest tests/test_gpu_reshape.py -q > gpurun_out/r2c/reshape.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu --durations=10 > gpurun_out/r2c/all.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c/smoke.txt 2>&1
