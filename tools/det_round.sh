mkdir -p gpurun_out/det2
timeout 300 python tools/det_bisect.py 128 4 > gpurun_out/det2/default.txt 2>&1
UAAMG_NO_TAIL=1 UAAMG_NO_TMA=1 UAAMG_NO_DIR_FUSE=1 timeout 300 python tools/det_bisect.py 128 4 > gpurun_out/det2/noall.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu --durations=10 > gpurun_out/det2/pytest.txt 2>&1
