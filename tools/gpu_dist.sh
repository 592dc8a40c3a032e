mkdir -p gpurun_out/dist2
timeout 600 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_dist.py -x -q > gpurun_out/dist2/tests.txt 2>&1
timeout 600 python bench.py --workload c2slab --steps 3 --warmup 3 > gpurun_out/dist2/c2slab_n1.json 2> gpurun_out/dist2/c2slab_n1.err
BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/dist2/c2slab_n2.json 2> gpurun_out/dist2/c2slab_n2.err
timeout 900 python bench.py --workload c4 --steps 2 --warmup 3 > gpurun_out/dist2/c4_n1.json 2> gpurun_out/dist2/c4_n1.err
timeout 900 python bench.py --workload c5 --steps 2 --warmup 3 > gpurun_out/dist2/c5_n1.json 2> gpurun_out/dist2/c5_n1.err
timeout 2400 python tests/golden/make_oracle_fixtures.py --only c5 --out gpurun_out/dist2 > gpurun_out/dist2/c5_oracle.log 2>&1
