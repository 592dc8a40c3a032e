mkdir -p gpurun_out/r2f
for k in 1 2; do
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2f/bench_$k.json 2> gpurun_out/r2f/bench_$k.err
UAAMG_NO_L2HINT=1 timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2f/bench_nohint_$k.json 2> gpurun_out/r2f/bench_nohint_$k.err
done
