python bench.py --no-cpu-baseline --no-at-scale --steps 5 --warmup 3 > gpurun_out/bench_r02o.json 2> gpurun_out/bench_r02o.log
python -m pytest tests/test_gpu_solver.py -q -p no:cacheprovider -x -k "golden or cfg1 or bitwise or modes" 2>&1 | tail -2
