timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -q -p no:cacheprovider -k "small_eig or golden or cfg1 or strict or modes or hl_coeffs or distribution" 2>&1 | tail -4
python scripts/chunk_exp.py 0
python bench.py --no-cpu-baseline --no-at-scale --steps 5 --warmup 3 > gpurun_out/bench_r02r.json 2>/dev/null
