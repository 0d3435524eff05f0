set -x
make -s -C oracle >/dev/null 2>&1
timeout 1500 python bench.py > gpurun_out/r02_bench_cfg1.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.err
