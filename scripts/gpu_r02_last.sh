set -x
make -s -C oracle >/dev/null 2>&1
timeout 1800 python -m pytest tests/ -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu.log 2>&1; tail -2 gpurun_out/r02_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/r02_bench_cfg1.json 2> gpurun_out/bench.err; tail -c 200 gpurun_out/bench.err
