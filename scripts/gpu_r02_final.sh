# round-2 final evidence: GPU suite, smoke, bench (ours + reference), launch lists of both stages
set -x
make -s -C oracle >/dev/null 2>&1
timeout 1800 python -m pytest tests/ -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu.log 2>&1; tail -3 gpurun_out/r02_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 1500 python bench.py > gpurun_out/r02_bench_cfg1.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.err
timeout 1500 python bench.py --impl reference > gpurun_out/r02_bench_reference_cfg1.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/bench_ref.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_ncu_launches_bench.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-at-scale > gpurun_out/ncu_bench.log 2>&1; tail -1 gpurun_out/ncu_bench.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 14000 -c 3000 --csv --log-file gpurun_out/r02_ncu_launches_bench_stage2.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-at-scale > gpurun_out/ncu_bench2.log 2>&1; tail -1 gpurun_out/ncu_bench2.log
