# round-2 bench evidence: default bench line, reference arm, ncu launch list of the bench command
set -x
make -s -C oracle >/dev/null 2>&1
timeout 1200 python bench.py > gpurun_out/r02_bench_cfg1.json 2> gpurun_out/bench.err; tail -c 400 gpurun_out/bench.err
timeout 1200 python bench.py --impl reference > gpurun_out/r02_bench_reference_cfg1.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/bench_ref.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_ncu_launches_bench.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-at-scale > gpurun_out/ncu_bench.log 2>&1; tail -2 gpurun_out/ncu_bench.log
