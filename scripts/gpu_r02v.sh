# refresh of the round-2 per-configuration numbers after the TMA-fed tensor-core kernels
set -x
make -s -C oracle >/dev/null 2>&1
timeout 600 python scripts/dense_shapes.py 2097152 > gpurun_out/r02_dense_shapes_2M.json 2> gpurun_out/r02_dense_shapes_2M.err
timeout 900 python scripts/cfg_run.py cfg4 --capped 4 > gpurun_out/r02_cfg4_1gpu_capped.json 2> gpurun_out/cfg4.err
timeout 900 python scripts/cfg_run.py cfg5 --capped 3 > gpurun_out/r02_cfg5_1gpu_capped.json 2> gpurun_out/cfg5.err
timeout 900 python scripts/cfg_run.py cfg2 --capped 40 --pinvit 40 > gpurun_out/r02_cfg2_capped.json 2> gpurun_out/cfg2.err
timeout 600 python scripts/one_solve.py > gpurun_out/one_solve.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 30000 -c 1500 --csv --log-file gpurun_out/r02_ncu_launches_cfg1_warm.csv python scripts/one_solve.py > gpurun_out/ncu1.log 2>&1
tail -c 600 gpurun_out/*.err
cat gpurun_out/r02_cfg4_1gpu_capped.json | head -c 1500
