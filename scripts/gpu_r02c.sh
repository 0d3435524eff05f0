mkdir -p gpurun_out
timeout 600 python scripts/dense_shapes.py 2097152 > gpurun_out/dense_shapes_2M.json 2> gpurun_out/dense_shapes_2M.log
timeout 600 python scripts/dense_shapes.py 16777216 > gpurun_out/dense_shapes_16M.json 2> gpurun_out/dense_shapes_16M.log
timeout 900 python scripts/cfg_run.py cfg4 --capped 4 > gpurun_out/r02_cfg4_capped.json 2> gpurun_out/r02_cfg4_capped.log
