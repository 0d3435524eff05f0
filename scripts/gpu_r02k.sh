python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_r02k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02k.log
timeout 600 python scripts/dense_shapes.py 2097152 > gpurun_out/dense_shapes_2M_k.json 2> gpurun_out/dense_shapes_2M_k.log
timeout 900 python scripts/cfg_run.py cfg4 --capped 4 > gpurun_out/r02_cfg4_capped_k.json 2> gpurun_out/r02_cfg4_capped_k.log
