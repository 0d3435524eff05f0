mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "tensor_cores or gram" > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
timeout 600 python scripts/dense_shapes.py 2097152 > gpurun_out/dense_shapes_2M_c.json 2> gpurun_out/dense_shapes_2M_c.log
