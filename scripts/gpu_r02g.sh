mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "tensor_cores or gram" > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
timeout 600 python scripts/dense_shapes.py 2097152 > gpurun_out/dense_shapes_2M_d.json 2> gpurun_out/dense_shapes_2M_d.log
ncu --set full --clock-control none -k regex:k_gram_tc -c 1 -o gpurun_out/tc_gram240b -f python scripts/tc_probe.py 2097152 240 240 1 > gpurun_out/ncu_tc.log 2>&1
