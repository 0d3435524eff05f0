timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "tensor_cores or gram or gemm" 2>&1 | tail -15
timeout 600 python scripts/dense_shapes.py 2097152 2>&1 >/dev/null | grep f32
