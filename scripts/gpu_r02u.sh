timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "tensor_cores or gemm" 2>&1 | tail -3
timeout 300 python scripts/tc_acc.py 2>&1 | grep gemm
timeout 300 python -m pytest tests/test_gpu_solver.py -q -p no:cacheprovider -x -k "tensor_core" 2>&1 | tail -2
timeout 600 python scripts/dense_shapes.py 2097152 2>&1 >/dev/null | grep "f32" | grep gemm
timeout 300 python scripts/dense_ax_bench.py 16384 96
