# k_gemm_tma2: correctness, accuracy, speed
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "gemm" 2>&1 | tail -5
timeout 300 python scripts/tc_acc.py 2>&1 | grep gemm
timeout 600 python scripts/dense_shapes.py 2097152 2>&1 >/dev/null | grep "f32" | grep gemm
timeout 600 python -m pytest tests/test_gpu_solver.py -q -p no:cacheprovider -x -k "tensor_core or large_block or wide_block" 2>&1 | tail -3
