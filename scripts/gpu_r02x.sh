set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "gemm" 2>&1 | tail -3
timeout 600 python scripts/dense_shapes.py 2097152 48,80,192 f32 2>&1 >/dev/null | grep gemm
MPEIG_OPTS=gemm_tma2=2 timeout 600 python scripts/dense_shapes.py 2097152 48,80 f32 2>&1 >/dev/null | grep gemm
