timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "gram or gemm" 2>&1 | tail -2
timeout 300 python scripts/tc_acc.py 2>&1 | grep gram
timeout 600 python scripts/dense_shapes.py 2097152 48,80,192 f32 2>&1 >/dev/null | grep gram | cut -c1-110
