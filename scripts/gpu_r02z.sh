timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "gram or gemm" 2>&1 | tail -2
for o in "" "tc_ablate=31"; do
echo "== $o"
MPEIG_OPTS=$o timeout 600 python scripts/dense_shapes.py 2097152 48,80 f32 2>&1 >/dev/null | cut -c1-100
done
