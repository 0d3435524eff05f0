for np in 8 4 2 1; do
echo "== nprod $np"
MPEIG_OPTS=tc_ablate=31,tc_nprod=$np timeout 600 python scripts/dense_shapes.py 2097152 80 f32 2>&1 >/dev/null | grep gemm | cut -c1-100
done
