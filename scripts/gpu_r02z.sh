ABL=0 python scripts/tc_stage_dbg.py 37888 240 160 2>&1 | grep -E "correct rows|stage="
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "gemm" 2>&1 | tail -2
for o in "" tc_stage=0; do
echo "== $o"
MPEIG_OPTS=$o timeout 600 python scripts/dense_shapes.py 2097152 48,80,192 f32 2>&1 >/dev/null | grep gemm | cut -c1-110
done
