nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv
for o in gemm_tma2=0 "" gemm_tma2=0 ""; do
echo "== $o"
MPEIG_OPTS=$o timeout 600 python scripts/dense_shapes.py 2097152 48,80,192 f32 2>&1 >/dev/null | grep gemm | cut -c1-110
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv
