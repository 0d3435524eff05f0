for o in gram_tma=1 gram_tma=2; do
echo "== $o"
MPEIG_OPTS=$o timeout 300 python scripts/tc_acc.py 2>&1 | grep gram
MPEIG_OPTS=$o timeout 600 python scripts/dense_shapes.py 2097152 16,48,80,192 f32 2>&1 >/dev/null | grep gram | cut -c1-105
done
