for o in "" gram_l2promo=0 gram_l2promo=1 gram_l2promo=2; do
echo "== $o"
MPEIG_OPTS=$o timeout 600 python scripts/dense_shapes.py 2097152 48,80,192 f32 2>&1 >/dev/null | grep gram | cut -c1-100
done
for p in 0 1; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_gram_tma -s 1 -c 1 env MPEIG_OPTS=gram_l2promo=$p python scripts/tc_gram_one.py 2>&1 | grep -E "dram__bytes|duration"
done
