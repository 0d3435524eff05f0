mkdir -p gpurun_out
python scripts/tc_probe.py 2097152 240 240 1 && \
ncu --set full --clock-control none -k regex:k_gram_tc -c 1 -o gpurun_out/tc_gram240 -f python scripts/tc_probe.py 2097152 240 240 1 > gpurun_out/ncu_tc.log 2>&1
echo rc=$?
