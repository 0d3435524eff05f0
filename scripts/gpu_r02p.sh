timeout 600 python scripts/dense_shapes.py 2097152 > gpurun_out/r02_dense_shapes_2M.json 2> /dev/null
ncu --set full --clock-control none --import-source on -k regex:k_gram_tc -c 1 -o gpurun_out/r02_ncu_tc_gram240 -f python scripts/tc_probe.py 2097152 240 240 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gram_dmma -c 1 -o gpurun_out/r02_ncu_dmma_gram240 -f python scripts/dense_shapes.py 2097152 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_csr_spmm -c 1 -o gpurun_out/r02_ncu_spmm -f python scripts/spmm_bw.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stencil7 -c 1 -o gpurun_out/r02_ncu_stencil -f python scripts/cfg_run.py cfg4_half --capped 1 --variants dlobpcg-dchol > /dev/null 2>&1
echo done
