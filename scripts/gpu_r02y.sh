set -x
timeout 300 python scripts/tc_gemm_one.py
timeout 600 ncu --set full --import-source on -k regex:k_gemm_tma2 -s 1 -c 1 -o gpurun_out/r02_ncu_gemm_tma2 python scripts/tc_gemm_one.py > gpurun_out/ncu_g2.log 2>&1
tail -3 gpurun_out/ncu_g2.log
