set -x
timeout 1800 python -m pytest tests/ -m gpu -q -p no:cacheprovider 2>&1 | tail -4
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemm_tma2 -s 1 -c 1 -o gpurun_out/r02_ncu_gemm_tma2_final python scripts/tc_gemm_one.py > gpurun_out/ncu_g2f.log 2>&1; tail -1 gpurun_out/ncu_g2f.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gram_tma -s 1 -c 1 -o gpurun_out/r02_ncu_gram_tma_final python scripts/tc_gram_one.py > gpurun_out/ncu_gtf.log 2>&1; tail -1 gpurun_out/ncu_gtf.log
