# full solves to tol 1e-10 on one GPU: 128^3 (k = 32, m = 48) and cfg4 (256^3, k = 64, m = 80)
timeout 900 python scripts/cfg_run.py lap3d128 --full --variants mplobpcg-schol --maxit 20000 > gpurun_out/r02_lap3d128_full.json 2> gpurun_out/l128.err
tail -2 gpurun_out/l128.err
timeout 3000 python scripts/cfg_run.py cfg4 --full --variants mplobpcg-schol --maxit 5000 > gpurun_out/r02_cfg4_1gpu_full.json 2> gpurun_out/cfg4full.err
tail -2 gpurun_out/cfg4full.err
