set -x
nproc
timeout 900 python -m pytest tests/test_gpu_spchol.py -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python scripts/sparse_cfg1.py > gpurun_out/r02_sparse_cfg1.json 2> gpurun_out/sp.err; tail -5 gpurun_out/sp.err
