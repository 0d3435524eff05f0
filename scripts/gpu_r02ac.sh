set -x
timeout 600 python scripts/dense_ax_bench.py 16384 96 > gpurun_out/r02_dense_ax.json 2> gpurun_out/dax.err; tail -5 gpurun_out/dax.err
timeout 900 python scripts/cfg3_dense.py > gpurun_out/r02_cfg3_dense.json 2> gpurun_out/cfg3.err; tail -3 gpurun_out/cfg3.err
timeout 300 python scripts/spmm_bw.py > gpurun_out/r02_spmm_bw_final.json 2> gpurun_out/spmm.err; tail -6 gpurun_out/spmm.err
