set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --shard --steps 3 --warmup 3 --no-cpu-baseline --no-at-scale > gpurun_out/r02_bench_cfg1_shard1.json 2> gpurun_out/shard1.err; tail -c 500 gpurun_out/shard1.err
