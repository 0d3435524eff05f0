python bench.py > gpurun_out/bench_r02n.json 2> gpurun_out/bench_r02n.log; echo "rc=$?" >> gpurun_out/bench_r02n.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --shard --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_shard1.json 2> gpurun_out/bench_shard1.log; echo "rc=$?" >> gpurun_out/bench_shard1.log
python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; echo "rc=$?" >> gpurun_out/bench_ref.log
