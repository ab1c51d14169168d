mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_distributed_gpu.py tests/test_shard_gpu.py -m gpu -x -q > gpurun_out/pytest24.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest24.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --sharded --steps 5 --warmup 3 > gpurun_out/bench_sharded.json 2> gpurun_out/bench_sharded.err; echo rc=$?; tail -c 1500 gpurun_out/bench_sharded.json; tail -5 gpurun_out/bench_sharded.err
