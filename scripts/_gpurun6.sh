mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2d.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_r2d.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err; echo bench rc=$?
tail -c 1500 gpurun_out/bench_r02d.json
