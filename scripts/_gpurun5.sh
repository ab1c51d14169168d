mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench_r02.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_r02.json 2> gpurun_out/bench_ref_r02.err; echo ref rc=$?
tail -c 1500 gpurun_out/bench_ref_r02.json
timeout 600 python scripts/probe_ncu_c4.py bytes 30 > gpurun_out/c4_bytes30.json 2>&1; echo c4bytes rc=$?
cat gpurun_out/c4_bytes30.json | tail -1
MORAP_GRAPHS=0 timeout 1200 ncu --kernel-name regex:k_greedy_sweep_cmp --launch-skip 29 --launch-count 1 --set full --clock-control none --import-source on -f -o gpurun_out/c4_sweep30 python scripts/probe_ncu_c4.py run 30 > gpurun_out/ncu_c4.log 2>&1; echo ncuc4 rc=$?
tail -3 gpurun_out/ncu_c4.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 1 --no-north-star --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
