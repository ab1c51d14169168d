mkdir -p gpurun_out
MORAP_BUILD_CHECKED=1 python -m paper_2305_04397_b200.build > gpurun_out/build_checked.log 2>&1; echo checked build rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_checked.log 2>&1; echo checked pytest rc=$?; tail -3 gpurun_out/pytest_checked.log
python -c "from paper_2305_04397_b200 import build as b; b.build_all(force=True)" > /dev/null 2>&1; echo rebuild rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench26.json 2> gpurun_out/bench26.err; echo bench rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_r02b.csv python bench.py --steps 2 --warmup 1 --no-north-star --no-cpu-baseline > gpurun_out/ncu_launch26.log 2>&1; echo launches rc=$?
timeout 900 ncu --kernel-name regex:k_eval_interleaved --launch-skip 3 --launch-count 1 --set full --clock-control none --import-source on -f -o gpurun_out/eval_inter python scripts/probe_query_ab.py c2 1 > gpurun_out/ncu_eval.log 2>&1; echo ncu eval rc=$?
