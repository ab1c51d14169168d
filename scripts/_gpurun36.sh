mkdir -p gpurun_out
python scripts/qp_probe.py c4 100 231 > gpurun_out/qp36.log 2>&1; cat gpurun_out/qp36.log
(time python scripts/replay_sandwich.py tests/golden/replay/c4_query.npz ours) > gpurun_out/replay_c4b.log 2>&1; tail -4 gpurun_out/replay_c4b.log
