mkdir -p gpurun_out
python scripts/qp_probe.py --profile c4 100 231 > gpurun_out/qp8.log 2>&1
(time python scripts/replay_sandwich.py tests/golden/replay/c4_query.npz ours) > gpurun_out/replay_c4.log 2>&1
(time python scripts/replay_sandwich.py tests/golden/replay/c3_query.npz ours) > gpurun_out/replay_c3.log 2>&1
