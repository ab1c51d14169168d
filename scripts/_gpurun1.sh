set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total --format=csv
free -g | head -2; nproc
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2a.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_r2a.log
timeout 900 python scripts/probe_full_query.py c3 500 > gpurun_out/full_c3.log 2>&1; echo c3 rc=$?
tail -3 gpurun_out/full_c3.log
timeout 1500 python scripts/probe_full_query.py c4 500 > gpurun_out/full_c4.log 2>&1; echo c4 rc=$?
tail -3 gpurun_out/full_c4.log
