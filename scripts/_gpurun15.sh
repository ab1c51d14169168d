mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest15.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest15.log
timeout 300 python scripts/probe_query_ab.py c2 10 > gpurun_out/ab15.log 2>&1; echo ab rc=$?; tail -1 gpurun_out/ab15.log | cut -c1-500
