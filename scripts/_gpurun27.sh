mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest27.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest27.log
timeout 300 python scripts/probe_query_ab.py c2 10 > gpurun_out/ab27.log 2>&1; tail -1 gpurun_out/ab27.log | cut -c1-420
