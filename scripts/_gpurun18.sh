mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest18.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest18.log
timeout 300 python scripts/probe_query_ab.py c2 10 > gpurun_out/ab18.log 2>&1; echo ab rc=$?; tail -1 gpurun_out/ab18.log | cut -c1-500
MORAP_EVAL_INTERLEAVED=0 timeout 300 python scripts/probe_query_ab.py c2 10 > gpurun_out/ab18b.log 2>&1; echo ab rc=$?; tail -1 gpurun_out/ab18b.log | cut -c1-500
timeout 300 python scripts/probe_eval_trace.py > gpurun_out/evtrace18.log 2>&1; tail -1 gpurun_out/evtrace18.log
