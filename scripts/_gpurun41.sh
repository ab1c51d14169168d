mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest41.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest41.log
bash scripts/_gpurun39.sh
timeout 300 python scripts/probe_eval_trace.py > gpurun_out/evtrace41.log 2>&1; tail -1 gpurun_out/evtrace41.log | cut -c1-300
