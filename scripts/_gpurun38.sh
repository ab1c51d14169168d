mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest38.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest38.log
timeout 300 python scripts/probe_upload.py > gpurun_out/upl38.log 2>&1; cat gpurun_out/upl38.log
