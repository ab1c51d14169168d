mkdir -p gpurun_out
timeout 300 python scripts/probe_query_ab.py c2 5 > gpurun_out/ab_flow.log 2>&1; echo flow rc=$?
tail -2 gpurun_out/ab_flow.log | cut -c1-600
MORAP_FLOW=0 timeout 300 python scripts/probe_query_ab.py c2 5 > gpurun_out/ab_lock.log 2>&1; echo lock rc=$?
tail -2 gpurun_out/ab_lock.log | cut -c1-600
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2c.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_r2c.log
timeout 300 python scripts/probe_query_ab.py c4 1 > gpurun_out/ab_flow_c4.log 2>&1; echo flowc4 rc=$?
tail -1 gpurun_out/ab_flow_c4.log | cut -c1-600
MORAP_FLOW=0 timeout 300 python scripts/probe_query_ab.py c4 1 > gpurun_out/ab_lock_c4.log 2>&1; echo lockc4 rc=$?
tail -1 gpurun_out/ab_lock_c4.log | cut -c1-600
