mkdir -p gpurun_out
timeout 300 python scripts/probe_query_ab.py c2 10 > gpurun_out/ab22.log 2>&1; tail -1 gpurun_out/ab22.log | cut -c1-420
timeout 900 python scripts/probe_query_ab.py c4 1 > gpurun_out/ab22c4.log 2>&1; tail -1 gpurun_out/ab22c4.log | cut -c1-420
