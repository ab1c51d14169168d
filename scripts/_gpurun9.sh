mkdir -p gpurun_out
cat gpurun_out/replay_c4.log gpurun_out/replay_c3.log 2>/dev/null | tail -4
MORAP_TRACE=1 timeout 300 python scripts/probe_query_ab.py c2 1 > gpurun_out/trace_c2.log 2> gpurun_out/trace_c2.err; echo rc=$?
