mkdir -p gpurun_out
MORAP_TRACE=1 timeout 900 python scripts/probe_full_query.py c3 500 > gpurun_out/full_c3.log 2> gpurun_out/full_c3.err; echo c3 rc=$?; tail -2 gpurun_out/full_c3.log | cut -c1-700
MORAP_TRACE=1 timeout 1500 python scripts/probe_full_query.py c4 500 > gpurun_out/full_c4.log 2> gpurun_out/full_c4.err; echo c4 rc=$?; tail -2 gpurun_out/full_c4.log | cut -c1-700
