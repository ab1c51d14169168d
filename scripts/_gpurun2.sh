mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_measured_configs.py tests/test_cli.py -m gpu -x -q > gpurun_out/pytest_r2b.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_r2b.log
MORAP_TRACE=1 timeout 900 python scripts/probe_full_query.py c3 500 > gpurun_out/full_c3.log 2> gpurun_out/full_c3.err; echo c3 rc=$?
MORAP_TRACE=1 timeout 1500 python scripts/probe_full_query.py c4 500 > gpurun_out/full_c4.log 2> gpurun_out/full_c4.err; echo c4 rc=$?
tail -2 gpurun_out/full_c3.log gpurun_out/full_c4.log | cut -c1-300
