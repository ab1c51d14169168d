mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_pareto_gpu.py tests/test_skip_gpu.py tests/test_kernels_gpu.py tests/test_measured_configs.py -m gpu -x -q > gpurun_out/pytest11.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest11.log
timeout 300 python scripts/probe_query_ab.py c2 10 > gpurun_out/ab11.log 2>&1; echo ab rc=$?; tail -1 gpurun_out/ab11.log | cut -c1-400
MORAP_TRACE=1 timeout 300 python scripts/probe_query_ab.py c2 1 > gpurun_out/trace11.log 2> gpurun_out/trace11.err; grep "optimize batch" gpurun_out/trace11.err | head -20
