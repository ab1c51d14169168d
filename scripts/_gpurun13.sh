mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_skip_gpu.py tests/test_variants_gpu.py tests/test_pareto_gpu.py tests/test_measured_configs.py tests/test_acceptance_gpu.py -m gpu -x -q > gpurun_out/pytest13.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest13.log
timeout 300 python scripts/probe_query_ab.py c2 10 > gpurun_out/ab13.log 2>&1; echo ab rc=$?; tail -1 gpurun_out/ab13.log | cut -c1-600
MORAP_FUSED=0 timeout 300 python scripts/probe_query_ab.py c2 10 > gpurun_out/ab13b.log 2>&1; echo ab rc=$?; tail -1 gpurun_out/ab13b.log | cut -c1-600
MORAP_TRACE=1 timeout 300 python scripts/probe_query_ab.py c2 1 > gpurun_out/trace13.log 2> gpurun_out/trace13.err; grep "supportingPoint" gpurun_out/trace13.err | tail -4
