mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_skip_gpu.py tests/test_kernels_gpu.py tests/test_pareto_gpu.py tests/test_measured_configs.py -m gpu -x -q > gpurun_out/pytest32.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest32.log
for v in 1 0; do MORAP_OPT_PERSISTENT=$v timeout 300 python scripts/probe_query_ab.py c2 10 > gpurun_out/ab32.log 2>&1; echo persistent=$v; tail -1 gpurun_out/ab32.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_query'], d['stats']['optimize_s'], d['opt_kernel_ms'], d['frac'])"; done
MORAP_TRACE=1 timeout 300 python scripts/probe_query_ab.py c2 1 > gpurun_out/t32.log 2> gpurun_out/t32.err; grep "persistent optimize" gpurun_out/t32.err | tail -2
