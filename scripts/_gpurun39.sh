mkdir -p gpurun_out
for i in 1 2; do timeout 300 python scripts/probe_query_ab.py c2 10 > gpurun_out/ab39.log 2>&1; tail -1 gpurun_out/ab39.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_query'], d['stats'])"; done
MORAP_TRACE=1 timeout 300 python scripts/probe_query_ab.py c2 1 > gpurun_out/t39.log 2> gpurun_out/t39.err; grep "supportingPoint" gpurun_out/t39.err | tail -3
