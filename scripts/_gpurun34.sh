mkdir -p gpurun_out
for b in normal diag normal diag; do
  if [ $b = diag ]; then MORAP_BUILD_DIAGNOSTICS=1 python -m paper_2305_04397_b200.build > /dev/null 2>&1; else python -c "from paper_2305_04397_b200 import build as b; b.build_all(force=True)" > /dev/null 2>&1; fi
  timeout 300 python scripts/probe_query_ab.py c2 10 > gpurun_out/ab34.log 2>&1; echo $b; tail -1 gpurun_out/ab34.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_query'], d['stats']['optimize_s'], d['opt_kernel_ms'], d['frac'])"
done
