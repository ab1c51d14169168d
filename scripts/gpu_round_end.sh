#!/usr/bin/env bash
# The round-end GPU checks, as run through gpurun:
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash scripts/gpu_round_end.sh'
# GPU test suite, smoke(), the headline bench (C2 + C4 leg), the reference arm, and the
# ncu launch list of the bench command (each profiler pass after its own clean run).
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print('c2 ms/query', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], 'frac', d['roofline']['frac'],
      'c4 s/iter', d['north_star']['s_per_iteration'], 'c4 frac', d['north_star']['roofline']['frac'])
r = json.loads(open('gpurun_out/bench_ref.json').read().strip().splitlines()[-1])
print('reference ms/query', r['ms_per_step'])
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-north-star --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
python scripts/launch_summary.py gpurun_out/launches.csv "ncu launch list of python bench.py --steps 2 --warmup 1 --no-north-star --no-cpu-baseline (C2)" > gpurun_out/launches.txt 2>&1; head -20 gpurun_out/launches.txt
# device product builder: C4 build trace, and one ncu --set full capture of the builder kernel (C2 measure pass)
MORAP_TRACE=1 timeout 300 python scripts/probe_device_build.py c4 0 > gpurun_out/devc4.json 2> gpurun_out/devc4.err; echo "device build rc=$?"
tail -1 gpurun_out/devc4.json; grep "build_products\|planDevice\|DeviceBuild" gpurun_out/devc4.err
timeout 600 ncu --kernel-name regex:k_build_products --launch-count 1 --set full --clock-control none --import-source on \
  -f -o gpurun_out/build_c2 python scripts/probe_device_build.py c2 0 > gpurun_out/ncu_build.log 2>&1; echo "ncu build rc=$?"
