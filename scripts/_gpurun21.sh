mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest21.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest21.log
timeout 300 python scripts/probe_upload.py > gpurun_out/upl21.log 2>&1; cat gpurun_out/upl21.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench21.json 2> gpurun_out/bench21.err; echo bench rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench21.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['e2e'].get('first_upload_s'), d['phase_s_per_query'], d['north_star']['s_per_iteration'], d['north_star']['roofline']['frac'], d['gpu_launches'])"
