mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest33.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest33.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench33.json 2> gpurun_out/bench33.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench33_ref.json 2> gpurun_out/bench33_ref.err; echo ref rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench33.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['phase_s_per_query'], d['north_star']['s_per_iteration'], d['north_star']['roofline']['frac'])
r=json.loads(open('gpurun_out/bench33_ref.json').read().strip().splitlines()[-1]); print(r['ms_per_step'], r['value'])"
