mkdir -p gpurun_out
python scripts/probe_ncu_sweep.py bytes 30 > gpurun_out/c2_bytes30.json 2>&1; tail -1 gpurun_out/c2_bytes30.json
MORAP_GRAPHS=0 timeout 900 ncu --kernel-name regex:k_greedy_sweep_cmp --launch-skip 29 --launch-count 1 --set full --clock-control none --import-source on -f -o gpurun_out/c2_sweep30 python scripts/probe_ncu_sweep.py run 30 > gpurun_out/ncu_c2.log 2>&1; echo ncu sweep rc=$?
MORAP_GRAPHS=0 timeout 900 ncu --kernel-name regex:k_select --launch-skip 29 --launch-count 1 --set full --clock-control none -f -o gpurun_out/c2_select30 python scripts/probe_ncu_sweep.py run 30 > gpurun_out/ncu_sel.log 2>&1; echo ncu select rc=$?
MORAP_TRACE=1 timeout 600 python -c "
import sys, time; sys.path.insert(0,'.')
import bench
from paper_2305_04397_b200.api import Instance, Solver
cfg, thr, eps, K = bench.workload('c4')
s = Solver(0); s.set_lean(True)
t = time.time(); inst = Instance.warehouse_streamed(cfg, s, chunk=bench.STREAMED['c4']); print('c4 build+upload', time.time()-t, flush=True)
" > gpurun_out/c4build.log 2> gpurun_out/c4build.err; tail -1 gpurun_out/c4build.log; grep "upload prep\|copied" gpurun_out/c4build.err | tail -4
