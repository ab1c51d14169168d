mkdir -p gpurun_out
for v in "2 1024 1" "4 512 1" "6 512 1" "3 768 1"; do
  set -- $v
  sed -i "s/constexpr int kEvU = [0-9];/constexpr int kEvU = $1;/" paper_2305_04397_b200/csrc/morap_cuda.cu
  NVCC_EXTRA="-DMORAP_PERSIST_THREADS=$2 -DMORAP_PERSIST_MINB=$3" python -c "
import os, subprocess
from paper_2305_04397_b200 import build as b
cmd=[b.NVCC,*b.CUDA_FLAGS,*os.environ['NVCC_EXTRA'].split(),'-o',b.CUDA_SO,os.path.join(b.CSRC,'morap_cuda.cu')]
subprocess.run(cmd,check=True)"
  echo "U=$1 threads=$2"
  timeout 300 python scripts/probe_query_ab.py c2 10 > gpurun_out/ab16.log 2>&1; tail -1 gpurun_out/ab16.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_query'], d['stats']['evaluate_batch_s'])"
done
