mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest25.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest25.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_$tool.log 2>&1; echo "$tool smoke rc=$?"; tail -3 gpurun_out/san_$tool.log
done
timeout 1200 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_skip_gpu.py tests/test_shard_gpu.py::test_multi_device_query_matches_reference -m gpu -x -q > gpurun_out/san_memcheck_tests.log 2>&1; echo "memcheck tests rc=$?"; tail -3 gpurun_out/san_memcheck_tests.log
timeout 1200 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_skip_gpu.py -m gpu -x -q > gpurun_out/san_racecheck_tests.log 2>&1; echo "racecheck tests rc=$?"; tail -3 gpurun_out/san_racecheck_tests.log
