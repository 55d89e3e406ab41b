set -u
mkdir -p gpurun_out/prof
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_graph.py tests/test_gpu_apf.py tests/test_gpu_verify.py tests/test_gpu_small.py tests/test_gpu_stats.py -q -p no:cacheprovider -rs -s > gpurun_out/r2_gputest6.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_gputest6.log
for c in cfg0 cfg3 cfg2 cfg2apf cfg1b cfg1c; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench6_$c.log 2>&1
  echo "bench rc=$?" >> gpurun_out/r2_bench6_$c.log
done
