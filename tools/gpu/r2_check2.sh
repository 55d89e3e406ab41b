set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_graph.py tests/test_gpu_dist.py tests/test_gpu_stats.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_noise.py -q -p no:cacheprovider -rs -s > gpurun_out/r2_gputest2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_gputest2.log
for c in cfg0 cfg3 cfg4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench2_$c.log 2>&1
  echo "bench rc=$?" >> gpurun_out/r2_bench2_$c.log
done
