set -u
mkdir -p gpurun_out/prof
timeout 2400 python -m pytest tests/test_gpu_guard.py tests/test_gpu_sanitize.py tests/test_gpu_graph.py tests/test_gpu_parity.py tests/test_gpu_apf.py tests/test_gpu_verify.py tests/test_gpu_noise.py -q -p no:cacheprovider -rs -s > gpurun_out/r2_gputest5.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_gputest5.log
for c in cfg4 cfg0 cfg3 cfg2; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench5_$c.log 2>&1
  echo "bench rc=$?" >> gpurun_out/r2_bench5_$c.log
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/prof/launches_cfg0_r2.csv python bench.py --config cfg0 --steps 5 --warmup 3 --no-cpu-baseline --profile > gpurun_out/prof/launches_cfg0_r2.log 2>&1
