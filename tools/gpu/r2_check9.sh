set -u
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2_smoke.log
timeout 900 python -m pytest tests/test_gpu_noise.py tests/test_gpu_stats.py -q -p no:cacheprovider -rs -s > gpurun_out/r2_gputest9.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_gputest9.log
timeout 600 python tools/e2e_profile.py cfg2 > gpurun_out/r2_e2e_cfg2.log 2>&1
