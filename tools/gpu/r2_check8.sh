set -u
mkdir -p gpurun_out/prof
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/r2_gputest8.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_gputest8.log
timeout 600 python tools/e2e_profile.py cfg0 > gpurun_out/r2_e2e_cfg0.log 2>&1
timeout 600 python tools/e2e_profile.py cfg3 > gpurun_out/r2_e2e_cfg3.log 2>&1
