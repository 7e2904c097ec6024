# the complete GPU suite (fast + slow at-scale scans) and the reference's own suite through the shim
mkdir -p gpurun_out
nproc
timeout 3000 python -m pytest tests -m gpu -v -p no:cacheprovider -rf --durations=30 > gpurun_out/r2_gpu_tests_all.log 2>&1
echo "gpu tests rc=$?"
grep -E "FAILED|ERROR| passed| failed" gpurun_out/r2_gpu_tests_all.log | tail -12
bash tools/gpu/run_reference_suite.sh
