# GPU test suite (fast part, verbose), then the default bench line.
mkdir -p gpurun_out
nproc
timeout 1500 python -m pytest tests -m "gpu and not slow" -v -p no:cacheprovider -rf --durations=20 \
  > gpurun_out/r2_gpu_tests_fast.log 2>&1
echo "fast tests rc=$?"
grep -E "FAILED|ERROR|passed|failed" gpurun_out/r2_gpu_tests_fast.log | tail -15
timeout 900 python bench.py --steps 5 --warmup 3 --cpu-seconds 5 > gpurun_out/r2_bench_1.json 2> gpurun_out/r2_bench_1.err
echo "bench rc=$?"
tail -c 1500 gpurun_out/r2_bench_1.err
