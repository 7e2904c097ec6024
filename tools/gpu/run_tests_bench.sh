set -x
nproc
python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=25 > gpurun_out/r2_gpu_tests_1.log 2>&1
tail -5 gpurun_out/r2_gpu_tests_1.log
python bench.py --steps 5 --warmup 3 --cpu-seconds 5 > gpurun_out/r2_bench_1.json 2> gpurun_out/r2_bench_1.err
tail -c 3000 gpurun_out/r2_bench_1.json
