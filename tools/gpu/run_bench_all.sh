# final measurements: default bench line, reference arm, secondary configs, launch list
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_bench_reference_arm.err; echo "ref rc=$?"
timeout 1500 python tools/bench_configs.py > gpurun_out/r02_configs.log 2>&1; echo "configs rc=$?"; cp gpurun_out/configs.json gpurun_out/r02_configs.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --test-rows 0 > gpurun_out/r02_launches_bench.log 2>&1; echo "ncu rc=$?"
tail -c 600 gpurun_out/r02_bench_default.json; tail -c 400 gpurun_out/r02_bench_reference_arm.json
