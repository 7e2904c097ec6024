# the round's final evidence pass: GPU suite, reference suite, bench lines,
# secondary configs, launch list, ncu of the headline overlap kernel
mkdir -p gpurun_out/ncu
nproc
timeout 2400 python -m pytest tests -m gpu -v -p no:cacheprovider -rf --durations=30 > gpurun_out/r02_gpu_tests_all.log 2>&1
echo "gpu tests rc=$?"; grep -E " passed| failed" gpurun_out/r02_gpu_tests_all.log | tail -2
bash tools/gpu/run_reference_suite.sh | tail -2
timeout 900 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_bench_reference_arm.err; echo "ref rc=$?"
timeout 1800 python tools/bench_configs.py > gpurun_out/r02_configs.log 2>&1; echo "configs rc=$?"; cp gpurun_out/configs.json gpurun_out/r02_configs.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --test-rows 0 > gpurun_out/r02_launches_bench.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:overlap_o1 -c 1 -o gpurun_out/ncu/o1_6400 --force-overwrite \
  python tools/prof_overlap.py --n 6400 --reps 1 > gpurun_out/ncu/o1_6400.log 2>&1; echo "ncu o1 rc=$?"
python tools/ncu_summary.py gpurun_out/ncu/o1_6400.ncu-rep > gpurun_out/ncu/o1_6400.summary.txt 2>&1
ncu -i gpurun_out/ncu/o1_6400.ncu-rep --page source --csv --print-source sass > /tmp/o1.src.csv 2>/dev/null && python tools/ncu_opcodes.py /tmp/o1.src.csv >> gpurun_out/ncu/o1_6400.summary.txt
rm -f gpurun_out/ncu/o1_6400.ncu-rep
cat gpurun_out/ncu/o1_6400.summary.txt | head -16
tail -c 700 gpurun_out/r02_bench_default.json
