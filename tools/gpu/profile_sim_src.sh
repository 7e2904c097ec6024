# source-line attribution of sim_kernel<24,128> (config 3 shape, 296 states = 2 per SM)
mkdir -p gpurun_out/ncu
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:sim_kernel<.int.24," -c 1 \
  -o gpurun_out/ncu/sim24src --force-overwrite python tools/prof_configs.py c3_cap24 --n 296 --sim-only > gpurun_out/ncu/sim24src.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/ncu/sim24src.ncu-rep --page source --csv --print-source cuda > gpurun_out/ncu/sim24src_cuda.csv 2>/dev/null
ncu -i gpurun_out/ncu/sim24src.ncu-rep --page source --csv --print-source sass > /tmp/s.csv 2>/dev/null; python tools/ncu_opcodes.py /tmp/s.csv > gpurun_out/ncu/sim24src_ops.txt
python tools/ncu_summary.py gpurun_out/ncu/sim24src.ncu-rep > gpurun_out/ncu/sim24src_summary.txt
rm -f gpurun_out/ncu/sim24src.ncu-rep
ls -la gpurun_out/ncu/
