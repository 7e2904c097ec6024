# ncu captures of the secondary-config kernels (one launch each), summarised
# ON the box (the .ncu-rep files are large): overlap_mma_kernel at capacities
# 8 / 12 / 24 / 96 (--set full) and sim_kernel at 24 (--set full) and
# 48 / 128 (reduced sections: one launch runs for seconds).
mkdir -p gpurun_out/ncu
summ() {  # name
  python tools/ncu_summary.py gpurun_out/ncu/$1.ncu-rep > gpurun_out/ncu/$1.summary.txt 2>&1
  ncu -i gpurun_out/ncu/$1.ncu-rep --page source --csv --print-source sass > /tmp/$1.src.csv 2>/dev/null \
    && python tools/ncu_opcodes.py /tmp/$1.src.csv >> gpurun_out/ncu/$1.summary.txt 2>&1
  ncu -i gpurun_out/ncu/$1.ncu-rep --page raw --csv > gpurun_out/ncu/$1.raw.csv 2>/dev/null
  rm -f gpurun_out/ncu/$1.ncu-rep
}
run() {  # name config n kernel-regex extra-ncu-args...
  local name=$1 cfg=$2 n=$3 k=$4; shift 4
  timeout 900 ncu --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -c 1 "$@" \
      -o gpurun_out/ncu/$name --force-overwrite python tools/prof_configs.py $cfg --n $n \
      > gpurun_out/ncu/$name.log 2>&1
  echo "$name rc=$?"
  summ $name
}
for c in "mma8 c5_d2_cap8 512 overlap_mma_kernel<.int.8>" "mma12 c2_cap12 512 overlap_mma_kernel<.int.12>" \
         "mma24 c3_cap24 256 overlap_mma_kernel<.int.24>" "mma96 c5_d8_cap96 64 overlap_mma_kernel<.int.96>"; do
  set -- $c
  run $1 $2 $3 "$4" --set full
done
RED="--section SpeedOfLight --section WarpStateStats --section Occupancy --section LaunchStats --section InstructionStats --section SourceCounters"
run sim24 c3_cap24 148 "sim_kernel<.int.24," --set full
run sim48 c5_d6_cap48 148 "sim_kernel<.int.48," $RED
run sim128 s6_b24_cap128 16 "sim_kernel<.int.128," $RED
ls -la gpurun_out/ncu; du -sh gpurun_out
