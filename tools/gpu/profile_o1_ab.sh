# ncu --set full of one overlap_o1_kernel launch for two libraries; summaries only
mkdir -p gpurun_out/o1ab
for L in libmpskq_base libmpskq_nospec; do
  MPSKQ_LIB=paper_2411_09336_b200/$L.so ncu --set full --import-source on --clock-control none -k regex:overlap_o1 -c 1 \
    -o gpurun_out/o1ab/$L --force-overwrite python tools/prof_overlap.py --n 2048 --reps 1 > gpurun_out/o1ab/$L.log 2>&1
  ncu -i gpurun_out/o1ab/$L.ncu-rep --page source --csv --print-source sass > gpurun_out/o1ab/$L.src.csv 2>/dev/null
  python tools/ncu_opcodes.py gpurun_out/o1ab/$L.src.csv > gpurun_out/o1ab/$L.opcodes.txt 2>&1
  python tools/ncu_summary.py gpurun_out/o1ab/$L.ncu-rep > gpurun_out/o1ab/$L.summary.txt 2>&1
  rm -f gpurun_out/o1ab/$L.ncu-rep gpurun_out/o1ab/$L.src.csv
done
