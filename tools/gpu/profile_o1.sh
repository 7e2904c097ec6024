# ncu --set full capture of ONE overlap_o1_kernel launch (headline shape,
# N=2048 rows) with source correlation, for SASS-level stall analysis here.
mkdir -p gpurun_out
python tools/prof_overlap.py --n 2048 --reps 1 > gpurun_out/prof_o1_plain.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:overlap_o1 -c 1 \
    -o gpurun_out/o1_full --force-overwrite python tools/prof_overlap.py --n 2048 --reps 1 \
    > gpurun_out/prof_o1_ncu.log 2>&1
tail -3 gpurun_out/prof_o1_ncu.log
