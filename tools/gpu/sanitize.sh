# compute-sanitizer on the smallest headline-shape run (64 rows: sim_kernel<4,8>,
# the ket ordering / packing kernels, overlap_o1_kernel with its mbarrier ring)
# and a capacity-8 run (overlap_mma_kernel<8>).  usage: sanitize.sh racecheck|synccheck|memcheck
tool=$1
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/prof_overlap.py --n 64 --reps 1 \
  > gpurun_out/sanitizer_${tool}_o1.log 2>&1
echo "o1 rc=$?"; tail -4 gpurun_out/sanitizer_${tool}_o1.log
timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/prof_configs.py c5_d2_cap8 --n 16 \
  > gpurun_out/sanitizer_${tool}_mma8.log 2>&1
echo "mma8 rc=$?"; tail -4 gpurun_out/sanitizer_${tool}_mma8.log
