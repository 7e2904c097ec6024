bash tools/gpu/ab_o1.sh
bash tools/gpu/profile_kernels.sh
