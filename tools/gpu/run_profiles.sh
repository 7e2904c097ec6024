bash tools/gpu/profile_o1.sh
bash tools/gpu/profile_kernels.sh
bash tools/gpu/run_reference_suite.sh
