mkdir -p gpurun_out
timeout 600 python tools/diag_fixture.py stretch_m165_d6_b24 > gpurun_out/diag_b24_default.log 2>&1
MPSKQ_LIB=paper_2411_09336_b200/libmpskq_noise0.so timeout 600 python tools/diag_fixture.py stretch_m165_d6_b24 > gpurun_out/diag_b24_noise0.log 2>&1
cat gpurun_out/diag_b24_default.log gpurun_out/diag_b24_noise0.log
timeout 900 python -m pytest tests/test_gpu_distributed.py -q -p no:cacheprovider -x > gpurun_out/r2_dist.log 2>&1
tail -3 gpurun_out/r2_dist.log
timeout 900 python tools/bench_configs.py config2_m50_d2 config3_m100_d4 config5_m100_d2 config5_m100_d6 > gpurun_out/r2_configs_a.log 2>&1
cat gpurun_out/r2_configs_a.log
