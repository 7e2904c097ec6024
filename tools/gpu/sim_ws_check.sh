mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not d7 and not d8" > gpurun_out/ws_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ws_tests.log
CFGS="config2_m50_d2 config3_m100_d4 config5_m100_d2 config5_m100_d3 config5_m100_d4 config5_m100_d5 config5_m100_d6 config4_m165_d6_1e-16" bash tools/gpu/run_configs_each.sh
