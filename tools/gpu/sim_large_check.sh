mkdir -p gpurun_out
CFGS="config4_m165_d6_1e-24 config5_m100_d8" bash tools/gpu/run_configs_each.sh
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "d7 or d8 or stretch or escalation" > gpurun_out/large_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/large_tests.log
