mkdir -p gpurun_out
timeout 2400 python tools/bench_configs.py "$@" > gpurun_out/configs_run.log 2>&1; echo "rc=$?"
grep -o '^[a-z0-9_-]* \|"sim_ms": [0-9.]*\|"overlap_ms": [0-9.]*' gpurun_out/configs_run.log | paste - - -
