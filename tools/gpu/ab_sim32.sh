for c in "100 4 1e-16 1600 24" "100 5 1e-16 800 32" "100 3 1e-16 1600 16"; do timeout 600 python tools/ab_sim_abi.py $c; done
timeout 1500 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_parity.py tests/test_gpu_ops.py tests/test_gpu_edges.py -x -q -m gpu -k "not d6 and not d7 and not d8" 2>&1 | tail -3
