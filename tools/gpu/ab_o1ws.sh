mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_edges.py tests/test_gpu_ops.py -m "gpu and not slow" -q -p no:cacheprovider -x > gpurun_out/ws_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/ws_tests.log
for k in 1 2; do
  for L in paper_2411_09336_b200/libmpskq_ws0.so paper_2411_09336_b200/libmpskq.so; do
    MPSKQ_LIB=$L timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/ab_ws_$(basename $L .so)_$k.json 2>/dev/null
  done
done
for f in gpurun_out/ab_ws_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', 'ov', round(d['phases_ms']['overlap'],2), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['ms_per_step'],2), 'test_ov', round(d['test_kernel']['phases_ms']['overlap'],2), d['parity_spot_check']['bond_dims_equal'], d['e2e']['k_bitwise_equal_device_path'])"; done
