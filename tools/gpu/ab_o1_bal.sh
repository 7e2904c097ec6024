mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_distributed.py tests/test_gpu_ops.py -q -p no:cacheprovider -x > gpurun_out/bal_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/bal_tests.log
for k in 1 2; do
  for L in libmpskq_nobal libmpskq; do
    MPSKQ_LIB=paper_2411_09336_b200/$L.so timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/abb_${L}_$k.json 2>/dev/null
  done
done
for f in gpurun_out/abb_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', 'ov', round(d['phases_ms']['overlap'],2), 'frac', round(d['roofline']['frac'],4), 'step', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), 'test_ov', round(d['test_kernel']['phases_ms']['overlap'],2), d['e2e']['k_bitwise_equal_device_path'], d['parity_spot_check'])" 2>&1 | tail -1; done
