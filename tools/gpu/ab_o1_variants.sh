# A/B of headline overlap variants (interleaved, 2 rounds) + escalation / stretch checks
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_ops.py tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "escalation or capacit or largest" > gpurun_out/esc_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/esc_tests.log
for k in 1 2; do
  for L in libmpskq libmpskq_cn1 libmpskq_ps200 libmpskq_cnps; do
    MPSKQ_LIB=paper_2411_09336_b200/$L.so timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 --test-rows 0 > gpurun_out/abv_${L}_$k.json 2>/dev/null
  done
done
for f in gpurun_out/abv_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', 'ov', round(d['phases_ms']['overlap'],2), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['ms_per_step'],2), d['e2e']['k_bitwise_equal_device_path'])" 2>&1 | tail -1; done
timeout 1500 python tools/bench_configs.py config4_m165_d6_1e-24 > gpurun_out/stretch.log 2>&1; echo "stretch rc=$?"; tail -2 gpurun_out/stretch.log | cut -c1-400
