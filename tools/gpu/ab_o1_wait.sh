mkdir -p gpurun_out
for k in 1 2; do
  for L in libmpskq libmpskq_w200 libmpskq_w2000; do
    MPSKQ_LIB=paper_2411_09336_b200/$L.so timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/abwt_${L}_$k.json 2>/dev/null
  done
done
for f in gpurun_out/abwt_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', 'ov', round(d['phases_ms']['overlap'],2), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['ms_per_step'],2), 'test_ov', round(d['test_kernel']['phases_ms']['overlap'],2), d['e2e']['k_bitwise_equal_device_path'])" 2>&1 | tail -1; done
