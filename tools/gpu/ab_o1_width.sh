# A/B of the O1 block-width variants (interleaved, 2 rounds)
mkdir -p gpurun_out
for k in 1 2; do
  for L in libmpskq_base libmpskq libmpskq_w4 libmpskq_nospec; do
    MPSKQ_LIB=paper_2411_09336_b200/$L.so timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 --test-rows 0 > gpurun_out/abw_${L}_$k.json 2>/dev/null
  done
done
for f in gpurun_out/abw_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', 'ov', round(d['phases_ms']['overlap'],2), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['ms_per_step'],2), d['parity_spot_check']['bond_dims_equal'], d['parity_spot_check'].get('max_abs_err'))" 2>&1 | tail -1; done
