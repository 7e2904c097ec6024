# A/B of the headline overlap: libmpskq_base.so (previous commit) vs the tree
mkdir -p gpurun_out
for k in 1 2; do
  for L in paper_2411_09336_b200/libmpskq_base.so paper_2411_09336_b200/libmpskq.so; do
    MPSKQ_LIB=$L timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 --test-rows 0 > gpurun_out/ab_o1_$(basename $L .so)_$k.json 2>/dev/null
  done
done
for f in gpurun_out/ab_o1_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', round(d['phases_ms']['overlap'],2), round(d['roofline']['frac'],4), round(d['e2e']['ms_per_step'],2), d['parity_spot_check'])"; done
