mkdir -p gpurun_out
MPSKQ_LIB=paper_2411_09336_b200/libmpskq_w4s4.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_distributed.py -q -p no:cacheprovider -x -k "headline or reference or pinned or streams or two_ranks or nccl or c_abi" > gpurun_out/w4_tests.log 2>&1; echo "w4 tests rc=$?"; tail -1 gpurun_out/w4_tests.log
for k in 1 2; do
  for L in libmpskq libmpskq_w4s4; do
    MPSKQ_LIB=paper_2411_09336_b200/$L.so timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/abw_${L}_$k.json 2>/dev/null
  done
done
for f in gpurun_out/abw_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', 'ov', round(d['phases_ms']['overlap'],2), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['ms_per_step'],2), 'test_ov', round(d['test_kernel']['phases_ms']['overlap'],2), d['e2e']['k_bitwise_equal_device_path'])" 2>&1 | tail -1; done
