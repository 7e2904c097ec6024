mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider > gpurun_out/qc_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/qc_tests.log
bash tools/gpu/run_reference_suite.sh | tail -1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/qc_bench.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/qc_bench.json').read().strip().splitlines()[-1])
print('ov', round(d['phases_ms']['overlap'],2), 'frac', round(d['roofline']['frac'],4), 'step', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), 'c_abi', round(d['e2e_c_abi']['ms_per_step'],2), 'test', round(d['test_kernel']['ms_per_step'],2))"
