# secondary configs, one process per config (no cross-config allocator / hint state)
mkdir -p gpurun_out/cfg
CFGS="${CFGS:-config1_m8_d1 config2_m50_d2 config3_m100_d4 config5_m100_d1 config5_m100_d2 config5_m100_d3 config5_m100_d4 \
         config5_m100_d5 config5_m100_d6 config5_m100_d7 config5_m100_d8 config4_m165_d6_1e-16 config4_m165_d6_1e-24}"
for c in $CFGS; do
  timeout 1200 python tools/bench_configs.py $c > gpurun_out/cfg/$c.log 2>&1
  cp gpurun_out/configs.json gpurun_out/cfg/$c.json
  grep -o '^[a-z0-9_-]* \|"sim_ms": [0-9.]*\|"overlap_ms": [0-9.]*' gpurun_out/cfg/$c.log | paste - - -
done
python - <<'PY'
import json, glob
out = {}
for f in sorted(glob.glob('gpurun_out/cfg/*.json')):
    d = json.load(open(f)); out.update(d)
json.dump(out, open('gpurun_out/r02_configs.json', 'w'), indent=1)
PY
