# A/B of paper_2411_09336_b200/libmpskq_a.so (baseline variant) against the tree on the secondary configs
mkdir -p gpurun_out
for k in 1 2; do
for L in paper_2411_09336_b200/libmpskq_a.so paper_2411_09336_b200/libmpskq.so; do
  nvidia-smi --query-gpu=clocks.sm,clocks_event_reasons.active,temperature.gpu,power.draw --format=csv,noheader
  MPSKQ_LIB=$L timeout 900 python tools/bench_configs.py config2_m50_d2 config5_m100_d2 config5_m100_d3 > gpurun_out/ab_configs_$(basename $L .so)_$k.log 2>&1
  echo "$L run $k"; grep -o '^[a-z0-9_]* \|"sim_ms": [0-9.]*\|"overlap_ms": [0-9.]*' gpurun_out/ab_configs_$(basename $L .so)_$k.log | paste - - - 
done
done
