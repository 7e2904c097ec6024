# A/B of simulator variants at the large capacities (AB_LIBS), parity of the variants first
set -x
for L in ${AB_LIBS:-paper_2411_09336_b200/libmpskq.so}; do
  MPSKQ_LIB=$L python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "capacit or largest or large_chi" 2>&1 | tail -2
done
for L in ${AB_LIBS:-paper_2411_09336_b200/libmpskq.so}; do
  MPSKQ_LIB=$L timeout 600 python tools/ab_sim_cfg.py 100 7 1e-16 296 64
  MPSKQ_LIB=$L timeout 600 python tools/ab_sim_cfg.py 100 8 1e-16 148 96
  MPSKQ_LIB=$L timeout 600 python tools/ab_sim_cfg.py 165 6 1e-24 148 128
done
[ -n "$AB_HALF" ] && timeout 600 python tools/ab_sim_cfg.py 165 6 1e-24 74 128
exit 0
