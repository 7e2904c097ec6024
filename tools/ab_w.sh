# A/B of simulator variants at the large capacities + the full GPU suite
set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -5
for L in ${AB_LIBS:-paper_2411_09336_b200/libmpskq.so}; do
  MPSKQ_LIB=$L timeout 600 python tools/ab_sim_cfg.py 100 7 1e-16 296 64
  MPSKQ_LIB=$L timeout 600 python tools/ab_sim_cfg.py 100 8 1e-16 148 96
done
