# simulation A/B through the stable C ABI: round-1 library vs the tree
for L in paper_2411_09336_b200/libmpskq_r1.so paper_2411_09336_b200/libmpskq.so; do
  MPSKQ_LIB=$L timeout 600 python tools/ab_sim_abi.py 100 7 1e-16 800 64
  MPSKQ_LIB=$L timeout 600 python tools/ab_sim_abi.py 100 8 1e-16 800 96
  MPSKQ_LIB=$L timeout 600 python tools/ab_sim_abi.py 100 4 1e-16 1600 24
  MPSKQ_LIB=$L timeout 600 python tools/ab_sim_abi.py 165 1 1e-24 6400 4
done
