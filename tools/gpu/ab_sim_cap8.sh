# lanes per state at capacity 8 (and capacity 12 placement)
for k in 1 2; do for L in libmpskq libmpskq_nt8_64 libmpskq_nt8_64g; do
  MPSKQ_LIB=paper_2411_09336_b200/$L.so timeout 600 python tools/ab_sim_abi.py 100 2 1e-16 800 8
  MPSKQ_LIB=paper_2411_09336_b200/$L.so timeout 600 python tools/ab_sim_abi.py 50 2 1e-24 800 12
done; done
