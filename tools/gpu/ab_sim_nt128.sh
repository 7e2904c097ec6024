# threads per state at capacities 64-128
for L in libmpskq libmpskq_nt256 libmpskq_nt256_m2 libmpskq_nt256_m3; do
  MPSKQ_LIB=paper_2411_09336_b200/$L.so timeout 600 python tools/ab_sim_abi.py 100 7 1e-16 400 64
  MPSKQ_LIB=paper_2411_09336_b200/$L.so timeout 600 python tools/ab_sim_abi.py 100 8 1e-16 300 96
done
