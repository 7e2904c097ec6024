# lanes per state at capacity 48 with the global workspace
for L in libmpskq libmpskq_nt48_96 libmpskq_nt48_128m4; do
  MPSKQ_LIB=paper_2411_09336_b200/$L.so timeout 600 python tools/ab_sim_abi.py 100 6 1e-16 800 48
  MPSKQ_LIB=paper_2411_09336_b200/$L.so timeout 600 python tools/ab_sim_abi.py 165 6 1e-16 296 48
done
