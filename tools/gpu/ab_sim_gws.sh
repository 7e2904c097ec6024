# capacity 12 workspace placement; threads per state at capacity 48
for L in libmpskq libmpskq_ab8; do
  MPSKQ_LIB=paper_2411_09336_b200/$L.so timeout 600 python tools/ab_sim_abi.py 50 2 1e-24 800 12
  MPSKQ_LIB=paper_2411_09336_b200/$L.so timeout 600 python tools/ab_sim_abi.py 100 3 1e-16 1600 16
done
for L in libmpskq libmpskq_nt48_128 libmpskq_nt48_64; do
  MPSKQ_LIB=paper_2411_09336_b200/$L.so timeout 600 python tools/ab_sim_abi.py 100 6 1e-16 400 48
done
