# threads per state at capacities 32 / 48 (after LogW at 24-32)
for L in libmpskq libmpskq_nt32_192 libmpskq_nt32_256; do
  MPSKQ_LIB=paper_2411_09336_b200/$L.so timeout 600 python tools/ab_sim_abi.py 100 5 1e-16 800 32
done
for L in libmpskq libmpskq_nt48_128 libmpskq_nt48_256; do
  MPSKQ_LIB=paper_2411_09336_b200/$L.so timeout 600 python tools/ab_sim_abi.py 100 6 1e-16 400 48
done
