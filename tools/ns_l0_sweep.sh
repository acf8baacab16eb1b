for l0 in ${L0S:-1e-7 1e-8 1e-9 1e-10}; do
  SBO_NS_L0_BIG=$l0 timeout 300 python tools/profile_iteration.py --m 1048576 --scene 4096 --p-edge 16 --K 32 --s0 16 2>&1 | grep -E "jacobi sweeps|rmse" | tr '\n' ' '; echo " l0=$l0"
done
