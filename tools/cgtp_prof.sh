# in-kernel cycle accounting of the tcgen05 CGTP block kernel at several L (env TPO_CGTP_PROF=1)
for L in ${LS:-3 6 10}; do
  TPO_CGTP_PROF=1 timeout -s KILL 60 python tools/profile_kernel.py --kind cgtp --L $L --reps 2 2>&1 | grep -E "tpo-prof" | tail -1
done
