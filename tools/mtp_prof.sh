# in-kernel cycle accounting of the tcgen05 MTP kernel at several L (env TPO_MTP_PROF=1)
for L in ${LS:-1 4 6}; do
  TPO_MTP_PROF=1 timeout -s KILL 60 python tools/profile_kernel.py --kind mtp --L $L --reps 2 2>&1 | grep -E "tpo-prof" | tail -1
done
