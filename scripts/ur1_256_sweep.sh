#!/bin/bash
# Development aid: the one-register-unit shared-memory plan (plan 9) on 256 threads, two searches per SM,
# against the default two-register-unit plan at n = 129..190 (two symmetric matrices, packed keys).
for s in tai132a tai144a tai160a tai176a sko180 tai188a; do
  n=${s//[a-z]/}; nb=$(( (n + 3) / 4 )); noff=$(( nb * (nb - 1) / 2 )); us=$(( (noff - 256 + 255) / 256 ))
  python scripts/time_one.py $s tabu 296 640 | sed "s/^/default           /"
  QAPB_PLAN=1,256,$us,1,113 python scripts/time_one.py $s tabu 296 640 | sed "s/^/1,256,$us,1,113     /"
done
