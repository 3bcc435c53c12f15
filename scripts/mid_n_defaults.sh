#!/bin/bash
# Development aid: default plans at n = 129..190 (two symmetric matrices), tabu and 2opt.
for s in tai132a tai144a tai148a tai156a tai160a tai164a tai176a sko180 sko140 sko152; do
  python scripts/time_one.py $s tabu 296 640
  python scripts/time_one.py $s 2opt 296 320
done
python scripts/time_one.py tai160a tabu 148 640
