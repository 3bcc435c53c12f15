#!/bin/bash
# Development aid: default plans at n = 129..190 (two symmetric matrices), tabu and 2opt.
for s in tai132a tai144a tai148a tai156a tai160a sko140 sko152; do
  python scripts/time_one.py $s tabu 296 640
  python scripts/time_one.py $s 2opt 296 320
done
