#!/bin/bash
# Development aid: warps per CTA of the one-warp-per-search kernel (QAPB_WPC, default 4).
for w in 1 2 3 4 6 8; do
  QAPB_WPC=$w python scripts/time_one.py tai30a tabu 1776 240 | sed "s/^/wpc=$w /"
  QAPB_WPC=$w python scripts/time_one.py nug12 tabu 4736 96 | sed "s/^/wpc=$w /"
done
