#!/bin/bash
# usage: plan_sweep.sh shape "plan1" "plan2" ...   (development aid: compares hybrid plans on one shape)
shape=$1; shift
for p in "$@"; do
  if [ "$p" = "default" ]; then python scripts/time_one.py $shape tabu 296 400 | sed "s/^/default        /"
  elif [ "$p" = "nodsm" ]; then QAPB_NO_DSM=1 python scripts/time_one.py $shape tabu 296 400 | sed "s/^/nodsm          /"
  else QAPB_PLAN=$p python scripts/time_one.py $shape tabu 296 400 | sed "s/^/$p      /"; fi
done
