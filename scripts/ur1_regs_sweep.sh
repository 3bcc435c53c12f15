#!/bin/bash
# Development aid: plan 9 (one register unit + shared-memory units, DSM) at other CTA sizes / register caps
# (dev builds: scripts/devbuild.sh 40 r<regs> -DQAPB_DEV_REGS=<regs>), two searches per SM at n = 157..190.
run() { QAPB_LIB=build/libqapb_dev40r$1.so QAPB_PLAN=$2 python scripts/time_one.py $3 tabu 296 640 | sed "s/^/r$1 $2  /"; }
for s in tai148a tai156a; do python scripts/time_one.py $s tabu 296 640 | sed "s/^/default /"; QAPB_PLAN=1,256,2,1,113 python scripts/time_one.py $s tabu 296 640 | sed "s/^/1,256,2,1,113 /"; done
run 112 1,288,2,1,113 tai160a
run 96 1,320,2,1,113 tai160a
run 88 1,352,2,1,113 tai160a
run 112 1,288,2,1,113 tai156a
run 96 1,320,2,1,113 tai176a
run 88 1,352,2,1,113 tai176a
run 88 1,352,2,1,113 sko180
run 96 1,320,2,1,113 tai150b
