#!/bin/bash
# Development build of ONE search-kernel instantiation (seconds instead of minutes):
#   scripts/devbuild.sh <preset> [tag] [extra nvcc flags...]   ->  build/libqapb_dev<preset><tag>.so
# Presets are the QAPB_DEV_ONLY cases at the top of csrc/qapb.cu.  Use with QAPB_LIB=<path>.
set -e
cd "$(dirname "$0")/.."
preset=$1; tag=${2:-}; shift; shift || true
mkdir -p build
out=build/libqapb_dev${preset}${tag}.so
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -shared -Xcompiler -fPIC -Xptxas=-v \
  -DQAPB_DEV_ONLY=${preset} "$@" -o "$out" paper_2307_11248_b200/csrc/qapb.cu 2>&1 | grep -E "error|hybrid|spill|Used" | grep -A2 -E "error|Compiling.*hybrid" | grep -vE "^--|Compiling" | head -12
echo "$out"
