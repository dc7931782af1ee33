#!/bin/bash
# hoisted-K6 build with a __syncwarp() before the empty-barrier arrive: does it still hang? then A/B vs in-tree
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
o=gpurun_out/k6_hoist2.log; : > $o
K6_SYNCWARP=1 python tools/debug/k6_hoist.py > /dev/null 2>&1 || { echo build failed >> $o; exit 1; }
echo "== hoisted+syncwarp, 4 atoms" >> $o; timeout 120 python tools/profile_pi.py --atoms 4 --steps 1 --lib /tmp/k6h/libsse.so >> $o 2>&1; rc=$?; echo "rc=$rc" >> $o
if [ $rc -eq 0 ]; then
  for r in 1 2; do
    echo "in-tree: $(timeout 300 python tools/profile_pi.py --atoms 96 --steps 2 2>&1 | tail -1)" >> $o
    echo "hoisted: $(timeout 300 python tools/profile_pi.py --atoms 96 --steps 2 --lib /tmp/k6h/libsse.so 2>&1 | tail -1)" >> $o
  done
fi
cat $o
