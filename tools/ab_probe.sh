#!/bin/bash
# A/B of library builds on one box with tools/probe.py (device-resident):
#   bash tools/ab_probe.sh "c2 c5" build/variants/a/libplzgpu.so build/variants/b/libplzgpu.so ...
# each workload x build twice, interleaved.
WL=$1; shift
for rep in 1 2; do
  for w in $WL; do
    for lib in "$@"; do
      echo "$w $(basename $(dirname $lib)) $(PLZGPU_LIB=$lib timeout 300 python tools/probe.py $w 5 2>&1 | grep -v generated | tr '\n' ' ')"
    done
  done
done
