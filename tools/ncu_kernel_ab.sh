#!/bin/bash
# Per-kernel duration / DRAM throughput of one kernel across library builds (ncu, c5 probe):
#   bash tools/ncu_kernel_ab.sh KERNEL_REGEX WORKLOAD lib1.so lib2.so ...
K=$1; W=$2; shift 2
for lib in "$@"; do
  PLZGPU_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum \
      --clock-control none -k "regex:$K" --csv python tools/probe.py $W 1 2>/dev/null | grep -E "gpu__time|dram__|inst_exec" | \
      awk -F'","' -v L=$(basename $(dirname $lib)) '{gsub(/"/,"",$NF); print L, $(NF-2), $NF}'
done
