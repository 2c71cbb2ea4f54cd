# TMA Kernel III ring sizes (6/8/16 KiB per warp) vs the register-staged kernel
mkdir -p gpurun_out
PLZGPU_LIB=build/variants/r8/libplzgpu.so timeout 900 python -m pytest tests -m gpu -x -q -k "parity or golden or fullsize_bit_exact_vs_reference or shards or hostpaths" > gpurun_out/r2t_gputest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2t_gputest.log
for v in r6 r8 r16; do
  for w in c5 c2; do
    echo "$v $w"; PLZGPU_LIB=build/variants/$v/libplzgpu.so timeout 600 ncu --metrics gpu__time_duration.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
      --clock-control none -k regex:plz_assemble -s 1 -c 1 --csv python tools/probe.py $w 1 2>/dev/null | grep -E 'assemble' | awk -F'","' '{print $5, $(NF-2), $NF}'
  done
done
