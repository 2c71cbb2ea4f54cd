# Kernel III variants: duration + DRAM throughput (ncu) on c5 and c2
mkdir -p gpurun_out
for v in asm_orig asm_b6 asm_b8; do
  for w in c5 c2; do
    PLZGPU_LIB=build/variants/$v/libplzgpu.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active \
      --clock-control none -k regex:plz_assemble -s 1 -c 1 --csv python tools/probe.py $w 1 2>/dev/null | grep -E '"plz_assemble|assemble' | awk -F'","' -v v=$v -v w=$w '{print v, w, $(NF-2), $NF}'
  done
done
PLZGPU_LIB=build/variants/asm_b6/libplzgpu.so timeout 600 python -m pytest tests -m gpu -x -q -k "parity or golden or fullsize_bit_exact_vs_reference or shards" 2>&1 | tail -2
