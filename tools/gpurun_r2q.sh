# Kernel III through the TMA ring vs the register-staged kernel: parity + ncu duration/DRAM on c5, c2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or golden or fullsize_bit_exact_vs_reference or shards or hostpaths or dist" > gpurun_out/r2q_gputest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2q_gputest.log
for t in 0 1; do
  for w in c5 c2 c4; do
    PLZGPU_ASM_TMA=$t timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed \
      --clock-control none -k regex:plz_assemble -s 1 -c 1 --csv python tools/probe.py $w 1 2>/dev/null | grep -E 'assemble' | awk -F'","' '{print $5, $(NF-2), $NF}'
  done
done
