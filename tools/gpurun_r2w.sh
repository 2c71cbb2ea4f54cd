# Kernel I: two steps per lane (8 per round) for W > 128
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "parity or golden or fullsize_bit_exact_vs_reference or shards or tools or dropin" > gpurun_out/r2w_gputest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2w_gputest.log
for w in c2 c3 c4 c5; do timeout 300 python tools/probe.py $w 5 2>&1 | grep "^compress"; done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:plz_bitmatch_kernel<.*16>' -s 1 -c 1 -o gpurun_out/prof_bm_r2w python tools/probe.py c2 1 > /dev/null 2>&1; echo ncu rc=$?
