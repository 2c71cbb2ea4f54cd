# decode phase A: predicated stores, hoisted payload check
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or golden or fullsize_bit_exact_vs_reference or shards or hostpaths" > gpurun_out/r2u_gputest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2u_gputest.log
for w in c2 c3 c4 c5; do timeout 300 python tools/probe.py $w 5 2>&1 | grep decompress; done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:plz_decode_kernel -s 3 -c 1 -o gpurun_out/prof_dec_r2u python tools/probe.py c2 1 > /dev/null 2>&1; echo ncu rc=$?
