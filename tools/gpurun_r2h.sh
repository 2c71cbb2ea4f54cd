set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or golden or dropin or hostpaths or fullsize" > gpurun_out/r2h_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2h_gputest.log
for w in c2 c5 c3; do timeout 300 python tools/probe.py $w 5; done 2>&1 | grep -v generated
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:plz_decode_kernel -s 3 -c 1 \
    -o gpurun_out/prof_plz_decode_kernel_r2h python tools/probe.py c5 1 > /dev/null 2>&1
ls gpurun_out | grep r2h
