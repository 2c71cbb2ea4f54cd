mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:plz_decode_kernel<[^>]*0, [^>]*1>' -s 1 -c 1 \
    -o gpurun_out/prof_plz_decode_kernel_r2 python tools/probe.py c5 1 > gpurun_out/dec_prof.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/dec_prof.log
timeout 900 python tools/config_sweep.py --cpu > gpurun_out/config_sweep.jsonl 2> gpurun_out/config_sweep.err; echo "sweep rc=$?"
