# session-3: source-level ncu captures of decode (c2, c5) and Kernel III (c5) at HEAD
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:plz_decode_kernel -s 3 -c 1 -o gpurun_out/s3b_dec_c5 python tools/probe.py c5 1 > /dev/null 2>&1; echo ncu rc=$?
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:plz_decode_kernel -s 3 -c 1 -o gpurun_out/s3b_dec_c2 python tools/probe.py c2 1 > /dev/null 2>&1; echo ncu rc=$?
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:plz_assemble -s 1 -c 1 -o gpurun_out/s3b_asm_c5 python tools/probe.py c5 1 > /dev/null 2>&1; echo ncu rc=$?
ls -la gpurun_out
