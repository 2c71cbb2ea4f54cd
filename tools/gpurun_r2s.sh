# ncu capture of the TMA Kernel III on c5
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:plz_assemble_tma -s 1 -c 1 -o gpurun_out/prof_asmtma_r2s python tools/probe.py c5 1 > /dev/null 2>&1; echo ncu rc=$?
