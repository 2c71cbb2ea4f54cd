# ncu capture of the grouped first pass on c2
mkdir -p gpurun_out
PLZGPU_GROUP_ROWS=16 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:plz_groupmatch -s 1 -c 1 -o gpurun_out/prof_gm_r2k python tools/probe.py c2 1 > gpurun_out/r2k.log 2>&1
tail -3 gpurun_out/r2k.log
