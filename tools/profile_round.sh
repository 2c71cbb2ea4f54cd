#!/bin/bash
# Round profiling recipe (run under gpurun, one GPU): bench line, launch list,
# one full ncu capture per hot kernel.  Outputs land in gpurun_out/.
set -x
R=${1:-r1}
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$R.json 2>&1
PLZGPU_NO_PIPE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:plz_ -c 400 --csv \
    --log-file gpurun_out/launches_$R.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
# Kernel I: the first bitmap pass (16 rows) of the second compress call
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:plz_bitmatch_kernel<.*16>' -s 1 -c 1 \
    -o gpurun_out/prof_plz_bitmatch_$R python tools/probe.py c2 1 > /dev/null 2>&1
for k in plz_scan plz_assemble plz_headers plz_parse plz_decode_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/prof_${k}_$R python tools/probe.py c2 1 > /dev/null 2>&1
done
# the cuSZ use case: the quantizer's z-walk and the inverse's strided scan
for k in plz_lorenzo_tiled plz_scan_strided; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/prof_${k}_$R python tools/cusz_pipeline.py --steps 1 > /dev/null 2>&1
done
ls -la gpurun_out
