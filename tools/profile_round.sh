#!/bin/bash
# Round profiling recipe (run under gpurun, one GPU): bench line, launch list,
# one full ncu capture per hot kernel on the bench workload (c5).  Outputs land
# in gpurun_out/; tools/summarize_profiles.py <round> turns them into profiles/<round>/.
set -x
R=${1:-r2}
W=${2:-c5}
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$R.json 2>&1
# every launch of one compress + decompress step (serialised, cold): shares, not absolutes
PLZGPU_NO_PIPE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:plz_ --csv \
    --log-file gpurun_out/launches_$R.csv python tools/probe.py $W 1 > /dev/null 2>&1
# Kernel I: the first bitmap pass (12 rows) of the second compress call
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:plz_bitmatch_kernel<.*12>' -s 1 -c 1 \
    -o gpurun_out/prof_plz_bitmatch_$R python tools/probe.py $W 1 > /dev/null 2>&1
for k in plz_scan plz_assemble plz_headers plz_parse; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/prof_${k}_$R python tools/probe.py $W 1 > /dev/null 2>&1
done
# the decode kernel instance that takes the S = 2 containers (<kPipe = 0, kKindS2 = 1>; the
# other widths' instances only return), of the second decompress call
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:plz_decode_kernel<[^>]*0, [^>]*1>' -s 1 -c 1 \
    -o gpurun_out/prof_plz_decode_kernel_$R python tools/probe.py $W 1 > /dev/null 2>&1
ls -la gpurun_out
