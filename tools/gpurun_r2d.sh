# round-2 iteration: GPU tests, probes, ncu of decode/assemble, c1 launch list
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/r2d_gputest.log 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/r2d_gputest.log
for w in c2 c5 c4 c1 c3; do timeout 300 python tools/probe.py $w 5; done > gpurun_out/r2d_probe.txt 2>&1
grep -v generated gpurun_out/r2d_probe.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:plz_decode_kernel -s 3 -c 1 \
    -o gpurun_out/prof_plz_decode_kernel_r2d python tools/probe.py c2 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:plz_assemble -s 1 -c 1 \
    -o gpurun_out/prof_plz_assemble_r2d python tools/probe.py c2 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:plz_ --csv \
    --log-file gpurun_out/launches_c1_r2d.csv python tools/probe.py c1 1 > /dev/null 2>&1
ls -la gpurun_out | tail -6
