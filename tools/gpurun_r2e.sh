# round-2 iteration: GPU tests, probes, ncu of decode/assemble, c1 launch list
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/r2e_gputest.log 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/r2e_gputest.log
for w in c2 c5 c4 c1 c3; do timeout 300 python tools/probe.py $w 5; done > gpurun_out/r2e_probe.txt 2>&1
grep -v generated gpurun_out/r2e_probe.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:plz_decode_kernel -s 3 -c 1 \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:plz_assemble -s 1 -c 1 \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:plz_ --csv \
ls -la gpurun_out | tail -6
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:plz_ --csv \
    --log-file gpurun_out/launches_c1_r2e.csv python tools/probe.py c1 1 > /dev/null 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r2e_bench.json
