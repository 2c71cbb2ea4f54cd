# round-2 iteration: GPU tests, device-resident probes, ncu of the changed kernels
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r2c_gputest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r2c_gputest.log
for w in c2 c5 c4 c1 c3; do timeout 300 python tools/probe.py $w 5; done > gpurun_out/r2c_probe.txt 2>&1
cat gpurun_out/r2c_probe.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:plz_decode_kernel -s 1 -c 1 \
    -o gpurun_out/prof_plz_decode_kernel_r2c python tools/probe.py c2 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:plz_assemble -s 1 -c 1 \
    -o gpurun_out/prof_plz_assemble_r2c python tools/probe.py c2 1 > /dev/null 2>&1
ls -la gpurun_out | tail
