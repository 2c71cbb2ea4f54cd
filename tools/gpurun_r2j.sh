# group-pass first check: parity + timings with each first-pass variant
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or golden or fullsize_bit_exact_vs_reference" > gpurun_out/r2j_gputest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2j_gputest.log
for v in 0 16 12; do for w in c2 c3 c4; do PLZGPU_GROUP_ROWS=$v timeout 300 python tools/probe.py $w 5 2>&1 | grep compress; done; done
