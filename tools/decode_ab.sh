# decode A/B: parity tests on the in-tree build, then probe c5 and c3 at I = 16 / 8 per build
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "golden or parity or fullsize or decode" > gpurun_out/dec_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/dec_tests.log
for rep in 1 2; do
for cfg in "c5 2" "c3 16" "c3 8"; do
  set -- $cfg
  for lib in build/variants/base/libplzgpu.so paper_2304_07342_b200/lib/libplzgpu.so; do
    echo "$1 I=$2 $lib $(PROBE_I=$2 PLZGPU_LIB=$lib timeout 300 python tools/probe.py $1 5 2>&1 | grep -v generated | tr '\n' ' ')"
  done
done
done
