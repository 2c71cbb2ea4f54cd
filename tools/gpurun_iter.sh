# Iteration run on one B200: bash tools/gpurun_iter.sh TAG "pytest -k expr" "probe workloads" [ncu kernel regex]
# GPU tests (filtered), device-resident probes, optional ncu capture of one kernel on c5.
TAG=$1; K=${2:-"parity or golden or fullsize_bit_exact_vs_reference or shards or hostpaths"}; WL=${3:-"c2 c5"}; NK=$4
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_gputest.log
for w in $WL; do timeout 300 python tools/probe.py $w 5 2>&1 | grep -v generated | sed "s/^/$w /"; done
if [ -n "$NK" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$NK" -s ${NCU_SKIP:-3} -c 1 -o gpurun_out/${TAG}_ncu python tools/probe.py ${NCU_WL:-c5} 1 > /dev/null 2>&1; echo ncu rc=$?
fi
