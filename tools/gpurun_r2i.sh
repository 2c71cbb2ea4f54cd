set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r2i_gputest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r2i_gputest.log
for w in c1 c2 c3 c4 c5; do timeout 300 python tools/probe.py $w 5; done 2>&1 | grep -v generated
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2i.json 2> gpurun_out/bench_r2i.err; echo "bench rc=$?"
cat gpurun_out/bench_r2i.json
