# session-3 baseline at HEAD: all GPU tests, bench (c5), reference arm, probes of every config
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/s3a_gputest.log 2>&1; echo "pytest rc=$?"
tail -14 gpurun_out/s3a_gputest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s3a_bench.json 2> gpurun_out/s3a_bench.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/s3a_bench.json; tail -5 gpurun_out/s3a_bench.err
for w in c1 c2 c3 c4 c5; do timeout 300 python tools/probe.py $w 5 2>&1 | grep -v generated; done
