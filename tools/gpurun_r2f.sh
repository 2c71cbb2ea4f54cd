# round-2: latency-mode classify check (c1), multi-rank bench paths on one GPU
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or golden or dropin or hostpaths" > gpurun_out/r2f_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2f_gputest.log
for w in c1 c2; do timeout 300 python tools/probe.py $w 5; done 2>&1 | grep -v generated
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:plz_ --csv --log-file gpurun_out/launches_c1_r2f.csv python tools/probe.py c1 1 > /dev/null 2>&1
BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --standalone --nproc-per-node 2 bench.py --gpus 2 --steps 3 --warmup 1 --no-pageable > gpurun_out/r2f_bench_n2.json 2> gpurun_out/r2f_bench_n2.err; echo "bench n2 rc=$?"
tail -c 2500 gpurun_out/r2f_bench_n2.json; tail -5 gpurun_out/r2f_bench_n2.err
timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 2 bench.py --impl reference --gpus 2 --steps 2 --warmup 0 > gpurun_out/r2f_ref_n2.json 2>&1; echo "ref n2 rc=$?"
tail -c 600 gpurun_out/r2f_ref_n2.json
