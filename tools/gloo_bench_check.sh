mkdir -p gpurun_out
for N in 2 4; do
BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 3 --warmup 3 > gpurun_out/gloo_bench_$N.json 2> gpurun_out/gloo_bench_$N.err; echo "N=$N rc=$?"
tail -c 600 gpurun_out/gloo_bench_$N.json
done
