set -x
nproc; free -g | head -2; nvidia-smi --query-gpu=name,memory.total --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2_gputest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r2_gputest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2_bench.json; tail -20 gpurun_out/r2_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref.json 2>&1; echo "ref rc=$?"
cat gpurun_out/r2_bench_ref.json | tail -c 2000
