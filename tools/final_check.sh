# Round-end style validation on one B200: every GPU test, smoke(), bench (+ reference arm)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/final_gputest.log 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/final_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/final_bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'dec', d['decompress']['value'], 'e2e', d['e2e']['value'], d['e2e']['decompress']['value'], 'frac', d['roofline']['frac'], 'III', d['stages']['kernel_III']['frac'], 'dec_frac', d['roofline_decompress']['frac'], 'clocks', d['clocks'])"
timeout 900 python bench.py --impl reference > gpurun_out/final_bench_ref.json 2>&1; echo "ref rc=$?"; tail -c 300 gpurun_out/final_bench_ref.json
