# decode: wave chase only where a source lies in the wave; cached container lookup
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or golden or fullsize_bit_exact_vs_reference or shards or hostpaths" > gpurun_out/r2l_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2l_gputest.log
for w in c2 c3 c4 c5; do timeout 300 python tools/probe.py $w 5 2>&1 | grep decompress; done
