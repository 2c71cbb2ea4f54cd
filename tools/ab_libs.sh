#!/bin/bash
# A/B of library builds on one box: bash tools/ab_libs.sh build/var/a.so build/var/b.so ...
# prints device-resident compress / decompress GB/s (c2) per build, twice, interleaved.
for rep in 1 2; do
  for lib in "$@"; do
    PLZGPU_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
    python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$lib', round(d['value'], 2), round(d['decompress']['value'], 1))" || tail -2 gpurun_out/ab.err
  done
done
