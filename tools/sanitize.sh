# compute-sanitizer passes over small compress/decompress workloads (one B200)
mkdir -p gpurun_out
cat > /tmp/san_case.py <<'PY'
import sys, os
sys.path.insert(0, "."); sys.path.insert(0, "tests"); sys.path.insert(0, "oracle")
import torch, inputs
from paper_2304_07342_b200 import plz
for S, C, W, I, kind, n in [(2, 2048, 255, 2, "quant", 300000), (1, 4096, 128, 1, "runs", 200000),
                            (4, 1024, 255, 4, "quant", 200000), (2, 1024, 64, 1, "alpha", 150000)]:
    data = inputs.make(kind, n, 3, S)
    p = plz.validate(plz.Params(S, W, C, I))
    d = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
    img = plz.compress(d, p)
    back = plz.decompress_bytes(img)
    assert bytes(back.cpu().numpy().tobytes()) == data
    himg = plz.compress(data, p)
    assert plz.decompress_bytes(himg) == data
# batched Kernel III (>= 16 Ki chunks)
data = inputs.make("quant", 17000 * 2048, 4, 1)
p = plz.validate(plz.Params(1, 64, 1024, 1, 1021 * 1024))
img = plz.compress(torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda(), p)
assert bytes(plz.decompress_bytes(img).cpu().numpy().tobytes()) == data
print("sanitize case ok")
PY
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --num-cuda-barriers 65536 --print-limit 20 python /tmp/san_case.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Invalid|sanitize case" gpurun_out/san_$tool.log | head -8
done
