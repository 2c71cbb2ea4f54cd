# compute-sanitizer memcheck / synccheck over the decode paths changed in session 4
# (token table per width, one __syncwarp per wave pair), plus the standard cases
mkdir -p gpurun_out
for tool in memcheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --num-cuda-barriers 65536 --print-limit 20 \
      python -m pytest tests/test_gpu_parity.py -q -x -k "token_table or configs_bit_exact and quant" \
      > gpurun_out/san_dec_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_dec_$tool.log | head -4
done
bash tools/sanitize.sh
