mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "token_table or corrupted" > gpurun_out/t2.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t2.log
bash tools/profile_round.sh r2 > gpurun_out/profile_round.log 2>&1; echo "profile rc=$?"
