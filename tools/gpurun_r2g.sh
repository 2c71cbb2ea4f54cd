set -x
timeout 2400 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/r2g_gputest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/r2g_gputest.log
timeout 300 python tools/probe.py c1 5 2>&1 | grep -v generated
bash tools/profile_round.sh r2 c5
