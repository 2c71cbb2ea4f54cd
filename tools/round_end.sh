# Round-end refresh on one B200: every GPU test, smoke(), then the profiling recipe
# (bench line, reference arm, launch list, one ncu capture per hot kernel).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=3 > gpurun_out/final_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/final_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/profile_round.sh ${1:-r2} > gpurun_out/profile_round.log 2>&1; echo "profile rc=$?"
tail -c 400 gpurun_out/bench_${1:-r2}.json
