mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2l_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2l_gputest.log 2>&1
python bench.py > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err
bash tools/profile_round.sh r2l > gpurun_out/r2l_profile.log 2>&1
tail -3 gpurun_out/r2l_gputest.log; tail -1 gpurun_out/r2l_smoke.log; cut -c1-400 gpurun_out/r2l_bench.json
