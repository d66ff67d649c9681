mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2t_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2t_gputest.log 2>&1
BC_FUZZ_CASES=600 timeout 1800 python -m pytest tests/test_gpu_fuzz.py -q > gpurun_out/r2t_fuzz_long.log 2>&1
python bench.py > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err
bash tools/profile_round.sh r2t > gpurun_out/r2t_profile.log 2>&1
tail -2 gpurun_out/r2t_gputest.log; tail -2 gpurun_out/r2t_fuzz_long.log; tail -1 gpurun_out/r2t_smoke.log; cut -c1-300 gpurun_out/r2t_bench.json
