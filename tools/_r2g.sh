mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "materialize2 or literal" > gpurun_out/r2g_gputest.log 2>&1
python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
bash tools/profile_round.sh r2g > gpurun_out/r2g_profile.log 2>&1
tail -3 gpurun_out/r2g_gputest.log; ls gpurun_out/summary
