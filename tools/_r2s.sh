mkdir -p gpurun_out
./tools/intpipe_bench > gpurun_out/r2s_intpipe.json 2> gpurun_out/r2s_intpipe.err
python tools/time_party_fp.py > gpurun_out/r2s_party.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_party_peer.py tests/test_gpu_sanitizer.py -x -q -k "party or large or full_precision or high_global or sanitizer" > gpurun_out/r2s_gputest.log 2>&1
cat gpurun_out/r2s_intpipe.json | head -30; cat gpurun_out/r2s_party.log; tail -3 gpurun_out/r2s_gputest.log
