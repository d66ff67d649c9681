mkdir -p gpurun_out
python tools/debug_transcript.py guard 8 > gpurun_out/r2e_debug.log 2>&1
python tools/debug_transcript.py literal 20 >> gpurun_out/r2e_debug.log 2>&1
python tools/time_ops.py drelu drelu:mode=literal relu relu:mode=literal drelu:mode=literal,rounds=8 > gpurun_out/r2e_time.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "literal or l16x7f0l or l64x7f24l" > gpurun_out/r2e_gputest.log 2>&1
timeout 900 python -m pytest tests/test_gpu_party_peer.py tests/test_gpu_multiproc_bench.py tests/test_gpu_fault.py -x -q >> gpurun_out/r2e_gputest.log 2>&1
cat gpurun_out/r2e_debug.log | head -40; cat gpurun_out/r2e_time.log; tail -5 gpurun_out/r2e_gputest.log
