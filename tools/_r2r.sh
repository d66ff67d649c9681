mkdir -p gpurun_out
TIME_LX=7 python tools/time_party_fp.py > gpurun_out/r2r_party.log 2>&1
python tools/time_party_fp.py >> gpurun_out/r2r_party.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_party_peer.py tests/test_gpu_party_staged.py tests/test_gpu_fault.py tests/test_gpu_sanitizer.py tests/test_gpu_multiproc_bench.py -x -q -k "party or fuzz or fault or sanitizer or high_global or fallback or abi or bench" > gpurun_out/r2r_gputest.log 2>&1
cat gpurun_out/r2r_party.log; tail -3 gpurun_out/r2r_gputest.log
