mkdir -p gpurun_out
python tools/time_ops.py drelu:lx=31,f=0 relu:lx=31,f=0 drelu:lx=31,f=0,mode=literal drelu drelu drelu > gpurun_out/r2n_time.log 2>&1
python tools/time_party_fp.py > gpurun_out/r2n_party_fp.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_party_peer.py -x -q -k "large or full_precision or high_global or party or fuzz" > gpurun_out/r2n_gputest.log 2>&1
cat gpurun_out/r2n_time.log; tail -1 gpurun_out/r2n_party_fp.log; tail -2 gpurun_out/r2n_gputest.log
