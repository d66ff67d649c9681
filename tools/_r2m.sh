mkdir -p gpurun_out
python tools/time_ops.py drelu:lx=31,f=0 relu:lx=31,f=0 drelu:lx=31,f=0,mode=literal > gpurun_out/r2m_time.log 2>&1
python tools/time_party_fp.py > gpurun_out/r2m_party_fp.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -k "large or full_precision or high_global or party_phases or fuzz" > gpurun_out/r2m_gputest.log 2>&1
cat gpurun_out/r2m_time.log; tail -5 gpurun_out/r2m_party_fp.log; tail -2 gpurun_out/r2m_gputest.log
