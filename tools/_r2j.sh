mkdir -p gpurun_out
python tools/time_ops.py drelu relu drelu:mode=literal relu:mode=literal drelu:lx=31,f=0 relu:lx=31,f=0 > gpurun_out/r2j_time.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > gpurun_out/r2j_gputest.log 2>&1
cat gpurun_out/r2j_time.log; tail -2 gpurun_out/r2j_gputest.log
