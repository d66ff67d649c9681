mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2f_gputest.log 2>&1
tail -5 gpurun_out/r2f_gputest.log; tail -2 gpurun_out/r2f_smoke.log
