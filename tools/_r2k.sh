mkdir -p gpurun_out
python bench.py --no-extras --op drelu_rss --steps 200 > gpurun_out/r2k_rss.json 2>&1
python bench.py --no-extras --op relu_rss --steps 200 >> gpurun_out/r2k_rss.json 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "rss" > gpurun_out/r2k_gputest.log 2>&1
cut -c1-300 gpurun_out/r2k_rss.json; tail -2 gpurun_out/r2k_gputest.log
