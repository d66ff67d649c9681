mkdir -p gpurun_out
python bench.py > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2p_reference.json 2> gpurun_out/r2p_reference.err
timeout 900 python -m pytest tests/test_gpu_multiproc_bench.py tests/test_gpu_party_peer.py -q > gpurun_out/r2p_gputest.log 2>&1
cut -c1-300 gpurun_out/r2p_bench.json; cut -c1-300 gpurun_out/r2p_reference.json; tail -2 gpurun_out/r2p_gputest.log
