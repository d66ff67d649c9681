mkdir -p gpurun_out
export VARIANT_LIST='[{}, {"BC_P2_DIST": 0}, {"BC_TPB_T": 576}, {"BC_TPB_T": 640}, {"BC_TBL_V2": 0, "BC_P2_DIST": 0}]'
python tools/variants.py time > gpurun_out/r2d_variants.log 2>&1
cp gpurun_out/variants.json gpurun_out/r2d_variants_drelu.json
VARIANT_OP=relu python tools/variants.py time > gpurun_out/r2d_variants_relu.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_parity or fallback or full_size_exact or config1 or party_phases or high_global" > gpurun_out/r2d_gputest.log 2>&1
timeout 900 python -m pytest tests/test_gpu_party_peer.py tests/test_gpu_multiproc_bench.py tests/test_gpu_fault.py -x -q >> gpurun_out/r2d_gputest.log 2>&1
tail -4 gpurun_out/r2d_gputest.log; cat gpurun_out/r2d_variants.log gpurun_out/r2d_variants_relu.log
