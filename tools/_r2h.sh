mkdir -p gpurun_out
export VARIANT_LIST='[{}, {"BC_ILV": 1}]'
python tools/variants.py time > gpurun_out/r2h_variants.log 2>&1
BICOPTOR_LIB=paper_2309_04909_b200/variants/lib_ilv1.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_parity or fallback or full_size_exact or sharding or high_global or config1" > gpurun_out/r2h_gputest_ilv.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_parity or fallback or full_size_exact or high_global or materialize2" > gpurun_out/r2h_gputest.log 2>&1
cat gpurun_out/r2h_variants.log; tail -2 gpurun_out/r2h_gputest_ilv.log gpurun_out/r2h_gputest.log
