mkdir -p gpurun_out
export VARIANT_LIST='[{}, {"BC_RELU_PRE": 1}]'
VARIANT_OP=relu python tools/variants.py time > gpurun_out/r2i_variants_relu.log 2>&1
BICOPTOR_LIB=paper_2309_04909_b200/variants/lib_default.so python tools/time_ops.py drelu drelu:mode=literal relu:mode=literal > gpurun_out/r2i_time.log 2>&1
BICOPTOR_LIB=paper_2309_04909_b200/variants/lib_relu_pre1.so python tools/time_ops.py relu relu:mode=literal >> gpurun_out/r2i_time.log 2>&1
BICOPTOR_LIB=paper_2309_04909_b200/variants/lib_relu_pre1.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_parity or fallback or full_size_exact or high_global" > gpurun_out/r2i_gputest.log 2>&1
cat gpurun_out/r2i_variants_relu.log gpurun_out/r2i_time.log; tail -2 gpurun_out/r2i_gputest.log
