mkdir -p gpurun_out
export VARIANT_LIST='[{}, {"BC_HB_UNROLL": 2}, {"BC_CHACHA_UNROLL": 3}]'
python tools/variants.py time > gpurun_out/r2o_variants.log 2>&1
VARIANT_OP=relu python tools/variants.py time > gpurun_out/r2o_variants_relu.log 2>&1
cat gpurun_out/r2o_variants.log gpurun_out/r2o_variants_relu.log
