# Developer A/B of one eval_map variant library against the in-tree build on a GPU box:
# map-parity GPU tests run against the variant, then alternating timing runs.
#   gpurun -- 'bash tools/ab_variant_run.sh TAG variants/libplt_x.so'
set -u
tag=$1; lib=$2
PLT_LIB=$lib timeout 900 python -m pytest tests/test_gpu_map_splat.py tests/test_gpu_fitted_maps.py tests/test_gpu_edge_cases.py tests/test_gpu_fused_splat.py -q -x > gpurun_out/${tag}_tests.log 2>&1; echo "exit $?" >> gpurun_out/${tag}_tests.log; tail -3 gpurun_out/${tag}_tests.log
bash tools/ab_map.sh $tag paper_2605_04017_b200/libplt.so $lib
