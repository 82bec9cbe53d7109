set -u
PLT_LIB=variants/libplt_pair.so timeout 900 python -m pytest tests/test_gpu_map_splat.py tests/test_gpu_fitted_maps.py tests/test_gpu_edge_cases.py tests/test_gpu_fused_splat.py -q -x > gpurun_out/pair_tests.log 2>&1; echo "exit $?" >> gpurun_out/pair_tests.log; tail -3 gpurun_out/pair_tests.log
bash tools/ab_map.sh ab_pair paper_2605_04017_b200/libplt.so variants/libplt_pair.so
