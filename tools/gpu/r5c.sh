for r in 1 2; do
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r5c_cur_$r.log 2>&1
PGX_LIB=$PWD/exp/libpgx_lazy.so timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r5c_lazy_$r.log 2>&1
PGX_LIB=$PWD/exp/libpgx_lazybc.so timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r5c_lazybc_$r.log 2>&1
done
PGX_LIB=$PWD/exp/libpgx_lazy.so timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_c5.py tests/test_gpu_properties.py -x -q -p no:cacheprovider > gpurun_out/r5c_tests.log 2>&1; echo "rc=$?"
