for r in 1 2 3; do
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r5j_cur_$r.log 2>&1
for v in val valbc bc; do PGX_LIB=$PWD/exp/libpgx_$v.so timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r5j_${v}_$r.log 2>&1; done
done
PGX_LIB=$PWD/exp/libpgx_valbc.so timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_c5.py tests/test_gpu_properties.py -x -q -p no:cacheprovider > gpurun_out/r5j_tests.log 2>&1; echo "rc=$?"
