for r in 1 2; do
timeout 600 python tools/probe.py C1,C2,C3,C4 5 > gpurun_out/r5e_cur_$r.log 2>&1
for v in nosc nosc_red red; do PGX_LIB=$PWD/exp/libpgx_$v.so timeout 600 python tools/probe.py C1,C2,C3,C4 5 > gpurun_out/r5e_${v}_$r.log 2>&1; done
done
timeout 900 python tools/seg_check.py C5 shipped > gpurun_out/r5e_c5_cur.log 2>&1
PGX_LIB=$PWD/exp/libpgx_nosc.so timeout 900 python tools/seg_check.py C5 shipped > gpurun_out/r5e_c5_nosc.log 2>&1
PGX_LIB=$PWD/exp/libpgx_nosc_red.so timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_properties.py tests/test_gpu_partitioned.py -x -q -p no:cacheprovider > gpurun_out/r5e_tests.log 2>&1; echo "rc=$?"
