set -x
timeout 600 python tools/probe.py C3 5 > gpurun_out/r3y_bu.log 2>&1
timeout 600 python tools/probe.py C3 5 pull_min_edges=1025 > gpurun_out/r3y_push.log 2>&1
for v in u1 u4 r2; do PGX_LIB=$PWD/exp/libpgx_$v.so timeout 600 python tools/probe.py C3 5 > gpurun_out/r3y_$v.log 2>&1; done
timeout 600 python tools/probe.py C3 5 pull_min_edges=0 > gpurun_out/r3y_buall.log 2>&1
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_properties.py -x -q -p no:cacheprovider > gpurun_out/r3y_tests.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/r3y_tests.log
