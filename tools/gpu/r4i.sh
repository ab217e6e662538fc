set -x
timeout 600 python tools/probe.py C3 5 > gpurun_out/r4i_bu.log 2>&1
for v in t u4; do PGX_LIB=$PWD/exp/libpgx_$v.so timeout 600 python tools/probe.py C3 3 > gpurun_out/r4i_$v.log 2>&1; done
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_properties.py -x -q -p no:cacheprovider > gpurun_out/r4i_tests.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/r4i_tests.log
