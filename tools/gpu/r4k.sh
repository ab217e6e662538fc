PGX_LIB=$PWD/exp/libpgx_t.so timeout 600 python tools/probe.py C3 2 > gpurun_out/r4k_t.log 2>&1
timeout 600 python tools/probe.py C3 5 > gpurun_out/r4k_bu.log 2>&1
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_properties.py -x -q -p no:cacheprovider > gpurun_out/r4k_tests.log 2>&1; echo "rc=$?"
