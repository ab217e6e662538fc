for r in 1 2; do
timeout 600 python tools/probe.py C3 5 > gpurun_out/r5f_cur_$r.log 2>&1
for v in pipe pipe4; do PGX_LIB=$PWD/exp/libpgx_$v.so timeout 600 python tools/probe.py C3 5 > gpurun_out/r5f_${v}_$r.log 2>&1; done
done
PGX_LIB=$PWD/exp/libpgx_pipet.so timeout 600 python tools/probe.py C3 2 > gpurun_out/r5f_pipet.log 2>&1
PGX_LIB=$PWD/exp/libpgx_pipe.so timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_properties.py -x -q -p no:cacheprovider -k "sssp or golden or random or large" > gpurun_out/r5f_tests.log 2>&1; echo "rc=$?"
