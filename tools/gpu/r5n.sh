for r in 1 2; do
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r5n_cur_$r.log 2>&1
PGX_LIB=$PWD/exp/libpgx_pairs.so timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r5n_pairs_$r.log 2>&1
done
PGX_LIB=$PWD/exp/libpgx_pairs.so timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_c5.py -x -q -p no:cacheprovider > gpurun_out/r5n_tests.log 2>&1; echo "rc=$?"
