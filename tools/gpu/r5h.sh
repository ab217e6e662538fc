timeout 900 python tools/seg_check.py C5 shipped > gpurun_out/r5h_cur.log 2>&1
PGX_LIB=$PWD/exp/libpgx_nosv.so timeout 900 python tools/seg_check.py C5 shipped > gpurun_out/r5h_nosv.log 2>&1
