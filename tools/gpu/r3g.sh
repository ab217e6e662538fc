set -x
timeout 900 python tools/seg_check.py C2,C5,C3 shipped > gpurun_out/r3g_cur.log 2>&1
PGX_LIB=$PWD/exp/libpgx_v6.so timeout 900 python tools/seg_check.py C2,C5,C3 shipped > gpurun_out/r3g_v6.log 2>&1
PGX_LIB=$PWD/exp/libpgx_v8.so timeout 900 python tools/seg_check.py C2,C5,C3 off shipped > gpurun_out/r3g_v8.log 2>&1
