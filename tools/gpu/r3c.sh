set -x
PGX_LIB=$PWD/exp/libpgx_v4.so timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3c_v4.log 2>&1
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3c_cur.log 2>&1
