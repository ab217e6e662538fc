set -x
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3a_cur.log 2>&1
PGX_LIB=$PWD/exp/libpgx_v2.so timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3a_v2.log 2>&1
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3a_cur2.log 2>&1
