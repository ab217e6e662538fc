set -x
timeout 900 python tools/seg_check.py C2 shipped shipped shipped > gpurun_out/r3j_cur.log 2>&1
PGX_LIB=$PWD/exp/libpgx_head.so timeout 900 python tools/seg_check.py C2 shipped shipped shipped > gpurun_out/r3j_head.log 2>&1
timeout 900 python tools/seg_check.py C2 shipped shipped shipped > gpurun_out/r3j_cur2.log 2>&1
