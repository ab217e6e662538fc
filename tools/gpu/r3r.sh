set -x
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3r_cur.log 2>&1
PGX_LIB=$PWD/exp/libpgx_v12.so timeout 900 python tools/seg_check.py C2,C5 off shipped > gpurun_out/r3r_v12.log 2>&1
