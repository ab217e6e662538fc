set -x
PGX_LIB=$PWD/exp/libpgx_oldrun.so timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3b_old.log 2>&1
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3b_cur.log 2>&1
