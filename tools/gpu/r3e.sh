set -x
PGX_LIB=$PWD/exp/libpgx_f1d.so timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3e_f1d.log 2>&1
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3e_cur.log 2>&1
