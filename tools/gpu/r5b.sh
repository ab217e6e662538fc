timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r5b_cur.log 2>&1
PGX_LIB=$PWD/exp/libpgx_bc.so timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r5b_bc.log 2>&1
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r5b_cur2.log 2>&1
PGX_LIB=$PWD/exp/libpgx_bc.so timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r5b_bc2.log 2>&1
