set -x
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3h_cur.log 2>&1
PGX_LIB=$PWD/exp/libpgx_v9.so timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3h_v9.log 2>&1
timeout 600 python tools/probe.py C3,C1,C4 3 > gpurun_out/r3h_probe_cur.log 2>&1
PGX_LIB=$PWD/exp/libpgx_v9.so timeout 600 python tools/probe.py C3,C1,C4 3 > gpurun_out/r3h_probe_v9.log 2>&1
