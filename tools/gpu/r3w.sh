set -x
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3w_cur.log 2>&1
PGX_LIB=$PWD/exp/libpgx_v14.so timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3w_v14.log 2>&1
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3w_cur2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:min_run_kernel -c 1 -o gpurun_out/r3w_ncu_c3 python tools/probe.py C3 1 > gpurun_out/r3w_ncu_c3.log 2>&1; echo "ncu rc=$?"
