set -x
for v in o2 exp o1; do
PGX_LIB=$PWD/exp/libpgx_$v.so timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3q_$v.log 2>&1
PGX_LIB=$PWD/exp/libpgx_$v.so timeout 600 python tools/probe.py C3,C4 3 > gpurun_out/r3q_probe_$v.log 2>&1
done
timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3q_cur.log 2>&1
timeout 600 python tools/probe.py C3,C4 3 > gpurun_out/r3q_probe_cur.log 2>&1
