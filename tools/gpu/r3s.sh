set -x
for b in 768 896; do
PGX_LIB=$PWD/exp/libpgx_b$b.so timeout 900 python tools/seg_check.py C2,C5 shipped > gpurun_out/r3s_b$b.log 2>&1
PGX_LIB=$PWD/exp/libpgx_b$b.so timeout 600 python tools/probe.py C3,C4,C1 3 > gpurun_out/r3s_probe_b$b.log 2>&1
done
