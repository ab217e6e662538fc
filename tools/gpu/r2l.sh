set -x
export PGX_LIB=$PWD/exp/libpgx_b1024.so
timeout 900 python tools/seg_check.py C2,C5 off shipped L=14 L=15 > gpurun_out/r2l_seg.log 2>&1; echo "seg rc=$?"
timeout 600 python tools/probe.py C1,C3,C4 3 > gpurun_out/r2l_probe.log 2>&1; echo "probe rc=$?"
unset PGX_LIB
timeout 600 python tools/probe.py C1,C3,C4 3 > gpurun_out/r2l_probe512.log 2>&1; echo "probe512 rc=$?"
