set -x
PGX_LIB=$PWD/exp/libpgx_nospec.so timeout 900 python tools/seg_check.py C2,C5,C3 shipped > gpurun_out/r2u_nospec.log 2>&1; echo "nospec rc=$?"
timeout 900 python tools/seg_check.py C2,C5,C3 shipped > gpurun_out/r2u_spec.log 2>&1; echo "spec rc=$?"
